// pack_tc.cu — canonical A_n / A_i1 / A_i2 (App. A) -> the tensor-core "window" form used by
// spmm_tc.cu (include/vnm.h).  Pure data movement + integer logic, HBM-bound.
//
// Window form, V >= 32, 4 <= M <= 8: block b of a row becomes the 8 consecutive X^T channels
// [b*M, b*M + 8) split into two 2:4 groups (channels 0-3 "lo", 4-7 "hi").  The row's two kept values
// (block columns c0 < c1) sit at their own positions; each group is completed to exactly two entries with
// zero values at the lowest free positions.  For M = 4 two blocks form one 8-channel window and the form is
// A_n / A_i2 unchanged (col_idx is always 0,1,2,3).
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_form.cuh"
#include "vnm_internal.h"

namespace vnm {
namespace {

struct PackTcArgs {
    const uint16_t* values;
    const uint8_t* col_idx;
    const uint32_t* meta;
    uint16_t* values_tc;
    uint32_t* meta_tc;
    int32_t V, M, rows_p, rows_w, nb_pad, ld_val, ld_meta, n_mma, n_stage, ld_tc;
};

// the 8-nibble metadata word of MMA `mi` for row r (rows >= rows_p: zero weights, nibble 0x4)
__device__ uint32_t mma_word(const PackTcArgs& a, int r, int mi) {
    if (r >= a.rows_p || mi >= a.n_mma) return 0x44444444u;
    if (a.M == 4) return a.meta[static_cast<int64_t>(r) * a.ld_meta + mi];
    uint32_t w = 0;
    const uint8_t* ci_row = a.col_idx + static_cast<int64_t>(r / a.V) * a.nb_pad * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b = 4 * mi + i;
        const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
        const uint8_t* ci = ci_row + b * 4;
        const int c0 = ci[nib & 3u], c1 = ci[nib >> 2];
        w |= tc_encode_block(c0, c1, 0, 0).nibs << (8 * i);
    }
    return w;
}

// values_tc: one thread per (row, block) for M >= 5 (4 values); a row copy for M = 4
__global__ void pack_tc_values_kernel(const PackTcArgs a) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(a.rows_w) * a.nb_pad;
    if (idx >= total) return;
    const int r = static_cast<int>(idx / a.nb_pad), b = static_cast<int>(idx % a.nb_pad);
    if (a.M == 4) {
        uint32_t v = 0;
        if (r < a.rows_p) v = reinterpret_cast<const uint32_t*>(a.values + static_cast<int64_t>(r) * a.ld_val)[b];
        reinterpret_cast<uint32_t*>(a.values_tc + static_cast<int64_t>(r) * a.ld_tc)[b] = v;
        return;
    }
    uint16_t out[4] = {0, 0, 0, 0};
    if (r < a.rows_p) {
        const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
        const uint8_t* ci = a.col_idx + (static_cast<int64_t>(r / a.V) * a.nb_pad + b) * 4;
        const int c0 = ci[nib & 3u], c1 = ci[nib >> 2];
        const uint16_t v0 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b];
        const uint16_t v1 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b + 1];
        const TcBlock t = tc_encode_block(c0, c1, v0, v1);
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = t.val[q];
    }
    uint2 pk;
    pk.x = static_cast<uint32_t>(out[0]) | (static_cast<uint32_t>(out[1]) << 16);
    pk.y = static_cast<uint32_t>(out[2]) | (static_cast<uint32_t>(out[3]) << 16);
    *reinterpret_cast<uint2*>(a.values_tc + static_cast<int64_t>(r) * a.ld_tc + 4 * b) = pk;
}

// meta_tc[tile][stage][lane][k]: lane L of the M = 128 TMEM metadata layout (csrc/probes.cu MB1):
// bits 0-15 = K-groups 4h..4h+3 of row (L%8) + 16(L/16), bits 16-31 = the same of that row + 8, h = (L/8)%2
__global__ void pack_tc_meta_kernel(const PackTcArgs a) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = static_cast<int64_t>(a.rows_w / 128) * a.n_stage * 128 * 4;
    if (idx >= total) return;
    const int k = static_cast<int>(idx % 4);
    const int L = static_cast<int>((idx / 4) % 128);
    const int64_t ts = idx / 512;
    const int st = static_cast<int>(ts % a.n_stage);
    const int tile = static_cast<int>(ts / a.n_stage);
    const int mi = st * 4 + k;
    const int h = (L / 8) % 2;
    const int row_a = tile * 128 + (L % 8) + 16 * (L / 16);
    const uint32_t wa = mma_word(a, row_a, mi), wb = mma_word(a, row_a + 8, mi);
    a.meta_tc[idx] = ((wa >> (16 * h)) & 0xFFFFu) | (((wb >> (16 * h)) & 0xFFFFu) << 16);
}

}  // namespace

int launch_pack_tc(const vnm_packed& P, cudaStream_t stream) {
    const vnm_geom& g = P.g;
    PackTcArgs a;
    a.values = P.values;
    a.col_idx = P.col_idx;
    a.meta = P.meta;
    a.values_tc = P.values_tc;
    a.meta_tc = P.meta_tc;
    a.V = g.V;
    a.M = g.M;
    a.rows_p = g.rows_p;
    a.rows_w = (g.rows_p + 127) / 128 * 128;
    a.nb_pad = g.nb_pad;
    a.ld_val = g.ld_val;
    a.ld_meta = g.ld_meta;
    a.n_mma = g.nb_pad / (g.M == 4 ? 8 : 4);
    a.n_stage = (a.n_mma + 3) / 4;
    a.ld_tc = 16 * a.n_mma;
    const int64_t nv = static_cast<int64_t>(a.rows_w) * a.nb_pad;
    const int64_t nm = static_cast<int64_t>(a.rows_w / 128) * a.n_stage * 512;
    pack_tc_values_kernel<<<static_cast<unsigned>((nv + 255) / 256), 256, 0, stream>>>(a);
    count_launch();
    pack_tc_meta_kernel<<<static_cast<unsigned>((nm + 255) / 256), 256, 0, stream>>>(a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
