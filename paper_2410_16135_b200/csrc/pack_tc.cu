// pack_tc.cu — canonical A_n / A_i1 / A_i2 (App. A) -> the tensor-core "window" form used by
// spmm_tc.cu (include/vnm.h).  Pure data movement + integer logic, HBM-bound.
//
// Window form, V >= 32, 4 <= M <= 8: block b of a row becomes the 8 consecutive X^T channels
// [b*M, b*M + 8) split into two 2:4 groups (channels 0-3 "lo", 4-7 "hi").  The row's two kept values
// (block columns c0 < c1) sit at their own positions; each group is completed to exactly two entries with
// zero values at the lowest free positions.  For M = 4 two blocks form one 8-channel window and the form is
// A_n / A_i2 unchanged (col_idx is always 0,1,2,3).
//
// Window-16 form, 8 < M <= 16 with M % 4 != 0 (include/vnm.h): block b becomes the 16 channels [b*M, b*M + 16)
// as four 2:4 groups; MMA 2j + h covers the half-windows h (groups 2h, 2h+1 = channels 8h .. 8h+7) of blocks
// 4j .. 4j+3, so its B operand is the window-form one (K-group stride M rows) started 8h rows further.
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
    int32_t w16;  // window-16 form (8 < M <= 16)
};

// the 8-nibble metadata word of MMA `mi` for row r (rows >= rows_p: zero weights, nibble 0x4)
__device__ uint32_t mma_word(const PackTcArgs& a, int r, int mi) {
    if (r >= a.rows_p || mi >= a.n_mma) return 0x44444444u;
    if (a.M == 4) return a.meta[static_cast<int64_t>(r) * a.ld_meta + mi];
    uint32_t w = 0;
    const uint8_t* ci_row = a.col_idx + static_cast<int64_t>(r / a.V) * a.nb_pad * 4;
    if (a.w16) {  // MMA mi = 2j + h: half-windows h of blocks 4j .. 4j+3
        const int j = mi >> 1, h = mi & 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int b = 4 * j + i;
            if (b >= a.nb_pad) { w |= 0x44u << (8 * i); continue; }
            const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
            const uint8_t* ci = ci_row + b * 4;
            const int c0 = ci[nib & 3u], c1 = ci[nib >> 2];
            w |= ((tc_encode_block16(c0, c1, 0, 0).nibs >> (8 * h)) & 0xFFu) << (8 * i);
        }
        return w;
    }
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
    if (a.w16) {  // 8 values: half h -> MMA 2(b/4) + h, slots 4(b%4) .. +3
        uint16_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (r < a.rows_p) {
            const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
            const uint8_t* ci = a.col_idx + (static_cast<int64_t>(r / a.V) * a.nb_pad + b) * 4;
            const int c0 = ci[nib & 3u], c1 = ci[nib >> 2];
            const uint16_t v0 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b];
            const uint16_t v1 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b + 1];
            const TcBlock16 t = tc_encode_block16(c0, c1, v0, v1);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = t.val[q];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint2 pk;
            pk.x = static_cast<uint32_t>(o[4 * h]) | (static_cast<uint32_t>(o[4 * h + 1]) << 16);
            pk.y = static_cast<uint32_t>(o[4 * h + 2]) | (static_cast<uint32_t>(o[4 * h + 3]) << 16);
            *reinterpret_cast<uint2*>(a.values_tc + static_cast<int64_t>(r) * a.ld_tc + 16 * (2 * (b / 4) + h) +
                                      4 * (b % 4)) = pk;
        }
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

// ---- natural 2:4 form for M % 4 == 0, M > 8 (include/vnm.h).  A V:2:M-masked row keeps 2 values per block of
// M channels, and a block is a whole number of 4-channel groups, so every group of 4 consecutive channels holds
// at most 2 nonzeros: the masked W is 2:4-sparse in the natural channel order.  The tensor-core form is then
// the plain 2:4 packing over groups (the M = 4 layout with groups as blocks): per group the row's nonzeros at
// their own positions, completed to two entries with zeros at the lowest free positions.
struct Nat24Args {
    const uint16_t* values;
    const uint8_t* col_idx;
    const uint32_t* meta;
    uint16_t* values_tc;
    uint32_t* meta_tc;
    int32_t V, M, rows_p, rows_w, nb_pad, ld_val, ld_meta;
    int32_t ng_pad, n_mma, n_stage, ld_tc;  // groups (padded to 8), MMAs (8 groups each), stages, values per row
};

// group q of row r: 2:4 nibble (pos_a | pos_b << 2) and the two stored values (M a compile-time constant: the
// block / group arithmetic without integer division)
template <int M>
__device__ __forceinline__ uint32_t nat24_group(const Nat24Args& a, int r, int q, uint16_t* va, uint16_t* vb) {
    *va = 0;
    *vb = 0;
    const int b = 4 * q / M;
    if (r >= a.rows_p || b >= a.nb_pad) return 0x4u;
    const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
    const uint8_t* ci = a.col_idx + (static_cast<int64_t>(r / a.V) * a.nb_pad + b) * 4;
    const int base = 4 * q - b * M;
    const int c0 = ci[nib & 3u] - base, c1 = ci[nib >> 2] - base;  // block columns c0 < c1, group-relative
    const bool in0 = c0 >= 0 && c0 < 4, in1 = c1 >= 0 && c1 < 4;
    const uint16_t v0 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b];
    const uint16_t v1 = a.values[static_cast<int64_t>(r) * a.ld_val + 2 * b + 1];
    if (in0 && in1) {
        *va = v0;
        *vb = v1;
        return static_cast<uint32_t>(c0) | (static_cast<uint32_t>(c1) << 2);
    }
    if (in0 || in1) {
        const int p = in0 ? c0 : c1;
        const uint16_t v = in0 ? v0 : v1;
        const int f = p == 0 ? 1 : 0;
        if (p < f) *va = v; else *vb = v;
        return static_cast<uint32_t>(p < f ? p : f) | (static_cast<uint32_t>(p < f ? f : p) << 2);
    }
    return 0x4u;
}

// grid (ceil(nbk / 256), rows_w): thread = block b of row blockIdx.y, writing its M/4 groups (one load of the
// block's nibble word, kept columns and value pair); blocks past nb_pad write the zero groups up to ng_pad
template <int M>
__global__ void pack_nat24_values_kernel(const Nat24Args a) {
    constexpr int G = M / 4;
    const int b = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (b * G >= a.ng_pad) return;
    uint32_t* out = reinterpret_cast<uint32_t*>(a.values_tc + static_cast<int64_t>(r) * a.ld_tc) + b * G;
    const int ng = min(G, a.ng_pad - b * G);
    if (r >= a.rows_p || b >= a.nb_pad) {
        for (int i = 0; i < ng; ++i) out[i] = 0u;
        return;
    }
    const uint32_t nib = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
    const uint32_t ci = *reinterpret_cast<const uint32_t*>(a.col_idx + (static_cast<int64_t>(r / a.V) * a.nb_pad + b) * 4);
    const uint32_t vv = *reinterpret_cast<const uint32_t*>(a.values + static_cast<int64_t>(r) * a.ld_val + 2 * b);
    const int c0 = (ci >> (8 * (nib & 3u))) & 0xFF, c1 = (ci >> (8 * (nib >> 2))) & 0xFF;  // c0 < c1
    const uint32_t v0 = vv & 0xFFFFu, v1 = vv >> 16;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        if (i >= ng) break;
        const int p0 = c0 - 4 * i, p1 = c1 - 4 * i;
        const bool in0 = p0 >= 0 && p0 < 4, in1 = p1 >= 0 && p1 < 4;
        uint32_t w = 0;  // filler slots carry zeros; a lone value sits in slot a if its position < the filler's
        if (in0 && in1) w = v0 | (v1 << 16);
        else if (in0) w = p0 == 0 ? v0 : (v0 << 16);
        else if (in1) w = p1 == 0 ? v1 : (v1 << 16);
        out[i] = w;
    }
}

// the 8 group nibbles of MMA mi (groups 8mi .. 8mi+7) of row r; 0x44444444 past the rows / MMAs
template <int M>
__device__ uint32_t nat24_word(const Nat24Args& a, int r, int mi) {
    if (r >= a.rows_p || mi >= a.n_mma) return 0x44444444u;
    uint32_t w = 0;
    int bcur = -1, c0 = 0, c1 = 0;
    for (int i = 0; i < 8; ++i) {
        const int q = 8 * mi + i, b = 4 * q / M;
        uint32_t nib = 0x4u;
        if (b < a.nb_pad) {
            if (b != bcur) {  // the block's two kept columns, block-relative (c0 < c1)
                const uint32_t bn = (a.meta[static_cast<int64_t>(r) * a.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
                const uint8_t* ci = a.col_idx + (static_cast<int64_t>(r / a.V) * a.nb_pad + b) * 4;
                c0 = ci[bn & 3u];
                c1 = ci[bn >> 2];
                bcur = b;
            }
            const int base = 4 * q - b * M, p0 = c0 - base, p1 = c1 - base;
            const bool in0 = p0 >= 0 && p0 < 4, in1 = p1 >= 0 && p1 < 4;
            if (in0 && in1) {
                nib = static_cast<uint32_t>(p0) | (static_cast<uint32_t>(p1) << 2);
            } else if (in0 || in1) {
                const int p = in0 ? p0 : p1, f = p == 0 ? 1 : 0;
                nib = static_cast<uint32_t>(p < f ? p : f) | (static_cast<uint32_t>(p < f ? f : p) << 2);
            }
        }
        w |= nib << (4 * i);
    }
    return w;
}

// meta_tc[tile][stage][lane][k] in the M = 128 TMEM layout (as pack_tc_meta_kernel): one CTA per (tile, stage)
// computes the 128 rows x 4 MMA words once into shared memory, then writes the lane words coalesced
template <int M>
__global__ void __launch_bounds__(512) pack_nat24_meta_kernel(const Nat24Args a) {
    __shared__ uint32_t wsm[128][4];
    const int tile = blockIdx.x / a.n_stage, st = blockIdx.x % a.n_stage;
    const int i = threadIdx.x;
    wsm[i / 4][i % 4] = nat24_word<M>(a, tile * 128 + i / 4, st * 4 + i % 4);
    __syncthreads();
    const int L = i / 4, k = i % 4, h = (L / 8) % 2;
    const int ra = (L % 8) + 16 * (L / 16);
    const uint32_t wa = wsm[ra][k], wb = wsm[ra + 8][k];
    a.meta_tc[static_cast<int64_t>(blockIdx.x) * 512 + i] = ((wa >> (16 * h)) & 0xFFFFu) | (((wb >> (16 * h)) & 0xFFFFu) << 16);
}

template <int M>
void launch_nat24(const Nat24Args& a, cudaStream_t stream) {
    const int nbk = (a.ng_pad + M / 4 - 1) / (M / 4);  // blocks covering the padded groups
    pack_nat24_values_kernel<M><<<dim3((nbk + 255) / 256, a.rows_w), 256, 0, stream>>>(a);
    count_launch();
    pack_nat24_meta_kernel<M><<<static_cast<unsigned>(a.rows_w / 128 * a.n_stage), 512, 0, stream>>>(a);
    count_launch();
}

}  // namespace

int launch_pack_nat24(const vnm_packed& P, cudaStream_t stream) {
    const vnm_geom& g = P.g;
    Nat24Args a;
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
    a.ng_pad = (g.cols_p / 4 + 7) / 8 * 8;
    a.n_mma = a.ng_pad / 8;
    a.n_stage = (a.n_mma + 3) / 4;
    a.ld_tc = 16 * a.n_mma;
    switch (g.M) {
        case 12: launch_nat24<12>(a, stream); break;
        case 16: launch_nat24<16>(a, stream); break;
        case 20: launch_nat24<20>(a, stream); break;
        case 24: launch_nat24<24>(a, stream); break;
        case 28: launch_nat24<28>(a, stream); break;
        case 32: launch_nat24<32>(a, stream); break;
        default: return kLaunchUnsupported;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

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
    a.w16 = g.M > 8;
    a.n_mma = a.w16 ? g.nb_pad / 2 : g.nb_pad / (g.M == 4 ? 8 : 4);
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
