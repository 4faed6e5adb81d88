// spmm_dec.cu — the V:N:M SpMM for decode-sized token counts (T <= 16), SURVEY §8(a) rows a6-a8 and
// §8(d) config 4b.  PAPER.md §3 "Acceleration of V:N:M sparsity" P:106-109, App. A P:548.
//
// At T <= 16 the product is a stream of the packed weights (A_n 4/M B per weight, A_i2 0.5/M, A_i1) with a
// few MACs each; the kernel is built to keep HBM busy with the least work per byte:
//   * warp-level sparse tensor-core MMA (mma.sp m16n8k32, bf16 -> fp32): A comes straight from global
//     memory into registers in the fragment layout — A_n already IS the 2:4-compressed operand (2 values
//     per block = per group of 4 gathered channels, App. A) — so the weights touch neither shared
//     memory nor a TMA pipeline; the A_i2 words are the MMA metadata (rows g, g+8 of the 16-row tile,
//     one 16-bit half per thread pair, selector 0);
//   * the 4 kept X^T channels of every block (A_i1) are gathered from a shared-memory copy of the CTA's
//     X^T slice into the B fragment, once per 8 blocks and shared by the 4 row tiles of a 64-row group;
//   * CTA = one 64-row group (rows of one V-block) x a K range; 4 warps interleave k-steps and add their
//     partials in shared memory in warp order; K ranges of a row group (splits) meet in an fp32 workspace
//     and the last CTA to finish adds them in split order — deterministic, no second kernel.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kRows = 64;  // rows per CTA (4 m16 tiles)

struct DecArgs {
    const uint16_t* XT;
    int64_t ldx;
    const uint16_t* values;
    const uint8_t* col_idx;
    const uint32_t* meta;
    void* YT;
    int64_t ldy;
    float* ws;          // [splits][rows_p][16] fp32 partials (splits > 1)
    uint32_t* tickets;  // [n_rg] arrival counters (splits > 1), zeroed by the launch
    int32_t T, y_bf16, rows, cols, V, M, nb_pad, ld_val, ld_meta;
    int32_t n_ks, splits, ks_per;  // k-steps (8 blocks each), K splits, k-steps per split
};

__device__ __forceinline__ void mma_sp_16832(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[4], uint32_t e) {
    asm volatile(
        "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
        "{%8, %9, %10, %11}, {%0, %1, %2, %3}, %12, 0x0;"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(e));
}

__device__ __forceinline__ uint32_t ldg_nc(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// NT8 = token tiles of 8 (1: T <= 8, 2: T <= 16)
template <int NT8>
__global__ void __launch_bounds__(kThreads) vnm_spmm_dec_kernel(const DecArgs a) {
    constexpr int TP = 8 * NT8;  // tokens held per X^T channel in shared memory
    extern __shared__ __align__(16) uint8_t smem[];
    const int rg = blockIdx.x / a.splits, sp = blockIdx.x % a.splits;
    const int ks0 = sp * a.ks_per, ks1 = min(a.n_ks, ks0 + a.ks_per);
    const int nks = max(ks1 - ks0, 0);
    const int row0 = rg * kRows, vb = row0 / a.V;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, c = lane % 4;
    const int M = a.M, ch0 = ks0 * 8 * M, nch = nks * 8 * M;

    uint16_t* sX = reinterpret_cast<uint16_t*>(smem);                       // [nch][TP] bf16
    uint32_t* sC = reinterpret_cast<uint32_t*>(smem + static_cast<size_t>(a.ks_per) * 8 * M * TP * 2);  // [nks*8]
    float* sP = reinterpret_cast<float*>(sC + a.ks_per * 8);                 // [kWarps][kRows][TP] partials

    // ---- stage this CTA's X^T slice (zero past cols / T) and its A_i1 words
    {
        const int cpr = TP / 8;  // 16-byte chunks per channel row
        for (int i = threadIdx.x; i < nch * cpr; i += kThreads) {
            const int r = i / cpr, q = i % cpr, ch = ch0 + r, t = 8 * q;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (ch < a.cols && t < a.T) {
                const uint16_t* src = a.XT + static_cast<int64_t>(ch) * a.ldx + t;
                if (t + 8 <= a.T) {
                    v = *reinterpret_cast<const uint4*>(src);
                } else {
                    uint16_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    for (int k = 0; k < a.T - t; ++k) h[k] = src[k];
                    v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
                }
            }
            *reinterpret_cast<uint4*>(sX + r * TP + t) = v;
        }
        const uint32_t* ci = reinterpret_cast<const uint32_t*>(a.col_idx) + static_cast<int64_t>(vb) * a.nb_pad + ks0 * 8;
        for (int i = threadIdx.x; i < nks * 8; i += kThreads) sC[i] = ci[i];
    }
    __syncthreads();

    float acc[4][NT8][4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int n = 0; n < NT8; ++n)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[t][n][k] = 0.f;

    // row pointers of this thread's fragment rows (g, g + 8 of each m16 tile)
    const uint32_t* vrow = reinterpret_cast<const uint32_t*>(a.values) + static_cast<int64_t>(row0 + g) * (a.ld_val / 2) + c;
    const uint32_t* mrow = a.meta + static_cast<int64_t>(row0 + g) * a.ld_meta;
    const int64_t v8 = 8 * static_cast<int64_t>(a.ld_val / 2), m8 = 8 * static_cast<int64_t>(a.ld_meta);

    // A fragment of tile t, k-step s (compressed column j of the step = value j of block 8s + j/2):
    // a0 = row g cols 2c,2c+1; a1 = row g+8 cols 2c,2c+1; a2 = row g cols 2c+8,+9; a3 = row g+8 cols 2c+8,+9
    auto load_a = [&](int s, uint32_t (&A)[4][4], uint32_t (&E)[4]) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t* p = vrow + 16 * t * (a.ld_val / 2) + 8 * s;
            A[t][0] = ldg_nc(p);
            A[t][1] = ldg_nc(p + v8);
            A[t][2] = ldg_nc(p + 4);
            A[t][3] = ldg_nc(p + v8 + 4);
            // metadata (selector 0): thread c = 0 / 1 of each quad carries K-groups 0-3 / 4-7 (halfword c of the
            // A_i2 word) of row g in bits 0-15 and of row g + 8 in bits 16-31 (verified on B200 against the
            // oracle; the same pairing as the tcgen05 M = 128 layout, profiles/r01_probes.md MB1)
            const uint32_t* q = mrow + 16 * t * a.ld_meta + s;
            const uint32_t w0 = ldg_nc(q), w1 = ldg_nc(q + m8);
            const int h = 16 * (c & 1);
            E[t] = ((w0 >> h) & 0xFFFFu) | (((w1 >> h) & 0xFFFFu) << 16);
        }
    };

    // B fragment of k-step s (k = 2c + 8r + {0, 1} -> block c/2 + 2r, A_i1 positions 2(c%2), 2(c%2) + 1),
    // then the 4 x NT8 MMAs of the step
    auto step = [&](int s, const uint32_t (&A)[4][4], const uint32_t (&E)[4]) {
        const int ls = s - ks0;
        uint32_t B[NT8][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int blk = c / 2 + 2 * r;
            const uint32_t cw = sC[ls * 8 + blk] >> (16 * (c & 1));
            const int base = (ls * 8 + blk) * M;
            const uint16_t* x0 = sX + (base + (cw & 0xFF)) * TP + g;
            const uint16_t* x1 = sX + (base + ((cw >> 8) & 0xFF)) * TP + g;
#pragma unroll
            for (int n = 0; n < NT8; ++n) B[n][r] = static_cast<uint32_t>(x0[8 * n]) | (static_cast<uint32_t>(x1[8 * n]) << 16);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int n = 0; n < NT8; ++n) mma_sp_16832(acc[t][n], A[t], B[n], E[t]);
    };

    // warp w takes k-steps ks0 + w, + 4, ...; A of the next step is in flight while this one computes
    uint32_t A0[4][4], E0[4], A1[4][4], E1[4];
    int s = ks0 + warp;
    if (s < ks1) load_a(s, A0, E0);
    for (; s < ks1; s += 2 * kWarps) {
        if (s + kWarps < ks1) load_a(s + kWarps, A1, E1);
        step(s, A0, E0);
        if (s + kWarps >= ks1) break;
        if (s + 2 * kWarps < ks1) load_a(s + 2 * kWarps, A0, E0);
        step(s + kWarps, A1, E1);
    }

    // ---- warp partials -> shared, added in warp order
    // D fragment: d0,d1 = row g, tokens 2c, 2c+1; d2,d3 = row g+8
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int n = 0; n < NT8; ++n) {
            float* p = sP + (warp * kRows + 16 * t + g) * TP + 8 * n + 2 * c;
            p[0] = acc[t][n][0];
            p[1] = acc[t][n][1];
            p[8 * TP] = acc[t][n][2];
            p[8 * TP + 1] = acc[t][n][3];
        }
    __syncthreads();
    for (int i = threadIdx.x; i < kRows * TP; i += kThreads) {
        float v = sP[i];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += sP[w * kRows * TP + i];
        sP[i] = v;
    }
    __syncthreads();

    auto store_y = [&](int i, float v) {
        const int r = row0 + i / TP, t = i % TP;
        if (r >= a.rows || t >= a.T) return;
        if (a.y_bf16)
            reinterpret_cast<__nv_bfloat16*>(a.YT)[static_cast<int64_t>(r) * a.ldy + t] = __float2bfloat16_rn(v);
        else
            reinterpret_cast<float*>(a.YT)[static_cast<int64_t>(r) * a.ldy + t] = v;
    };
    if (a.splits == 1) {
        for (int i = threadIdx.x; i < kRows * TP; i += kThreads) store_y(i, sP[i]);
        return;
    }
    // ---- split-K: publish this split's partial; the last CTA of the row group adds all splits in order
    float* wsp = a.ws + (static_cast<int64_t>(sp) * a.rows + row0) * 16;
    for (int i = threadIdx.x; i < kRows * TP; i += kThreads)
        if (row0 + i / TP < a.rows) wsp[(i / TP) * 16 + i % TP] = sP[i];
    __threadfence();
    __syncthreads();
    __shared__ uint32_t last;
    if (threadIdx.x == 0) last = atomicAdd(&a.tickets[rg], 1u) == static_cast<uint32_t>(a.splits - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = threadIdx.x; i < kRows * TP; i += kThreads) {
        if (row0 + i / TP >= a.rows) continue;
        float v = 0.f;
        for (int q = 0; q < a.splits; ++q)
            v += __ldcg(a.ws + (static_cast<int64_t>(q) * a.rows + row0 + i / TP) * 16 + i % TP);
        store_y(i, v);
    }
    if (threadIdx.x == 0) a.tickets[rg] = 0;  // ready for the next call (same stream order)
}

struct DecPlan {
    int n_rg, n_ks, splits, ks_per;
    size_t smem;
};

DecPlan make_plan(const vnm_geom& g, int T) {
    DecPlan p;
    p.n_rg = g.rows_p / kRows;
    p.n_ks = g.nb_pad / 8;
    const int tp = T <= 8 ? 8 : 16;
    // enough CTAs for ~4 per SM, while one CTA's X^T slice stays <= 40 KB
    int splits = (4 * num_sms() + p.n_rg - 1) / p.n_rg;
    const int per_ks = 8 * g.M * tp * 2;
    const int min_splits = (p.n_ks * per_ks + 40 * 1024 - 1) / (40 * 1024);
    if (splits < min_splits) splits = min_splits;
    if (splits > p.n_ks) splits = p.n_ks;
    if (splits < 1) splits = 1;
    p.ks_per = (p.n_ks + splits - 1) / splits;
    p.splits = (p.n_ks + p.ks_per - 1) / p.ks_per;
    p.smem = static_cast<size_t>(p.ks_per) * per_ks + static_cast<size_t>(p.ks_per) * 8 * 4 +
             static_cast<size_t>(kWarps) * kRows * tp * 4;
    return p;
}

}  // namespace

bool spmm_dec_applies(const vnm_geom& g, int32_t T) {
    return T >= 1 && T <= 16 && g.V >= 64 && g.nb_pad > 0 && g.rows_p % kRows == 0;
}

size_t spmm_dec_workspace_bytes(const vnm_geom& g, int32_t T) {
    if (!spmm_dec_applies(g, T)) return 0;
    const DecPlan p = make_plan(g, T);
    if (p.splits == 1) return 0;
    const size_t ws = static_cast<size_t>(p.splits) * g.rows * 16 * 4;
    return (ws + 255) / 256 * 256 + static_cast<size_t>(p.n_rg) * 4;
}

int launch_spmm_dec(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (!spmm_dec_applies(g, L.T)) return kLaunchUnsupported;
    const DecPlan p = make_plan(g, L.T);
    DecArgs a;
    a.XT = L.XT;
    a.ldx = L.ldx;
    a.values = L.P->values;
    a.col_idx = L.P->col_idx;
    a.meta = L.P->meta;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.T = L.T;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.cols = g.cols;
    a.V = g.V;
    a.M = g.M;
    a.nb_pad = g.nb_pad;
    a.ld_val = g.ld_val;
    a.ld_meta = g.ld_meta;
    a.n_ks = p.n_ks;
    a.splits = p.splits;
    a.ks_per = p.ks_per;
    a.ws = nullptr;
    a.tickets = nullptr;
    if (p.splits > 1) {
        const size_t need = spmm_dec_workspace_bytes(g, L.T);
        if (!L.workspace || L.workspace_bytes < need) return kLaunchUnsupported;
        a.ws = static_cast<float*>(L.workspace);
        a.tickets = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(L.workspace) + (need - static_cast<size_t>(p.n_rg) * 4));
        cudaMemsetAsync(a.tickets, 0, static_cast<size_t>(p.n_rg) * 4, stream);
    }
    auto k = L.T <= 8 ? vnm_spmm_dec_kernel<1> : vnm_spmm_dec_kernel<2>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)) != cudaSuccess)
        return kLaunchCudaError;
    k<<<p.n_rg * p.splits, kThreads, p.smem, stream>>>(a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
