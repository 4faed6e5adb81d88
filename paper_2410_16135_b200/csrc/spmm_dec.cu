// spmm_dec.cu — the V:N:M SpMM for decode-sized token counts (T <= 16), SURVEY §8(a) rows a6-a8 and
// §8(d) config 4b.  PAPER.md §3 "Acceleration of V:N:M sparsity" P:106-109, App. A P:548.
//
// At T <= 16 the product is a stream of the packed weights (A_n 4/M B per weight, A_i2 0.5/M, A_i1) with a
// few MACs each, so the kernel is a TMA stream with light tensor-core work on top:
//   * unit of work = one 64-row group (4 m16 tiles, rows of one V-block) x one stage of 16 k-steps
//     (128 blocks): the A_n tile [64 x 256 values], its A_i2 tile [64 x 16 words], the X^T channels of those
//     128 blocks [128 M x TP tokens] and the 128 A_i1 words arrive by TMA / bulk copy into a 3-deep ring
//     (one producer warp);
//   * warp-level sparse MMA (mma.sp::ordered_metadata m16n8k32, bf16 -> fp32): A_n already IS the
//     2:4-compressed operand (2 values per block = per group of 4 gathered channels, App. A) and the
//     A_i2 word of a row is its metadata (thread 4g + c, c < 2: half c of rows g and g+8); the B fragment
//     gathers the 4 kept channels of each block (A_i1) from the staged X^T slice;
//   * 4 consumer warps, one m16 tile each, so no cross-warp reduction; persistent CTAs take equal shares of
//     the (row group, stage) list (stream-K); a row group cut between CTAs is finished by the last CTA to
//     arrive, which adds the fp32 partials in stage order (deterministic, no second kernel).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kCons = 4;                  // consumer warps (one m16 tile each)
constexpr int kThreads = 32 * (kCons + 1);
constexpr int kRows = 64;                 // rows per group (4 m16 tiles)
constexpr int kKS = 16;                   // k-steps (8 blocks each) per stage
constexpr int kStages = 3;
constexpr uint32_t kABytes = kRows * kKS * 16 * 2;  // 64 rows x 256 values bf16 = 32 KB
constexpr uint32_t kMBytes = kRows * kKS * 4;       // 64 rows x 16 words = 4 KB
constexpr uint32_t kCBytes = kKS * 8 * 4;           // 128 A_i1 words = 512 B

struct DecArgs {
    const uint8_t* col_idx;
    void* YT;
    int64_t ldy;
    float* ws;          // [n_rg][n_st][64][16] fp32 partials of cut row groups
    uint32_t* tickets;  // [n_rg] arrival counters, zeroed by the launch
    int32_t T, y_bf16, rows, V, M, nb_pad, n_ks;
    int32_t n_rg, n_st, units, grid;
    int32_t xrows;      // X^T rows staged per stage (multiple of 256 >= 128 M)
    uint32_t x_bytes, stage_bytes;
};

__device__ __forceinline__ void mma_sp_16832(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[4], uint32_t e) {
    asm volatile(
        "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
        "{%8, %9, %10, %11}, {%0, %1, %2, %3}, %12, 0x0;"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(e));
}

__device__ __forceinline__ int unit_owner(const DecArgs& a, int u) {  // CTA whose share contains unit u
    return static_cast<int>((static_cast<long long>(u + 1) * a.grid - 1) / a.units);
}

template <int NT8>
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_dec_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_m,
                        const __grid_constant__ CUtensorMap tm_x, const DecArgs a) {
    constexpr int TP = 8 * NT8;  // tokens held per X^T channel in shared memory
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ uint32_t last_flag;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int u0 = static_cast<int>(static_cast<long long>(blockIdx.x) * a.units / a.grid);
    const int u1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * a.units / a.grid);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCons);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCons) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_a);
            tma_prefetch_desc(&tm_m);
            tma_prefetch_desc(&tm_x);
            for (int u = u0, q = 0; u < u1; ++u, ++q) {
                const int rg = u / a.n_st, st = u % a.n_st, s = q % kStages;
                mbar_wait(&empty[s], ((q / kStages) & 1) ^ 1);
                uint8_t* base = smem + s * a.stage_bytes;
                const int nblk = min(kKS * 8, a.nb_pad - st * kKS * 8);  // A_i1 words of this stage
                mbar_arrive_expect_tx(&full[s], kABytes + kMBytes + a.x_bytes + 4 * nblk);
                tma_load_2d(base, &tm_a, st * kKS * 16, rg * kRows, &full[s]);
                tma_load_2d(base + kABytes, &tm_m, st * kKS, rg * kRows, &full[s]);
                for (int x = 0; x < a.xrows; x += 256)
                    tma_load_2d(base + kABytes + kMBytes + x * TP * 2, &tm_x, 0, st * kKS * 8 * a.M + x, &full[s]);
                const int vb = rg * kRows / a.V;
                bulk_load(base + kABytes + kMBytes + a.x_bytes,
                          a.col_idx + (static_cast<int64_t>(vb) * a.nb_pad + st * kKS * 8) * 4, 4 * nblk, &full[s]);
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers: warp w = m16 tile w
    const int g = lane / 4, c = lane % 4, t = warp;
    // kCh independent accumulator chains (k-step ks feeds chain ks % kCh) so consecutive MMAs do not wait on
    // each other; the chains are added in a fixed order at the end of a piece
    constexpr int kCh = 4;
    float acc[NT8][4], ch[kCh][NT8][4];
#pragma unroll
    for (int n = 0; n < NT8; ++n)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            acc[n][k] = 0.f;
#pragma unroll
            for (int j = 0; j < kCh; ++j) ch[j][n][k] = 0.f;
        }

    auto store_y = [&](int r, int tk, float v) {
        if (r < a.rows && tk < a.T) {
            if (a.y_bf16)
                reinterpret_cast<__nv_bfloat16*>(a.YT)[static_cast<int64_t>(r) * a.ldy + tk] = __float2bfloat16_rn(v);
            else
                reinterpret_cast<float*>(a.YT)[static_cast<int64_t>(r) * a.ldy + tk] = v;
        }
    };
    auto flush = [&](int rg, int st0, bool whole) {
        // D fragment: d0,d1 = row 16t + g, tokens 8n + 2c, +1; d2,d3 = row 16t + g + 8
#pragma unroll
        for (int n = 0; n < NT8; ++n)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[n][k] = (ch[0][n][k] + ch[1][n][k]) + (ch[2][n][k] + ch[3][n][k]);
#pragma unroll
                for (int j = 0; j < kCh; ++j) ch[j][n][k] = 0.f;
                const int rl = 16 * t + g + 8 * (k >> 1), tk = 8 * n + 2 * c + (k & 1);
                if (whole)
                    store_y(rg * kRows + rl, tk, acc[n][k]);
                else
                    a.ws[((static_cast<int64_t>(rg) * a.n_st + st0) * kRows + rl) * 16 + tk] = acc[n][k];
                acc[n][k] = 0.f;
            }
    };
    // a cut row group: publish, and the last CTA to arrive adds the pieces in stage order
    auto finish_cut = [&](int rg) {
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kCons));
        const int first = unit_owner(a, rg * a.n_st), last = unit_owner(a, rg * a.n_st + a.n_st - 1);
        if (threadIdx.x == 0) last_flag = atomicAdd(&a.tickets[rg], 1u) == static_cast<uint32_t>(last - first);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kCons));
        if (!last_flag) return;
        __threadfence();
        for (int i = threadIdx.x; i < kRows * TP; i += 32 * kCons) {
            const int r = i / TP, tk = i % TP;
            float v = 0.f;
            for (int cta = first; cta <= last; ++cta) {
                const int ub = static_cast<int>(static_cast<long long>(cta) * a.units / a.grid);
                const int st0 = max(ub, rg * a.n_st) - rg * a.n_st;
                v += __ldcg(a.ws + ((static_cast<int64_t>(rg) * a.n_st + st0) * kRows + r) * 16 + tk);
            }
            store_y(rg * kRows + r, tk, v);
        }
        if (threadIdx.x == 0) a.tickets[rg] = 0;  // ready for the next call (stream order)
    };

    int piece_st0 = u0 < u1 ? u0 % a.n_st : 0;
    for (int u = u0, q = 0; u < u1; ++u, ++q) {
        const int rg = u / a.n_st, st = u % a.n_st, s = q % kStages;
        mbar_wait(&full[s], (q / kStages) & 1);
        const uint8_t* base = smem + s * a.stage_bytes;
        const uint32_t* sA = reinterpret_cast<const uint32_t*>(base);                                   // [64][128]
        const uint32_t* sM = reinterpret_cast<const uint32_t*>(base + kABytes);                         // [64][16]
        const uint16_t* sX = reinterpret_cast<const uint16_t*>(base + kABytes + kMBytes);               // [xrows][TP]
        const uint32_t* sC = reinterpret_cast<const uint32_t*>(base + kABytes + kMBytes + a.x_bytes);  // [128]
        const int nks = min(kKS, a.n_ks - st * kKS);
        const uint32_t* arow = sA + (16 * t + g) * (kKS * 8) + c;
        const uint32_t* mrow = sM + (16 * t + g) * kKS;
        const int h = 16 * (c & 1);
        auto kstep = [&](int ks, float (&cc)[NT8][4]) {
            // A fragment (compressed column j of the step = value j of block 8 ks + j/2 of the stage)
            uint32_t A[4];
            A[0] = arow[8 * ks];
            A[1] = arow[8 * ks + 8 * kKS * 8];
            A[2] = arow[8 * ks + 4];
            A[3] = arow[8 * ks + 8 * kKS * 8 + 4];
            const uint32_t w0 = mrow[ks], w1 = mrow[ks + 8 * kKS];
            const uint32_t E = ((w0 >> h) & 0xFFFFu) | (((w1 >> h) & 0xFFFFu) << 16);
            // B fragment: k = 2c + 8r + {0,1} -> block c/2 + 2r of the step, A_i1 positions 2(c%2), 2(c%2)+1
            uint32_t B[NT8][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int blk = ks * 8 + c / 2 + 2 * r;
                const uint32_t cw = sC[blk] >> h;
                const uint16_t* x0 = sX + (blk * a.M + (cw & 0xFF)) * TP + g;
                const uint16_t* x1 = sX + (blk * a.M + ((cw >> 8) & 0xFF)) * TP + g;
#pragma unroll
                for (int n = 0; n < NT8; ++n) B[n][r] = static_cast<uint32_t>(x0[8 * n]) | (static_cast<uint32_t>(x1[8 * n]) << 16);
            }
#pragma unroll
            for (int n = 0; n < NT8; ++n) mma_sp_16832(cc[n], A, B[n], E);
        };
        if (nks == kKS) {
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) kstep(ks, ch[ks % kCh]);
        } else {
            for (int ks = 0; ks < nks; ks += kCh) {
#pragma unroll
                for (int j = 0; j < kCh; ++j)
                    if (ks + j < nks) kstep(ks + j, ch[j]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // end of a piece: the row group changes or the share ends
        if (st == a.n_st - 1 || u + 1 == u1) {
            const bool whole = piece_st0 == 0 && st == a.n_st - 1;
            flush(rg, piece_st0, whole);
            if (!whole) finish_cut(rg);
            piece_st0 = 0;
        }
    }
}

struct DecPlan {
    int n_rg, n_ks, n_st, units, grid, tp, xrows;
    uint32_t x_bytes, stage_bytes;
    size_t smem;
};

DecPlan make_plan(const vnm_geom& g, int T) {
    DecPlan p;
    p.n_rg = g.rows_p / kRows;
    p.n_ks = g.nb_pad / 8;
    p.n_st = (p.n_ks + kKS - 1) / kKS;
    p.units = p.n_rg * p.n_st;
    p.grid = p.units < num_sms() ? p.units : num_sms();
    p.tp = T <= 8 ? 8 : 16;
    p.xrows = (kKS * 8 * g.M + 255) / 256 * 256;
    p.x_bytes = static_cast<uint32_t>(p.xrows * p.tp * 2);
    p.stage_bytes = (kABytes + kMBytes + p.x_bytes + kCBytes + 127) / 128 * 128;
    p.smem = static_cast<size_t>(kStages) * p.stage_bytes + 128;
    return p;
}

}  // namespace

bool spmm_dec_applies(const vnm_geom& g, int32_t T) {
    return T >= 1 && T <= 16 && g.V >= 64 && g.M <= 8 && g.nb_pad > 0 && g.rows_p % kRows == 0 &&
           make_plan(g, T).smem <= kMaxSmem;
}

size_t spmm_dec_workspace_bytes(const vnm_geom& g, int32_t T) {
    if (!spmm_dec_applies(g, T)) return 0;
    const DecPlan p = make_plan(g, T);
    const size_t ws = static_cast<size_t>(p.n_rg) * p.n_st * kRows * 16 * 4;
    return (ws + 255) / 256 * 256 + static_cast<size_t>(p.n_rg) * 4;
}

int launch_spmm_dec(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (!spmm_dec_applies(g, L.T)) return kLaunchUnsupported;
    const DecPlan p = make_plan(g, L.T);
    const size_t need = spmm_dec_workspace_bytes(g, L.T);
    if (!L.workspace || L.workspace_bytes < need) return kLaunchUnsupported;
    DecArgs a;
    a.col_idx = L.P->col_idx;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.ws = static_cast<float*>(L.workspace);
    a.tickets = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(L.workspace) + (need - static_cast<size_t>(p.n_rg) * 4));
    a.T = L.T;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.V = g.V;
    a.M = g.M;
    a.nb_pad = g.nb_pad;
    a.n_ks = p.n_ks;
    a.n_rg = p.n_rg;
    a.n_st = p.n_st;
    a.units = p.units;
    a.grid = p.grid;
    a.xrows = p.xrows;
    a.x_bytes = p.x_bytes;
    a.stage_bytes = p.stage_bytes;
    CUtensorMap ta, tmm, tx;
    if (!encode_2d(&ta, L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_val) * 2, kKS * 16, kRows, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_2d(&tmm, L.P->meta, static_cast<uint64_t>(g.nb_pad / 8), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_meta) * 4, kKS, kRows, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_2d(&tx, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), static_cast<uint64_t>(L.ldx) * 2,
                   p.tp, 256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    cudaMemsetAsync(a.tickets, 0, static_cast<size_t>(p.n_rg) * 4, stream);
    auto k = L.T <= 8 ? vnm_spmm_dec_kernel<1> : vnm_spmm_dec_kernel<2>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)) != cudaSuccess)
        return kLaunchCudaError;
    k<<<p.grid, kThreads, p.smem, stream>>>(ta, tmm, tx, a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
