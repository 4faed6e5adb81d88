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
//   * 16 consumer warps: warp w owns m16 tile w % 4 and the k-steps = w / 4 (mod 4) of every stage (one warp
//     per tile left every SM sub-partition with a single dependent chain: 2.7 us per stage, measured); the
//     4 partials of a tile are added in warp order through shared memory at the end of a row group; A_n tiles
//     arrive as 128-byte-swizzled TMA boxes so the 8 rows of a fragment hit 8 different bank groups;
//   * persistent CTAs take equal shares of the (row group, stage) list (stream-K); a row group cut between
//     CTAs is finished by the last CTA to arrive, which adds the fp32 partials in stage order
//     (deterministic, no second kernel).
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

constexpr int kCons = 16;                 // consumer warps: m16 tile w % 4, k-steps = w / 4 (mod 4)
constexpr int kThreads = 32 * (kCons + 1);
constexpr int kRows = 64;                 // rows per group (4 m16 tiles)
constexpr int kKS = 16;                   // k-steps (8 blocks each) per stage
constexpr int kStages = 3;
constexpr uint32_t kABytes = kRows * kKS * 16 * 2;  // 64 rows x 256 values bf16 = 32 KB (4 SW128 boxes of 64)
constexpr uint32_t kMBytes = kRows * kKS * 4;       // 64 rows x 16 words = 4 KB
constexpr uint32_t kCBytes = kKS * 8 * 4;           // 128 A_i1 words = 512 B

struct DecArgs {
    const uint8_t* col_idx;
    void* YT;
    int64_t ldy;
    float* ws;          // [n_rg][n_st][64][16] fp32 partials of cut row groups
    uint32_t* tickets;  // [n_rg] arrival counters, zero at launch and left zero
    int32_t T, y_bf16, rows, V, M, nb_pad, n_ks;
    int32_t n_rg, n_st, units, grid;
    int32_t xrows;      // X^T rows staged per stage (multiple of 256 >= 128 M)
    const uint16_t* XT; // dense X^T (ldx == TP): the stage's slice is one contiguous bulk copy
    int32_t x_dense, cols;
    uint32_t x_bytes, stage_bytes;
    int32_t trace;  // VNM_SPMM_TRACE: %globaltimer of CTA 0 per unit (issue, data ready, consumed)
};

__device__ unsigned long long g_dec_t[3][64];
__device__ __forceinline__ unsigned long long dtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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
    // declared 1024-aligned (not re-aligned through an integer): the compiler then keeps plain loads from it
    // as shared-memory loads (LDS) instead of generic ones
    extern __shared__ __align__(1024) uint8_t smem[];
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
    if (a.x_dense) {  // X^T rows past cols are never copied in the dense path: they must read as zero
        for (int s = 0; s < kStages; ++s) {
            uint4* x4 = reinterpret_cast<uint4*>(smem + s * a.stage_bytes + kABytes + kMBytes);
            for (int i = threadIdx.x; i < static_cast<int>(a.x_bytes / 16); i += blockDim.x) x4[i] = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
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
                if (a.trace && blockIdx.x == 0 && q < 64) g_dec_t[0][q] = dtime();
                uint8_t* base = smem + s * a.stage_bytes;
                const int nblk = min(kKS * 8, a.nb_pad - st * kKS * 8);  // A_i1 words of this stage
                const uint32_t xb = a.x_dense ? min(kKS * 8 * a.M, a.cols - st * kKS * 8 * a.M) * TP * 2 : a.x_bytes;
                mbar_arrive_expect_tx(&full[s], kABytes + kMBytes + xb + 4 * nblk);
                for (int b = 0; b < 4; ++b) tma_load_2d(base + b * 8192, &tm_a, st * kKS * 16 + 64 * b, rg * kRows, &full[s]);
                tma_load_2d(base + kABytes, &tm_m, st * kKS, rg * kRows, &full[s]);
                const int ch0 = st * kKS * 8 * a.M;
                if (a.x_dense) {
                    // rows [ch0, ch0 + 128 M) are contiguous: one bulk copy; the tail past cols is zeroed once
                    // by the consumers at start (never overwritten: the copy length stops at cols)
                    const int nr = min(kKS * 8 * a.M, a.cols - ch0);
                    bulk_load(base + kABytes + kMBytes, a.XT + static_cast<int64_t>(ch0) * TP, nr * TP * 2, &full[s]);
                } else {
                    for (int x = 0; x < a.xrows; x += 256)
                        tma_load_2d(base + kABytes + kMBytes + x * TP * 2, &tm_x, 0, ch0 + x, &full[s]);
                }
                const int vb = rg * kRows / a.V;
                bulk_load(base + kABytes + kMBytes + a.x_bytes,
                          a.col_idx + (static_cast<int64_t>(vb) * a.nb_pad + st * kKS * 8) * 4, 4 * nblk, &full[s]);
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int g = lane / 4, c = lane % 4, t = warp % 4, kq = warp / 4;
    float* red = reinterpret_cast<float*>(smem + kStages * a.stage_bytes);  // [kCons][16 rows][16 tokens]
    // two accumulator chains (alternate k-steps), added in a fixed order at the end of a piece
    float acc[NT8][4], ch[2][NT8][4];
#pragma unroll
    for (int n = 0; n < NT8; ++n)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            acc[n][k] = 0.f;
            ch[0][n][k] = 0.f;
            ch[1][n][k] = 0.f;
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
        // this warp's partial of tile t -> shared; the kq = 0 warp of each tile adds the 4 in warp order
        // D fragment: d0,d1 = row g, tokens 8n + 2c, +1; d2,d3 = row g + 8 (within the m16 tile)
#pragma unroll
        for (int n = 0; n < NT8; ++n)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                red[(warp * 16 + g + 8 * (k >> 1)) * 16 + 8 * n + 2 * c + (k & 1)] = ch[0][n][k] + ch[1][n][k];
                ch[0][n][k] = 0.f;
                ch[1][n][k] = 0.f;
            }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kCons));
        if (kq == 0) {
#pragma unroll
            for (int n = 0; n < NT8; ++n)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int rl = g + 8 * (k >> 1), tk = 8 * n + 2 * c + (k & 1);
                    float v = 0.f;
#pragma unroll
                    for (int j = 0; j < 4; ++j) v += red[((t + 4 * j) * 16 + rl) * 16 + tk];
                    if (whole)
                        store_y(rg * kRows + 16 * t + rl, tk, v);
                    else
                        a.ws[((static_cast<int64_t>(rg) * a.n_st + st0) * kRows + 16 * t + rl) * 16 + tk] = v;
                }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kCons));
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
        if (a.trace && blockIdx.x == 0 && q < 64 && threadIdx.x == 0) g_dec_t[1][q] = dtime();
        const uint8_t* base = smem + s * a.stage_bytes;
        const uint32_t* sM = reinterpret_cast<const uint32_t*>(base + kABytes);                         // [64][16]
        const uint16_t* sX = reinterpret_cast<const uint16_t*>(base + kABytes + kMBytes);               // [xrows][TP]
        const uint32_t* sC = reinterpret_cast<const uint32_t*>(base + kABytes + kMBytes + a.x_bytes);  // [128]
        const int nks = min(kKS, a.n_ks - st * kKS);
        // A_n tile: 4 boxes [64 rows][64 values], 128-byte swizzle: 16-byte chunk q of row r sits at q ^ (r % 8)
        const uint8_t* abox = base + (16 * t + g) * 128 + 4 * c;
        const uint32_t* mrow = sM + (16 * t + g) * kKS;
        const int h = 16 * (c & 1);
        auto kstep = [&](int ks, float (&cc)[NT8][4]) {
            // A fragment: words 8 ks + c (+4) of rows g, g + 8 = chunks 2 (ks % 4) (+1) of box ks / 4
            const uint8_t* bp = abox + (ks >> 2) * 8192;
            const int q0 = (2 * (ks & 3)) ^ g, q1 = (2 * (ks & 3) + 1) ^ g;  // (row + 8) % 8 == row % 8
            uint32_t A[4];
            A[0] = *reinterpret_cast<const uint32_t*>(bp + 16 * q0);
            A[1] = *reinterpret_cast<const uint32_t*>(bp + 8 * 128 + 16 * q0);
            A[2] = *reinterpret_cast<const uint32_t*>(bp + 16 * q1);
            A[3] = *reinterpret_cast<const uint32_t*>(bp + 8 * 128 + 16 * q1);
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
#pragma unroll
        for (int i = 0; i < kKS / 4; ++i) {
            const int ks = kq + 4 * i;
            if (ks < nks) kstep(ks, ch[i & 1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (a.trace && blockIdx.x == 0 && q < 64 && threadIdx.x == 0) g_dec_t[2][q] = dtime();
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
    p.stage_bytes = (kABytes + kMBytes + p.x_bytes + kCBytes + 1023) / 1024 * 1024;
    p.smem = static_cast<size_t>(kStages) * p.stage_bytes + static_cast<size_t>(kCons) * 16 * 16 * 4 + 1024;
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
    a.XT = L.XT;
    a.cols = g.cols;
    a.x_dense = L.ldx == p.tp && (reinterpret_cast<uintptr_t>(L.XT) & 15u) == 0 ? 1 : 0;
    CUtensorMap ta, tmm, tx;
    if (!encode_2d(&ta, L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_val) * 2, 64, kRows, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_2d(&tmm, L.P->meta, static_cast<uint64_t>(g.nb_pad / 8), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_meta) * 4, kKS, kRows, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_2d(&tx, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), static_cast<uint64_t>(L.ldx) * 2,
                   p.tp, 256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    // tickets are zero at launch (the caller zero-fills the workspace once, vnm_spmm_workspace_init) and every
    // launch leaves them zero (the last CTA of a row group clears its ticket)
    auto k = L.T <= 8 ? vnm_spmm_dec_kernel<1> : vnm_spmm_dec_kernel<2>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)) != cudaSuccess)
        return kLaunchCudaError;
    a.trace = getenv("VNM_SPMM_TRACE") ? 1 : 0;
    k<<<p.grid, kThreads, p.smem, stream>>>(ta, tmm, tx, a);
    count_launch();
    if (a.trace) {
        unsigned long long h[3][64];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(h, g_dec_t, sizeof(h));
        const int n = static_cast<int>(static_cast<long long>(1) * p.units / p.grid);
        fprintf(stderr, "dec: grid %d units %d (CTA 0: %d) stage %u B\n", p.grid, p.units, n, p.stage_bytes);
        for (int q = 0; q < n && q < 64; ++q)
            fprintf(stderr, "  unit %d: issue %llu ready %llu done %llu ns\n", q, h[0][q] - h[0][0], h[1][q] - h[0][0],
                    h[2][q] - h[0][0]);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
