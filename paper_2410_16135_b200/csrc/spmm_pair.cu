// spmm_pair.cu — the small-T plan of the V:N:M SpMM (decode-sized token counts, T <= 32; V = 64, M <= 8).
// SURVEY §8(a) rows a6-a8; §3 "Acceleration of V:N:M sparsity" P:106-109 and App. A P:548.
//
// Why a separate plan.  With T <= 32 tokens a V-block tile is tiny in N, so the cost per stage is set by
// per-instruction overheads, not by bytes: a sparse MMA costs ~100 cycles whatever N <= 128
// (profiles/r01_probes.md MB2) and every mbarrier hand-off costs ~100 cycles of latency.  This plan
//   * puts TWO V-blocks (128 rows) in every M = 128 sparse MMA: their gathered X^T rows sit side by side in
//     N (V-block h in token columns h*nb_tok ..), the product is block-diagonal and only the diagonal
//     blocks are read back — twice the A_n bytes per MMA of the M = 64 form;
//   * brings everything by TMA: A_n (128 x 64 bf16, SW128), A_i2 (128 rows x 4 words), A_i1 (2 x 32 words)
//     and the DENSE X^T slice of the stage's 32 blocks (32*M channels x tp tokens, one bulk copy when X^T is
//     dense) — the X^T slice is shared by both V-blocks;
//   * lets 4 gather warps (stages dealt round-robin) pick the kept rows out of the slice in shared memory
//     and write the MN-major SW128 B tile plus the [128 lanes][16 B] image of the M = 128 TMEM metadata
//     layout, which the MMA thread moves with tcgen05.cp ahead of its MMAs (same tensor-pipe order);
//   * balances the work stream-K style: the stages of all tiles are split evenly over the persistent CTAs;
//     a tile cut between CTAs is finished by the last CTA to arrive (per-tile counter), which adds the fp32
//     partials in CTA order (deterministic) — no second kernel.
// Warps: 0-3 epilogue, 4-7 gather + metadata image, 8 TMA, 9 MMA.
//
// TMEM: accumulator a (segment parity) = columns 64a .. 64a + 2*nb_tok, row m -> lane m (M = 128);
// metadata slot of B-ring slot b = columns 256 + 4b; MMA k reads column (k & ~1) with id2 = k & 1.
// Metadata (M = 128, measured, csrc/probes.cu MB1): nibble (row m, K-group g) sits at lane
// (m % 8) + 8 (g / 4) + 16 (m / 16), nibble 4 ((m / 8) % 2) + g % 4.
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

constexpr int kV = 64;
constexpr int kRowsPair = 128;
constexpr int kBlocksPerStage = 32;  // 4 MMAs of logical K = 32 (8 blocks each)
constexpr int kMmaPerStage = 4;
constexpr int kKRows = 4 * kBlocksPerStage;  // gathered X^T rows per V-block and stage
constexpr int kGatherWarps = 4, kBRing = 4, kMaxRing = 12;
constexpr int kGather0 = 4, kTmaWarp = 8, kMmaWarp = 9, kThreads = 320;
constexpr int kABytes = kRowsPair * 128;        // A_n: 128 rows x 64 bf16 (SW128)
constexpr int kMBytes = kRowsPair * 16;         // A_i2: 128 rows x 4 words
constexpr int kCBytes = 2 * kBlocksPerStage * 4;  // A_i1: 2 V-blocks x 32 words
constexpr int kBBytes = kKRows * 128;           // B: 128 K-rows x 64 token columns (SW128, MN-major)
constexpr int kEBytes = 128 * 16;               // metadata image
constexpr uint32_t kMetaCol = 256;

__device__ unsigned long long g_pair_t[4][1024];  // VNM_SPMM_TRACE: %globaltimer per CTA (start, role ends)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct PairArgs {
    const uint16_t* XT;
    int64_t ldx;
    void* YT;
    int64_t ldy;
    float* ws;            // split tiles: fp32 partials [maxseg][rows_p][tstride]
    uint32_t* flags;      // [npairs][maxseg] segment-done flags, zero at launch and left zero
    int32_t tstride, maxseg;
    int32_t cols, T, tp, M, y_bf16, x_dense;
    int32_t rows, rows_p, nvb, npairs, n_stage, n_mma;
    int32_t total, grid, stream_k;  // stream_k: stages split evenly over the grid; else whole tiles round-robin
    int32_t ring, xs_bytes, nb_tok;
    int32_t trace;
};

// The segments (tile, k0, k1) of CTA c, in order.
struct SegIter {
    int x, x1, tile, k0, k1;
    __device__ __forceinline__ SegIter(const PairArgs& a, int c) {
        if (a.stream_k) {
            x = static_cast<int>(static_cast<long long>(c) * a.total / a.grid);
            x1 = static_cast<int>(static_cast<long long>(c + 1) * a.total / a.grid);
        } else {
            x = c * a.n_stage;
            x1 = a.total;
        }
    }
    __device__ __forceinline__ bool next(const PairArgs& a) {
        if (x >= x1) return false;
        tile = x / a.n_stage;
        k0 = x % a.n_stage;
        k1 = min(a.n_stage, k0 + (x1 - x));
        x += k1 - k0;
        if (!a.stream_k) x += (a.grid - 1) * a.n_stage;  // next tile of this CTA
        return true;
    }
};
__device__ __forceinline__ int stage_owner(const PairArgs& a, int x) {
    return static_cast<int>((static_cast<long long>(x + 1) * a.grid - 1) / a.total);
}

// the gathered rows of one V-block and stage for one warp (NI rows per lane group): all A_i1 words, then
// all slice reads, then all B writes, so the shared-memory round trips overlap
template <int NI>
__device__ __forceinline__ void gather_rows(uint32_t xs, uint32_t cs, uint32_t bs, int rsub, int cpos, int rows_it,
                                            int xrow, int M, bool lane_ok) {
    uint32_t cw[NI];
#pragma unroll
    for (int it = 0; it < NI; ++it)
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw[it]) : "r"(cs + 4 * ((it * rows_it + rsub) >> 2)));
    uint4 v[NI];
#pragma unroll
    for (int it = 0; it < NI; ++it) {
        const int r = it * rows_it + rsub;
        const int srow = (r >> 2) * M + static_cast<int>((cw[it] >> (8 * (r & 3))) & 0xFFu);
        if (lane_ok)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[it].x), "=r"(v[it].y), "=r"(v[it].z), "=r"(v[it].w)
                         : "r"(xs + srow * xrow));
    }
#pragma unroll
    for (int it = 0; it < NI; ++it) {
        const int r = it * rows_it + rsub;
        if (lane_ok)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                             bs + (r >> 3) * 1024 + (r & 7) * 128 + (((r ^ cpos) & 7) << 4)),
                         "r"(v[it].x), "r"(v[it].y), "r"(v[it].z), "r"(v[it].w)
                         : "memory");
    }
}

// metadata image of one stage for the M = 128 layout: image row L (= TMEM lane) holds, for MMA k, halfword
// (L/8)%2 of A_i2 word k of tile row (L%8) + 16(L/16) in bits 0-15 and of that row + 8 in bits 16-31.
// Rows past rows_p (odd V-block count) and MMAs past n_mma get the valid pad pattern 0x4.
__device__ __forceinline__ void meta_image(uint32_t sm, uint32_t es, int lane, int row0, int rows_p, int mi0,
                                           int n_mma) {
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
        const int L = 32 * j + lane;
        const int ra = (L & 7) + 16 * (L >> 4), h = (L >> 3) & 1;
        uint4 wa, wb;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(wa.x), "=r"(wa.y), "=r"(wa.z), "=r"(wa.w)
                     : "r"(sm + ra * 16));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(wb.x), "=r"(wb.y), "=r"(wb.z), "=r"(wb.w)
                     : "r"(sm + (ra + 8) * 16));
        const uint32_t a4[4] = {wa.x, wa.y, wa.z, wa.w}, b4[4] = {wb.x, wb.y, wb.z, wb.w};
        const bool ok_a = row0 + ra < rows_p, ok_b = row0 + ra + 8 < rows_p;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool mok = mi0 + k < n_mma;
            const uint32_t lo = (ok_a && mok) ? ((a4[k] >> (16 * h)) & 0xFFFFu) : 0x4444u;
            const uint32_t hi = (ok_b && mok) ? ((b4[k] >> (16 * h)) & 0xFFFFu) : 0x4444u;
            w[k] = lo | (hi << 16);
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(es + L * 16), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                     "r"(w[3])
                     : "memory");
    }
}

// 16 consecutive outputs of one Y^T row (fp32 or bf16 RNE), masked at T
__device__ __forceinline__ void store16(const PairArgs& a, int row, int t0, const float (&v)[16]) {
    if (!a.y_bf16) {
        float* y = reinterpret_cast<float*>(a.YT) + static_cast<int64_t>(row) * a.ldy + t0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (t0 + k < a.T) y[k] = v[k];
    } else {
        __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(a.YT) + static_cast<int64_t>(row) * a.ldy + t0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (t0 + k < a.T) y[k] = __float2bfloat16_rn(v[k]);
    }
}

// 10 warps: registers are split over the 4 SM sub-partitions, 3 warps on two of them => <= 168 per thread
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_m,
                         const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_x,
                         const PairArgs a) {
    const int S = a.ring;
    extern __shared__ __align__(1024) uint8_t smem[];  // (not re-aligned through an integer: keeps LDS/STS)
    uint8_t* sA = smem;                       // [S][16384]  SW128
    uint8_t* sB = sA + S * kABytes;           // [B][16384]  SW128
    uint8_t* sE = sB + kBRing * kBBytes;      // [B][2048]   metadata images
    uint8_t* sX = sE + kBRing * kEBytes;      // [S][xs]
    uint8_t* sM = sX + S * a.xs_bytes;        // [S][2048]   A_i2 words [128][4]
    uint8_t* sC = sM + S * kMBytes;           // [S][256]    A_i1 words [2][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(sC + S * kCBytes);
    uint64_t* empty = full + kMaxRing;
    uint64_t* bfull = empty + kMaxRing;
    uint64_t* tmem_full = bfull + kBRing;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (a.trace && threadIdx.x == 0) g_pair_t[0][blockIdx.x] = gtimer();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kBRing; ++b) mbar_init(&bfull[b], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_mbar_init();
    }
    if (a.x_dense) {
        // slice rows past cols are never copied: zero them once (a stale finite value times a zero weight is 0)
        uint4* x4 = reinterpret_cast<uint4*>(sX);
        for (int i = threadIdx.x; i < S * a.xs_bytes / 16; i += blockDim.x) x4[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
    if (warp == kTmaWarp && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_m);
        tma_prefetch_desc(&tmap_c);
        tma_prefetch_desc(&tmap_x);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_wait();    // the previous kernel's outputs (e.g. this layer's inputs) are visible
    grid_dep_launch();  // the next kernel may take SMs as this grid's CTAs exit

    if (warp >= kGather0 && warp < kGather0 + kGatherWarps) {
        // ------------------------------------------------------------ gather + metadata image
        constexpr int G = kGatherWarps;
        static_assert(G <= kBRing, "a gather warp may run at most kBRing stages ahead");
        const int gw = warp - kGather0;
        const int cu = (a.T + 7) / 8;  // 16-byte token chunks per V-block (<= 4)
        const int lg = cu <= 1 ? 0 : (cu <= 2 ? 1 : 2);
        const int chn = lane & ((1 << lg) - 1), rsub = lane >> lg;
        const bool lane_ok = chn < cu;
        const int xrow = 2 * a.tp, M_ = a.M, cb = a.nb_tok / 8;
        const uint32_t sX0 = smem_u32(sX) + 16 * chn, sB0 = smem_u32(sB), sC0 = smem_u32(sC);
        const uint32_t sM0 = smem_u32(sM), sE0 = smem_u32(sE);
        int q = 0;
        SegIter it(a, blockIdx.x);
        while (it.next(a)) {
            const bool two = 2 * it.tile + 1 < a.nvb;
            for (int ks = it.k0 + ((gw - q % G) % G + G) % G; ks < it.k1; ks += G) {
                const int qq = q + ks - it.k0;
                const int s = qq % S, b = qq % kBRing;
                mbar_wait(&full[s], (qq / S) & 1);
                // B slot b is free once the MMAs of stage qq - kBRing completed (one commit per stage, on empty[])
                if (qq >= kBRing) mbar_wait(&empty[(qq - kBRing) % S], ((qq - kBRing) / S) & 1);
                const uint32_t xs = sX0 + s * a.xs_bytes, cs = sC0 + s * kCBytes, bs = sB0 + b * kBBytes;
                for (int h = 0; h < (two ? 2 : 1); ++h) {
                    const uint32_t csh = cs + h * kBlocksPerStage * 4;
                    const int cpos = h * cb + chn;
                    if (lg == 0) {
                        gather_rows<4>(xs, csh, bs, rsub, cpos, 32, xrow, M_, lane_ok);
                    } else if (lg == 1) {
                        gather_rows<8>(xs, csh, bs, rsub, cpos, 16, xrow, M_, lane_ok);
                    } else {
                        gather_rows<8>(xs, csh, bs, rsub, cpos, 8, xrow, M_, lane_ok);
                        gather_rows<8>(xs, csh, bs, rsub + 64, cpos, 8, xrow, M_, lane_ok);
                    }
                }
                meta_image(sM0 + s * kMBytes, sE0 + b * kEBytes, lane, it.tile * kRowsPair, a.rows_p,
                           ks * kMmaPerStage, a.n_mma);
                fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
                __syncwarp();
                if (lane == 0) mbar_arrive(&bfull[b]);
            }
            q += it.k1 - it.k0;
        }
    } else if (warp == kTmaWarp) {
        // ------------------------------------------------------------ TMA: A_n, A_i2, A_i1, X^T slice
        if (lane == 0) {
            const uint32_t tx0 = kABytes + kMBytes + kCBytes;
            const int xrows = kBlocksPerStage * a.M;
            int q = 0;
            SegIter it(a, blockIdx.x);
            while (it.next(a)) {
                for (int ks = it.k0; ks < it.k1; ++ks, ++q) {
                    const int s = q % S;
                    mbar_wait(&empty[s], ((q / S) & 1) ^ 1);
                    const int c0 = ks * xrows;
                    const int nrow = a.x_dense ? max(0, min(xrows, a.cols - c0)) : xrows;
                    const uint32_t xbytes = static_cast<uint32_t>(nrow * 2 * a.tp);
                    mbar_arrive_expect_tx(&full[s], tx0 + xbytes);
                    tma_load_2d(sA + s * kABytes, &tmap_a, ks * (2 * kBlocksPerStage), it.tile * kRowsPair, &full[s]);
                    tma_load_2d(sM + s * kMBytes, &tmap_m, ks * kMmaPerStage, it.tile * kRowsPair, &full[s]);
                    tma_load_2d(sC + s * kCBytes, &tmap_c, ks * kBlocksPerStage, 2 * it.tile, &full[s]);
                    if (!a.x_dense)
                        tma_load_2d(sX + s * a.xs_bytes, &tmap_x, 0, c0, &full[s]);
                    else if (xbytes)
                        bulk_load(sX + s * a.xs_bytes, a.XT + static_cast<int64_t>(c0) * a.ldx, xbytes, &full[s]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer (warp-uniform, elected lane)
        const uint32_t n = 2 * a.nb_tok;
        const uint32_t idesc0 = idesc_bf16(128, n, true, 0, true);
        const uint32_t idesc1 = idesc_bf16(128, n, true, 1, true);
        const uint64_t adesc0 = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
        const uint64_t bdesc0 = sdesc(smem_u32(sB), kKRows * 128, 1024, kLayoutSW128);
        const uint64_t edesc0 = sdesc(smem_u32(sE), 16, 128, 0);
        int q = 0, tl = 0;
        SegIter it(a, blockIdx.x);
        while (it.next(a)) {
            const int acc = tl & 1;
            mbar_wait(&tmem_empty[acc], ((tl >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + 64u * acc;
            for (int ks = it.k0; ks < it.k1; ++ks, ++q) {
                const int s = q % S, b = q % kBRing;
                mbar_wait(&bfull[b], (q / kBRing) & 1);  // B + metadata image (the gather waited on full[s])
                tc_fence_after();
                const uint32_t e_tmem = tmem + kMetaCol + 4 * b;
                if (elect_one()) tmem_cp_128x128b(e_tmem, edesc0 + ((b * kEBytes) >> 4));
                mma_sp_x4(d_tmem, adesc0 + ((s * kABytes) >> 4), bdesc0 + ((b * kBBytes) >> 4), e_tmem, idesc0,
                          idesc1, ks > it.k0 ? 1u : 0u);
                mma_commit_elect(&empty[s]);  // frees ring slot s and B slot b
            }
            mma_commit_elect(&tmem_full[acc]);
            ++tl;
        }
        if (a.trace && lane == 0) g_pair_t[1][blockIdx.x] = gtimer();
    } else if (warp < 4) {
        // ------------------------------------------------------------ epilogue (+ stream-K fix-up)
        // A tile cut between CTAs: every segment but the head (k0 = 0) writes its fp32 partial and raises its
        // flag; the head segment — the LAST one its CTA processes, while the others are the first or the only
        // ones of theirs — waits for the flags and adds the partials, in segment order, to its accumulator.
        const int qd = warp;
        const int h = qd / 2;  // V-block of this warp's 32 rows
        int tl = 0;
        SegIter it(a, blockIdx.x);
        while (it.next(a)) {
            const int acc = tl & 1;
            const int row = it.tile * kRowsPair + 32 * qd + lane;
            const bool whole = it.k0 == 0 && it.k1 == a.n_stage;
            const int x_first = it.tile * a.n_stage;
            const int own0 = a.stream_k ? stage_owner(a, x_first) : 0;
            const int nseg = a.stream_k ? stage_owner(a, x_first + a.n_stage - 1) - own0 + 1 : 1;
            const int j = blockIdx.x - own0;  // segment index within the tile (0 = head)
            uint32_t* flags = a.flags + static_cast<int64_t>(it.tile) * a.maxseg;
            if (!whole && j == 0) {
                // head: the other segments' partials must have landed (they never wait on this CTA)
                if (threadIdx.x == 0)
                    for (int jj = 1; jj < nseg; ++jj) {
                        uint32_t f = 0;
                        for (;;) {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + jj) : "memory");
                            if (f) break;
                            __nanosleep(64);
                        }
                        flags[jj] = 0u;  // consumed: the workspace leaves every launch with its flags zero
                    }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            mbar_wait(&tmem_full[acc], (tl >> 1) & 1);
            tc_fence_after();
            for (int c = 0; c < a.nb_tok; c += 16) {
                uint32_t r[16];
                tmem_ld_32x32b_x16(tmem + ((32u * qd) << 16) + 64u * acc + h * a.nb_tok + c, r);
                tmem_wait_ld();
                float v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
                if (row < a.rows && c < a.T) {
                    if (whole) {
                        store16(a, row, c, v);
                    } else if (j == 0) {
                        for (int jj = 1; jj < nseg; ++jj) {
                            const float4* w = reinterpret_cast<const float4*>(
                                a.ws + ((static_cast<int64_t>(jj) * a.rows_p + row) * a.tstride + c));
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float4 p4 = __ldcg(w + k);
                                v[4 * k] += p4.x;
                                v[4 * k + 1] += p4.y;
                                v[4 * k + 2] += p4.z;
                                v[4 * k + 3] += p4.w;
                            }
                        }
                        store16(a, row, c, v);
                    } else {
                        float4* w = reinterpret_cast<float4*>(
                            a.ws + ((static_cast<int64_t>(j) * a.rows_p + row) * a.tstride + c));
#pragma unroll
                        for (int k = 0; k < 4; ++k) w[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[acc]);  // the MMAs of the next segment may start
            if (!whole && j > 0) {
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + j), "r"(1u) : "memory");
            }
            ++tl;
        }
    }
    if (a.trace && warp == 0 && lane == 0) g_pair_t[2][blockIdx.x] = gtimer();
    tc_fence_before();
    __syncthreads();
    if (a.trace && threadIdx.x == 0) g_pair_t[3][blockIdx.x] = gtimer();
    if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
}

struct PairPlan {
    int npairs, n_stage, total, grid, maxseg, stream_k, tstride;
    size_t part_bytes, ws_bytes;  // partials [maxseg][rows_p][tstride] fp32, then flags
};

PairPlan make_plan(const vnm_geom& g, int32_t T) {
    PairPlan p{};
    const int nvb = g.rows_p / kV;
    p.npairs = (nvb + 1) / 2;
    p.n_stage = (g.nb_pad / 8 + kMmaPerStage - 1) / kMmaPerStage;
    p.total = p.npairs * p.n_stage;
    const int G = num_sms();
    p.stream_k = p.npairs < 4 * G;  // enough whole tiles: round-robin them instead
    p.grid = p.stream_k ? (p.total < G ? p.total : G) : G;
    p.maxseg = 1;
    if (p.stream_k) {
        for (int t = 0; t < p.npairs; ++t) {
            const long long x0 = static_cast<long long>(t) * p.n_stage, x1 = x0 + p.n_stage - 1;
            const int o0 = static_cast<int>(((x0 + 1) * p.grid - 1) / p.total);
            const int o1 = static_cast<int>(((x1 + 1) * p.grid - 1) / p.total);
            if (o1 - o0 + 1 > p.maxseg) p.maxseg = o1 - o0 + 1;
        }
    }
    p.tstride = (T + 15) / 16 * 16;
    p.part_bytes = static_cast<size_t>(p.maxseg) * g.rows_p * p.tstride * 4;
    p.ws_bytes = p.stream_k ? p.part_bytes + static_cast<size_t>(p.npairs) * p.maxseg * 4 : 0;
    return p;
}

}  // namespace

bool spmm_pair_applies(const vnm_geom& g, int32_t T) { return g.V == kV && g.M <= 8 && T >= 1 && T <= 32 && g.nb_pad > 0; }

size_t spmm_pair_workspace_bytes(const vnm_geom& g, int32_t T) {
    return spmm_pair_applies(g, T) ? make_plan(g, T).ws_bytes : 0;
}

int launch_spmm_pair(const SpmmLaunch& L, cudaStream_t st) {
    const vnm_geom& g = L.P->g;
    if (!spmm_pair_applies(g, L.T)) return kLaunchUnsupported;
    const PairPlan p = make_plan(g, L.T);
    PairArgs a{};
    a.XT = L.XT;
    a.ldx = L.ldx;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.cols = g.cols;
    a.T = L.T;
    a.tp = (L.T + 7) / 8 * 8;
    a.M = g.M;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.x_dense = L.ldx == a.tp;
    a.rows = g.rows;
    a.rows_p = g.rows_p;
    a.nvb = g.rows_p / kV;
    a.npairs = p.npairs;
    a.n_stage = p.n_stage;
    a.n_mma = g.nb_pad / 8;
    a.total = p.total;
    a.grid = p.grid;
    a.stream_k = p.stream_k;
    a.nb_tok = L.T <= 16 ? 16 : 32;
    a.trace = VNM_ENV_INT("VNM_SPMM_TRACE", 0) ? 1 : 0;
    if (p.stream_k) {
        if (!L.workspace || L.workspace_bytes < p.ws_bytes) {  // no scratch: whole tiles only
            a.stream_k = 0;
            a.grid = p.npairs < num_sms() ? p.npairs : num_sms();
        } else {
            a.ws = static_cast<float*>(L.workspace);
            a.flags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(L.workspace) + p.part_bytes);
            a.maxseg = p.maxseg;
            a.tstride = p.tstride;
            // the flags are zero at launch (include/vnm.h: the caller zero-fills the workspace once,
            // vnm_spmm_workspace_init) and every launch leaves them zero (the head segment clears what it
            // consumed): no per-launch memset node.  VNM_SPMM_MEMSET=1 restores the memset (comparisons).
            static const bool always = [] { const char* e = getenv("VNM_SPMM_MEMSET"); return e && e[0] == '1'; }();
            if (always && cudaMemsetAsync(a.flags, 0, static_cast<size_t>(p.npairs) * p.maxseg * 4, st) != cudaSuccess)
                return kLaunchCudaError;
        }
    }
    a.xs_bytes = (kBlocksPerStage * g.M * 2 * a.tp + 1023) / 1024 * 1024;
    const int slot = kABytes + a.xs_bytes + kMBytes + kCBytes;
    const int fixed = kBRing * (kBBytes + kEBytes) + 1024 + 512;
    a.ring = static_cast<int>((kMaxSmem - fixed) / slot);
    if (a.ring > kMaxRing) a.ring = kMaxRing;
    if (a.ring < kBRing) return kLaunchUnsupported;
    const int smem = fixed + a.ring * slot;

    CUtensorMap ta, tm, tc, tx;
    if (!encode_2d(&ta, L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_val) * 2, 64, kRowsPair) ||
        !encode_2d(&tm, L.P->meta, static_cast<uint64_t>(g.nb_pad / 8), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_meta) * 4, kMmaPerStage, kRowsPair, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_2d(&tc, L.P->col_idx, static_cast<uint64_t>(g.nb_pad), static_cast<uint64_t>(a.nvb),
                   static_cast<uint64_t>(g.nb_pad) * 4, kBlocksPerStage, 2, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                   CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_2d(&tx, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols),
                   static_cast<uint64_t>(L.ldx) * 2, a.tp, kBlocksPerStage * g.M, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   CU_TENSOR_MAP_SWIZZLE_NONE)) {
        if (VNM_ENV_INT("VNM_DEBUG", 0)) fprintf(stderr, "vnm_spmm (pair plan): tensor-map encoding failed\n");
        return kLaunchCudaError;
    }
    cudaError_t e = cudaFuncSetAttribute(vnm_spmm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) {
        e = launch_pdl(true, vnm_spmm_pair_kernel, dim3(a.grid), dim3(kThreads), static_cast<size_t>(smem), st, ta, tm, tc, tx, a);
        count_launch();
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e == cudaSuccess && a.trace) {
        static unsigned long long h[4][1024];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_pair_t, sizeof(h));
        unsigned long long t0 = ~0ull;
        for (int i = 0; i < a.grid; ++i) t0 = h[0][i] < t0 ? h[0][i] : t0;
        fprintf(stderr, "pair plan: grid %d stream_k %d total %d ring %d\n", a.grid, a.stream_k, a.total, a.ring);
        for (int i = 0; i < a.grid; i += 7)
            fprintf(stderr, "  cta %3d start %6llu mma_done %6llu epi_done %6llu end %6llu ns\n", i, h[0][i] - t0,
                    h[1][i] - t0, h[2][i] - t0, h[3][i] - t0);
    }
    if (e != cudaSuccess && VNM_ENV_INT("VNM_DEBUG", 0))
        fprintf(stderr, "vnm_spmm (pair plan): %s (smem %d, grid %d)\n", cudaGetErrorString(e), smem, a.grid);
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
