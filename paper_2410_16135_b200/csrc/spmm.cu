// spmm.cu — the V:N:M SpMM  Y^T = W' X^T  on the 5th-generation sparse tensor cores (SURVEY §8(a)
// rows a6-a8; §3 "Acceleration of V:N:M sparsity" P:106-109 and App. A: "retrieve the
// retained weights and the corresponding tiles of the input matrix B ... align the data layout with
// that of a 2:4-sparse MM").
//
// Work unit (tile) = one V-block (64 rows of W) x NT tokens.  K is walked in stages of 32 column blocks
// (4 sparse MMAs of logical K = 32 = 8 blocks each).  Persistent CTAs (one per SM) walk the tiles in
// token-tile-major order so the CTAs resident at any time share X^T rows in L2.  Warp roles:
//   warps 8-15 gather: the 4 kept X^T rows of each block (A_i1) -> the stage's B tile, written straight
//              into the MN-major 128B-swizzled UMMA layout by 16-byte cp.async (zero fill past T tokens and
//              past the logical channels: the implicit padding of P:107-108); each thread's copies arrive
//              on the stage barrier asynchronously (cp.async.mbarrier.arrive.noinc).  TMA tile::gather4 was
//              measured at only 7-15 B/clk/SM (csrc/probes2.cu MB3b) and is not used;
//   warp 16    TMA: the stage's A_n tile (64 x 64 bf16, 128B swizzle, K-major);
//   warps 4-7  metadata: A_i2 words (staged in smem by the gather threads) -> TMEM in the M=64
//              sparse-metadata layout (tcgen05.st);
//   warp 17    one thread issues tcgen05.mma.sp.cta_group::1.kind::f16 M=64 N=NT into TMEM;
//   warps 0-3  epilogue: tcgen05.ld -> fp32 / bf16 -> Y^T.
// Two accumulators share TMEM columns: accumulator a (a = tile parity) and its metadata live in lanes
// 16a..16a+15 of every 32-lane sub-partition, so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// TMEM layouts (measured on B200 by csrc/probes*.cu):
//   D (M=64):  row m -> lane 16a + (m % 16) + 32 * (m / 16), column n.
//   E (M=64):  nibble (row m, K-group g) = nibble 4*((m/8)%2) + g%4 of the word at lane
//              16a + (m % 8) + 8*(g/4) + 32*(m/16), column e_col + id2 (e_col even).
//   D and E must carry the same lane offset (0 or 16).
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
constexpr int kBlocksPerStage = 32;
constexpr int kMmaPerStage = kBlocksPerStage / 8;
constexpr int kKRowsPerStage = 4 * kBlocksPerStage;  // 128 gathered X^T rows per stage
constexpr int kMaxGatherWarps = 8;
constexpr int kEpiWarp0 = 0, kMetaWarp0 = 4, kGatherWarp0 = 8, kProdWarp = 16, kMmaWarp = 17;
constexpr int kThreads = 32 * 18;
constexpr uint32_t kMetaCol = 256;
constexpr uint32_t kABytes = kV * 128;

struct SpmmArgs {
    const uint16_t* XT;
    int64_t ldx;
    int32_t cols;
    const uint8_t* col_idx;
    const uint32_t* meta;
    void* YT;
    int64_t ldy;
    int32_t T;
    int32_t y_bf16;
    int32_t rows, M, nb_pad, ld_meta, nvb, ntt, ntiles;
    int32_t vdiv;  // V / 64: 64-row tiles per V-block (they share the block's A_i1 row)
    // split-K (small T): unit u = (tile u / ks_n, K-slice u % ks_n of sps stages); partial sums go to
    // ws[k][row][t] (fp32) and a second kernel adds the ks_n slices in order (deterministic)
    int32_t ks_n, sps, nunits;
    float* ws;
    int32_t trace;  // VNM_SPMM_TRACE: record per-stage clock64 stamps of CTA 0 (g_trace)
};

// debug trace (VNM_SPMM_TRACE=1): clock64 stamps of CTA 0 per pipeline stage q:
// [0] A TMA issued, [2] MMA saw full + meta_ready, [3] gather issued, [4] MMA committed
__device__ unsigned long long g_trace[7][512];


template <int NT>
struct Cfg {
    static constexpr int kBBytes = kKRowsPerStage * NT * 2;
    static constexpr int kMetaBytes = kV * kMmaPerStage * 4;  // A_i2 words of the stage: [64 rows][4]
    static constexpr int kStageBytes = kABytes + kBBytes + kMetaBytes;
    static constexpr int kStages = NT == 256 ? 3 : (NT == 128 ? 5 : 8);
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 512;
    static constexpr int kGatherWarps = kStages < kMaxGatherWarps ? kStages : kMaxGatherWarps;
};

// arrive on `bar` once every cp.async this thread issued so far has landed (count pre-set in mbar_init)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ------------------------------------------------------------------ roles shared by both SpMM kernels
// metadata -> TMEM: the stage's A_i2 words ([64 rows][4] in shared memory, landed with full[s]) repacked
// into the M = 64 TMEM metadata layout (tcgen05.st).  Lanes of the other accumulator's half get the
// don't-care pattern (no in-flight MMA reads slot s); MMAs past n_mma get the valid pad pattern 0x4.
// `ready` has R slots: stage q arrives on ready[q % R].  With R < S (slab plan, where `ready` is the
// gathered-B barrier) the arrival waits until the MMAs of stage q - R completed (empty[(q - R) % S]), so
// no warp contributes to a phase of ready[] ahead of its consumer.
__device__ __forceinline__ void meta_role(const SpmmArgs& a, uint32_t tmem, const uint32_t* sMeta, uint64_t* full,
                                          uint64_t* empty, uint64_t* ready, int S, int R, int qd, int lane) {
    const int n_mma = a.nb_pad / 8;
    const int n_stage = (n_mma + kMmaPerStage - 1) / kMmaPerStage;
    const int ml = lane % 16, mh = ml / 8;
    const int ra = 16 * qd + (ml % 8), rb = ra + 8;  // rows of the V-block this lane combines
    int q = 0, tl = 0;
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
        const int k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
        const bool mine = (lane / 16) == (tl & 1);  // lanes 16*acc .. +15 carry this tile's metadata
        for (int ks = k0; ks < k1; ++ks, ++q) {
            const int s = q % S;
            // full[s] also implies the MMAs that read this TMEM slot in the previous round have completed
            mbar_wait(&full[s], (q / S) & 1);
            if (a.trace && blockIdx.x == 0 && qd == 0 && lane == 0 && q < 512) g_trace[5][q] = clock64();
            const uint4 wa4 = *reinterpret_cast<const uint4*>(sMeta + (s * kV + ra) * kMmaPerStage);
            const uint4 wb4 = *reinterpret_cast<const uint4*>(sMeta + (s * kV + rb) * kMmaPerStage);
            const uint32_t wa[4] = {wa4.x, wa4.y, wa4.z, wa4.w}, wb[4] = {wb4.x, wb4.y, wb4.z, wb4.w};
            uint32_t w[kMmaPerStage];
#pragma unroll
            for (int k = 0; k < kMmaPerStage; ++k)
                w[k] = (mine && ks * kMmaPerStage + k < n_mma)
                           ? (((wa[k] >> (16 * mh)) & 0xFFFFu) | (((wb[k] >> (16 * mh)) & 0xFFFFu) << 16))
                           : 0x44444444u;
            tmem_st_32x32b_x4(tmem + ((32 * qd) << 16) + kMetaCol + 4 * s, w[0], w[1], w[2], w[3]);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (R < S && q >= R) mbar_wait(&empty[(q - R) % S], ((q - R) / S) & 1);
            if (lane == 0) mbar_arrive(&ready[q % R]);
            if (a.trace && blockIdx.x == 0 && qd == 0 && lane == 0 && q < 512) g_trace[6][q] = clock64();
        }
    }
}

// epilogue: tcgen05.ld of accumulator (tile parity) -> fp32 partial of the K-slice (split-K) or Y^T (fp32/bf16)
template <int NT>
__device__ __forceinline__ void epilogue_role(const SpmmArgs& a, uint32_t tmem, uint64_t* tmem_full,
                                              uint64_t* tmem_empty, int qd, int lane) {
    int tl = 0;
    for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
        const int tile = u / a.ks_n, kspl = u % a.ks_n;
        const int vb = tile % a.nvb, n0 = (tile / a.nvb) * NT;
        const int acc = tl & 1;
        const uint32_t aph = (tl >> 1) & 1;
        mbar_wait(&tmem_full[acc], aph);
        tc_fence_after();
        const bool mine = (lane / 16) == acc;
        const int row = vb * kV + 16 * qd + (lane % 16);
        const bool row_ok = mine && row < a.rows;
#pragma unroll 1
        for (int c = 0; c < NT; c += 16) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(tmem + ((32 * qd) << 16) + c, v);
            tmem_wait_ld();
            const int tcol = n0 + c;
            if (row_ok && tcol < a.T) {
                if (a.ks_n > 1) {  // fp32 partial of K-slice kspl
                    float* y = a.ws + (static_cast<int64_t>(kspl) * a.rows + row) * a.T + tcol;
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (tcol + k < a.T) y[k] = __uint_as_float(v[k]);
                } else if (!a.y_bf16) {
                    float* y = reinterpret_cast<float*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                    if (tcol + 16 <= a.T) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            reinterpret_cast<uint4*>(y)[k] =
                                make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            if (tcol + k < a.T) y[k] = __uint_as_float(v[k]);
                    }
                } else {
                    uint16_t* y = reinterpret_cast<uint16_t*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                    uint32_t pk[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        __nv_bfloat162 h =
                            __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                        pk[k] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    if (tcol + 16 <= a.T) {
                        reinterpret_cast<uint4*>(y)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        reinterpret_cast<uint4*>(y)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            if (tcol + k < a.T) y[k] = static_cast<uint16_t>((pk[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);
                    }
                }
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_m,
                    const SpmmArgs a) {
    using C = Cfg<NT>;
    constexpr int S = C::kStages;
    extern __shared__ __align__(1024) uint8_t smem[];  // (not re-aligned through an integer: keeps LDS/STS)
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kABytes;
    uint32_t* sMeta = reinterpret_cast<uint32_t*>(sB + S * C::kBBytes);  // [S][64][4]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* meta_ready = empty + S;
    uint64_t* tmem_full = meta_ready + S;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_mma = a.nb_pad / 8;
    const int n_stage = (n_mma + kMmaPerStage - 1) / kMmaPerStage;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 32 + 1);  // one gather warp + the TMA thread
            mbar_init(&empty[s], 1);
            mbar_init(&meta_ready[s], 4);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
    if (warp == kProdWarp && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_m);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kGatherWarp0 && warp < kGatherWarp0 + C::kGatherWarps) {
        // ------------------------------------------------------------ gather producers (B = kept X^T rows)
        // Stages are dealt round-robin to the G = min(8, S) gather warps (G <= S keeps every wait on empty[s]
        // within one phase).  A warp fills all 128 gathered rows of its stage: lanes form groups of gsz
        // (a power of two >= the 16-byte chunks per row that hold tokens < T), one row per group and
        // instruction, so a decode stage (T <= 16) is 8 instructions and a 256-token stage 128 coalesced ones.
        constexpr int G = C::kGatherWarps;
        const int gw = warp - kGatherWarp0;
        int q = 0;  // stage sequence number shared with the TMA and MMA roles
        for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
            const int tile = u / a.ks_n, k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
            const int vb = tile % a.nvb, n0 = (tile / a.nvb) * NT;
            const uint32_t* ci_vb = reinterpret_cast<const uint32_t*>(a.col_idx) + static_cast<int64_t>(vb / a.vdiv) * a.nb_pad;
            const int tt_tok = min(a.T - n0, NT);
            const int cu = (tt_tok + 7) / 8;                    // 16-byte chunks per row holding tokens < T
            const int lg = cu <= 1 ? 0 : 32 - __clz(cu - 1);  // log2(gsz)
            const int chn = lane & ((1 << lg) - 1), rsub = lane >> lg;
            const int rows_it = 32 >> lg;  // rows per instruction
            const int n_it = kKRowsPerStage / rows_it;
            const bool lane_ok = chn < cu;
            int tokb = (tt_tok - 8 * chn) * 2;
            tokb = tokb > 16 ? 16 : (tokb < 0 ? 0 : tokb);
            const uint16_t* xt_lane = a.XT + n0 + 8 * chn;
            const uint32_t dst_lane = (chn >> 3) * (kKRowsPerStage * 128);
            const int M_ = a.M, cols_ = a.cols;
            const int64_t ldx_ = a.ldx;
            // first stage of this unit owned by this warp: (q + ks - k0) % G == gw
            int ks = k0 + ((gw - q % G) % G + G) % G;
            auto load_ci = [&](int kk) -> uint32_t {  // lane L: A_i1 word of block L of stage kk
                const int blk = kk * kBlocksPerStage + lane;
                return (kk < k1 && blk < a.nb_pad) ? __ldg(ci_vb + blk) : 0xFFFFFFFFu;
            };
            uint32_t ci = load_ci(ks);
            for (; ks < k1; ks += G) {
                const uint32_t ci_next = load_ci(ks + G);
                const int qq = q + ks - k0;
                const int s = qq % S;
                mbar_wait(&empty[s], ((qq / S) & 1) ^ 1);
                if (a.trace && blockIdx.x == 0 && lane == 0 && qq < 512) g_trace[1][qq] = clock64();
                const uint32_t bst = smem_u32(sB + s * C::kBBytes) + dst_lane;
                const int blk0 = ks * kBlocksPerStage;
#pragma unroll 4
                for (int it = 0; it < n_it; ++it) {
                    const int rl = it * rows_it + rsub;  // gathered row of the stage (0..127)
                    const uint32_t cw = __shfl_sync(0xffffffffu, ci, rl >> 2);
                    const int krow = (blk0 + (rl >> 2)) * M_ + static_cast<int>((cw >> (8 * (rl & 3))) & 0xFFu);
                    const int bytes = (cw == 0xFFFFFFFFu || krow >= cols_) ? 0 : tokb;  // padded channel: zero fill
                    if (lane_ok)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                         bst + (rl >> 3) * 1024 + (rl & 7) * 128 + (((rl ^ chn) & 7) << 4)),
                                     "l"(bytes ? xt_lane + krow * ldx_ : a.XT), "r"(bytes)
                                     : "memory");
                }
                cp_async_arrive_noinc(&full[s]);
                if (a.trace && blockIdx.x == 0 && lane == 0 && qq < 512) g_trace[3][qq] = clock64();
                ci = ci_next;
            }
            q += k1 - k0;
        }
    } else if (warp == kProdWarp) {
        // ------------------------------------------------------------ TMA producer (A_n tile + A_i2 words)
        if (lane == 0) {
            int q = 0;
            for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
                const int tile = u / a.ks_n, k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
                const int vb = tile % a.nvb;
                for (int ks = k0; ks < k1; ++ks, ++q) {
                    const int s = q % S;
                    const uint32_t ph = (q / S) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], kABytes + C::kMetaBytes);
                    tma_load_2d(sA + s * kABytes, &tmap_a, ks * (2 * kBlocksPerStage), vb * kV, &full[s]);
                    tma_load_2d(sMeta + s * kV * kMmaPerStage, &tmap_m, ks * kMmaPerStage, vb * kV, &full[s]);
                    if (a.trace && blockIdx.x == 0 && q < 512) g_trace[0][q] = clock64();
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        // The whole warp walks the loop (warp-uniform, no per-instruction re-convergence); one elected lane
        // issues.  Every stage issues its 4 MMAs: MMAs past n_mma see zero A (TMA fill past ld_val), zero B
        // (padded blocks) and the valid pattern 0x4 in every metadata nibble.
        const uint32_t idesc0 = idesc_bf16(64, NT, true, 0, true);
        const uint32_t idesc1 = idesc_bf16(64, NT, true, 1, true);
        const uint64_t adesc0 = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
        const uint64_t bdesc0 = sdesc(smem_u32(sB), kKRowsPerStage * 128, 1024, kLayoutSW128);
        int q = 0, tl = 0;
        for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
            const int k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
            const int acc = tl & 1;
            mbar_wait(&tmem_empty[acc], ((tl >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + ((16u * acc) << 16);
            for (int ks = k0; ks < k1; ++ks, ++q) {
                const int s = q % S;
                const uint32_t ph = (q / S) & 1;
                mbar_wait(&full[s], ph);
                mbar_wait(&meta_ready[s], ph);
                if (a.trace && blockIdx.x == 0 && lane == 0 && q < 512) g_trace[2][q] = clock64();
                tc_fence_after();
                mma_sp_x4(d_tmem, adesc0 + ((s * kABytes) >> 4), bdesc0 + ((s * C::kBBytes) >> 4),
                              d_tmem + kMetaCol + 4 * s, idesc0, idesc1, ks > k0 ? 1u : 0u);
                mma_commit_elect(&empty[s]);
                if (a.trace && blockIdx.x == 0 && lane == 0 && q < 512) g_trace[4][q] = clock64();
            }
            mma_commit_elect(&tmem_full[acc]);
        }
    } else if (warp >= kMetaWarp0 && warp < kMetaWarp0 + 4) {
        meta_role(a, tmem, sMeta, full, empty, meta_ready, S, S, warp - kMetaWarp0, lane);
    } else if (warp < kEpiWarp0 + 4) {
        epilogue_role<NT>(a, tmem, tmem_full, tmem_empty, warp - kEpiWarp0, lane);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
}

// Y^T[row][t] = sum over the ks K-slices, in slice order (deterministic), then fp32 or bf16 (RNE)
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int ks, int rows, int T, void* YT, int64_t ldy,
                                     int y_bf16) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(rows) * T) return;
    const int row = static_cast<int>(idx / T), t = static_cast<int>(idx % T);
    float acc = ws[idx];
    for (int k = 1; k < ks; ++k) acc += ws[static_cast<int64_t>(k) * rows * T + idx];
    if (y_bf16) {
        reinterpret_cast<__nv_bfloat16*>(YT)[static_cast<int64_t>(row) * ldy + t] = __float2bfloat16_rn(acc);
    } else {
        reinterpret_cast<float*>(YT)[static_cast<int64_t>(row) * ldy + t] = acc;
    }
}

// ------------------------------------------------------------------ host side
// Split K when the tiles cannot fill the GPU: minimise (waves of units) x (stages per unit + 1 for the
// per-unit epilogue / pipeline refill), K-slices of at least 2 stages.
int choose_ksplit(int ntiles, int n_stage) {
    const int G = num_sms();
    if (ntiles >= 2 * G) return 1;
    int best = 1;
    long best_cost = static_cast<long>((ntiles + G - 1) / G) * (n_stage + 1);
    for (int ks = 2; ks <= 16 && 2 * ks <= n_stage; ++ks) {
        const int sps = (n_stage + ks - 1) / ks;
        const long cost = static_cast<long>((ntiles * ks + G - 1) / G) * (sps + 1);
        if (cost < best_cost) {
            best_cost = cost;
            best = ks;
        }
    }
    return best;
}

void dump_trace(cudaStream_t st) {
    if (!VNM_ENV_INT("VNM_SPMM_TRACE", 0)) return;
    {
        static unsigned long long h[7][512];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
        const unsigned long long t0 = h[0][0];
        for (int qq = 0; qq < 64; ++qq)
            fprintf(stderr, "trace q=%d tma=%lld meta_start=%lld meta_done=%lld g_w=%lld g_done=%lld ready=%lld commit=%lld\n", qq,
                    (long long)(h[0][qq] - t0), (long long)(h[5][qq] - t0), (long long)(h[6][qq] - t0),
                    (long long)(h[1][qq] - t0), (long long)(h[3][qq] - t0),
                    (long long)(h[2][qq] - t0), (long long)(h[4][qq] - t0));
    }
}

void plan_units(SpmmArgs& a, const SpmmLaunch& L, int NT);
int launch_reduce(const SpmmArgs& a, int T, cudaStream_t st);

template <int NT>
int launch_nt(const SpmmLaunch& L, const CUtensorMap& ta, const CUtensorMap& tm, SpmmArgs a, cudaStream_t st) {
    auto k = vnm_spmm_kernel<NT>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NT>::kSmem) != cudaSuccess)
        return kLaunchCudaError;
    plan_units(a, L, NT);
    const int grid = a.nunits < num_sms() ? a.nunits : num_sms();
    k<<<grid, kThreads, Cfg<NT>::kSmem, st>>>(ta, tm, a);
    count_launch();
    dump_trace(st);
    return launch_reduce(a, L.T, st);
}

// split-K choice shared by both plans (and by vnm_spmm_workspace_bytes)
void plan_units(SpmmArgs& a, const SpmmLaunch& L, int NT) {
    a.ntt = (L.T + NT - 1) / NT;
    a.ntiles = a.nvb * a.ntt;
    const int n_stage = (a.nb_pad / 8 + kMmaPerStage - 1) / kMmaPerStage;
    a.trace = VNM_ENV_INT("VNM_SPMM_TRACE", 0);
    a.ks_n = 1;
    if (L.workspace) {
        const int ks = choose_ksplit(a.ntiles, n_stage);
        if (ks > 1 && L.workspace_bytes >= kWsTicketBytes + static_cast<size_t>(ks) * a.rows * L.T * 4) {
            a.ks_n = ks;
            a.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(L.workspace) + kWsTicketBytes);  // after the tickets
        }
    }
    a.sps = (n_stage + a.ks_n - 1) / a.ks_n;
    a.ks_n = (n_stage + a.sps - 1) / a.sps;  // no empty slices
    a.nunits = a.ntiles * a.ks_n;
}

int launch_reduce(const SpmmArgs& a, int T, cudaStream_t st) {
    if (a.ks_n > 1) {
        const int64_t n = static_cast<int64_t>(a.rows) * T;
        splitk_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(a.ws, a.ks_n, a.rows, T, a.YT,
                                                                                    a.ldy, a.y_bf16);
        count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}


}  // namespace

size_t spmm_workspace_bytes(const vnm_geom& g, int32_t T) {
    if (g.V < kV || T <= 0 || T > 64 || g.nb_pad == 0) return 0;  // split-K serves the small-T (gather) plan
    const int n_stage = (g.nb_pad / 8 + kMmaPerStage - 1) / kMmaPerStage;
    const int ks = choose_ksplit(g.rows_p / kV, n_stage);
    return ks > 1 ? kWsTicketBytes + static_cast<size_t>(ks) * g.rows * T * 4 : 0;
}

int launch_spmm(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    // V = 64: one V-block per 64-row tile; V = 128 / 256 (e.g. the paper's 128:2:M for M that has no tensor-core
    // form): 2 / 4 tiles share a V-block's column indices (each gathers them: correct, not faster)
    if (g.V < kV || g.V % kV) return kLaunchUnsupported;
    if (g.nb_pad == 0) {  // K == 0: Y = 0
        const size_t es = L.y_dtype == VNM_BF16 ? 2 : 4;
        return cudaMemset2DAsync(L.YT, static_cast<size_t>(L.ldy) * es, 0, static_cast<size_t>(L.T) * es, g.rows,
                                 stream) == cudaSuccess ? 0 : kLaunchCudaError;
    }
    // A_n: [rows_p][ld_val] bf16, box 64 values x 64 rows, 128B swizzle (values past ld_val zero-filled).
    CUtensorMap ta;
    if (!encode_2d(&ta, L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_val) * 2, 64, 64))
        return kLaunchCudaError;
    // A_i2: [rows_p][ld_meta] u32 (rows padded to 16 B, reading Q20), box 4 words x 64 rows, no swizzle; words
    // past nb_pad/8 zero-filled (the metadata warps substitute the pad pattern)
    CUtensorMap tm;
    if (!encode_2d(&tm, L.P->meta, static_cast<uint64_t>(g.nb_pad / 8), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_meta) * 4, kMmaPerStage, 64, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    SpmmArgs a;
    a.XT = L.XT;
    a.ldx = L.ldx;
    a.cols = g.cols;
    a.col_idx = L.P->col_idx;
    a.meta = L.P->meta;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.T = L.T;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.M = g.M;
    a.nb_pad = g.nb_pad;
    a.ld_meta = g.ld_meta;
    a.nvb = g.rows_p / kV;
    a.vdiv = g.V / kV;
    a.ntt = 0;
    a.ntiles = 0;
    if (L.T > 128) return launch_nt<256>(L, ta, tm, a, stream);
    if (L.T > 64) return launch_nt<128>(L, ta, tm, a, stream);
    return launch_nt<64>(L, ta, tm, a, stream);
}

}  // namespace vnm
