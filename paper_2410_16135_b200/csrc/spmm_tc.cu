// spmm_tc.cu — the V:N:M SpMM in the tensor-core "window" form (include/vnm.h values_tc / meta_tc,
// DESIGN.md §6), for V = 64 and 4 <= M <= 8 at prefill-sized T.
//
// Why a second formulation.  On B200 the M = 64 sparse MMA (one V-block) runs at half the M = 128 rate
// (csrc/probes.cu MB2), and gathering each V-block's 4 kept X^T rows per block (App. A) is bound by
// the gather path (TMA gather4 7-15 B/clk/SM, cp.async ~27 B/clk/SM: MB3b) rather than by the MMA.  Here
// every V x M block is an 8-channel window of the DENSE X^T tile — the sparse MMA's K-group stride is set
// to M rows (UMMA SBO = M * 128 B; measured exact, probes2.cu "window") — so one X^T tile loaded by plain
// 2D TMA serves all output rows: M = 128 MMAs (two V-blocks), and RT = 2 row tiles per CTA share each
// X^T tile in shared memory (a 2-CTA multicast of the tile was measured no faster: at cluster size <= 4
// multicast costs about the same L2 traffic as unicast).
// Cost in tensor-core work: 8 logical K per block instead of 4, i.e. the same MMA time as the M = 64 gather
// plan (2x K at 2x rate) for 5 <= M <= 8, with no gather at all.
//
// Tile = RT x 128 output rows x NT tokens; stage = 4 MMAs per row tile (16 blocks, or 32 for M = 4):
//   warp 0     TMA: A (values_tc 128 x 64 bf16) and the metadata chunk (2 KB bulk copy) of each row tile,
//              and the dense X^T tile (NT/64 boxes of 64 tokens x rows);
//   warp 1     MMA: tcgen05.cp (metadata smem -> TMEM) then 4 x RT tcgen05.mma.sp M=128 N=NT;
//   warps 4-7  epilogue: TMEM -> fp32 / bf16 -> shared staging -> TMA tensor store of Y^T (accumulators
//              double-buffered when TMEM allows).
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

// timing-ablation flags (VNM_ABL): a compile-time 0 in production builds, so no ablation test is left in the loops
#ifdef VNM_ABLATIONS
#define ABL(args) ((args).abl)
#else
#define ABL(args) 0
#endif

constexpr int kThreads = 256;
constexpr uint32_t kABytes = 128 * 128;  // 128 rows x 64 bf16
constexpr uint32_t kEBytes = 128 * 16;   // 128 lanes x 4 words
constexpr uint32_t kYBytes = 32 * 128;   // epilogue staging per warp: 32 rows x 128 B (SW128), one TMA store

struct TcArgs {
    const uint32_t* meta_tc;
    void* YT;
    int64_t ldy;
    int32_t T, y_bf16, rows, M;
    int32_t n_mma, n_stage, n_rt, n_tt, n_rg, work;
    int32_t row_major;   // tile order: row-tile-major (A reused across token tiles) or token-tile-major
    int32_t rows_stage;  // dense X^T rows advanced per stage
    int32_t rb;          // B rows per stage per chunk (multiple of 8)
    int32_t stages;      // pipeline depth
    uint32_t b_stage_bytes, stage_bytes;
    int32_t abl;         // VNM_ABL (timing ablations only, results invalid): see spmm_tc2.cu
    int32_t pf;          // L2 prefetch distance in stages (0: none): X^T streamed from HBM
};


// NT tokens per tile (NT/64 TMA chunks); RT row tiles of 128 rows per CTA share every B tile; NACC
// accumulator sets (double buffering when they fit in TMEM next to the metadata slots).
template <int NT, int RT>
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                       const __grid_constant__ CUtensorMap tmap_y, const TcArgs a) {
    constexpr int kChunks = NT / 64;
    constexpr int NACC = 2 * RT * NT + 16 * RT <= 512 ? 2 : 1;
    constexpr uint32_t kMetaCol = NACC * RT * NT;  // TMEM: accumulators, then 4 metadata columns per stage & tile
    extern __shared__ __align__(1024) uint8_t smem[];  // (not re-aligned through an integer: keeps LDS/STS)
    const int S = a.stages;
    // per stage: [A x RT][B chunks][E x RT]; then 4 epilogue staging buffers, then the barriers
    uint8_t* sY = smem + S * a.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sY + 4 * kYBytes);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const uint32_t b_off = RT * kABytes, e_off = RT * kABytes + a.b_stage_bytes;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_y);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_wait();    // the previous kernel's outputs (e.g. this layer's inputs) are visible
    grid_dep_launch();  // the next kernel may take SMs as this grid's CTAs exit

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int q = 0;
            for (int w = blockIdx.x; w < a.work; w += gridDim.x) {
                const int rg = a.row_major ? w / a.n_tt : w % a.n_rg, tt = a.row_major ? w % a.n_tt : w / a.n_rg;
                const int n0 = tt * NT;
                for (int st = 0; st < a.n_stage; ++st, ++q) {
                    const int s = q % S;
                    mbar_wait(&empty[s], ((q / S) & 1) ^ 1);
                    uint8_t* base = smem + s * a.stage_bytes;
                    if (ABL(a) & 4) {
                        mbar_arrive(&full[s]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[s], RT * (kABytes + kEBytes) + a.b_stage_bytes);
#pragma unroll
                    for (int j = 0; j < RT; ++j) {
                        const int rt = rg * RT + j;  // row tiles past n_rt read as zeros (TMA OOB)
                        tma_load_2d(base + j * kABytes, &tmap_a, st * 64, rt * 128, &full[s]);
                        const int rte = rt < a.n_rt ? rt : 0;
                        bulk_load(base + e_off + j * kEBytes, a.meta_tc + (static_cast<int64_t>(rte) * a.n_stage + st) * 512,
                                  kEBytes, &full[s]);
                    }
#pragma unroll
                    for (int c = 0; c < kChunks; ++c)
                        tma_load_2d(base + b_off + c * (a.rb * 128), &tmap_b, n0 + 64 * c, st * a.rows_stage, &full[s]);
                    if (a.pf && st + a.pf < a.n_stage) {  // warm L2 for a later stage of this tile (beyond the ring)
#pragma unroll
                        for (int c = 0; c < kChunks; ++c)
                            tma_prefetch_l2(&tmap_b, n0 + 64 * c, (st + a.pf) * a.rows_stage);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (converged warp, elected lane)
        int q = 0, tl = 0;
        const uint32_t idesc0 = idesc_bf16(128, NT, true, 0, true);
        const uint32_t idesc1 = idesc_bf16(128, NT, true, 1, true);
        // B descriptor advance per MMA (window-16 form, M > 8: +8 rows to the second half-windows, then the next
        // block group 4M rows on: ptx.cuh mma_sp_stage)
        const uint64_t b_step = (a.M == 4 ? 32u : a.M > 8 ? 8u : 4u * a.M) * 128u >> 4;
        const uint64_t b_step2 = a.M > 8 ? (4u * a.M * 128u) >> 4 : 2 * b_step;
        const uint32_t sbo = a.M == 4 ? 1024u : a.M * 128u;                 // K-group (window) stride
        const uint32_t b_lbo = a.rb * 128;
        for (int w = blockIdx.x; w < a.work; w += gridDim.x, ++tl) {
            const int acc = NACC == 2 ? (tl & 1) : 0;
            mbar_wait(&tmem_empty[acc], ((NACC == 2 ? (tl >> 1) : tl) & 1) ^ 1);
            tc_fence_after();
            for (int st = 0; st < a.n_stage; ++st, ++q) {
                const int s = q % S;
                mbar_wait(&full[s], (q / S) & 1);
                tc_fence_after();
                uint8_t* base = smem + s * a.stage_bytes;
                const uint32_t meta_s = tmem + kMetaCol + 4 * RT * s;
                if (!(ABL(a) & 8) || q < S) {
#pragma unroll
                    for (int j = 0; j < RT; ++j)
                        tmem_cp_elect<1>(meta_s + 4 * j, sdesc(smem_u32(base + e_off + j * kEBytes), 16, 128, 0));
                }
                const uint64_t bd = sdesc(smem_u32(base + b_off), b_lbo, sbo, kLayoutSW128);
                const int left = a.n_mma - st * 4;
                const uint32_t n = left < 4 ? static_cast<uint32_t>(left) : 4u;
#pragma unroll
                for (int j = 0; j < RT; ++j)
                    mma_sp_stage<1>(tmem + (acc * RT + j) * NT, sdesc(smem_u32(base + j * kABytes), 16, 1024, kLayoutSW128),
                                    bd, b_step, b_step2, meta_s + 4 * j, idesc0, idesc1, st > 0 ? 1u : 0u, n);
                mma_commit_elect(&empty[s]);
            }
            mma_commit_elect(&tmem_full[acc]);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        // TMEM -> registers -> bf16 / fp32 -> the warp's 32 x 128 B staging buffer (SW128: 16-byte chunk c of
        // row r at c ^ (r % 8), conflict-free) -> one TMA tensor store per chunk of 128 B per row; the store
        // clips rows >= rows and tokens >= T.
        const int qd = warp - 4;
        uint8_t* buf = sY + qd * kYBytes;
        const uint32_t buf_row = smem_u32(buf) + lane * 128;
        const int cw = a.y_bf16 ? 64 : 32;  // tokens per 128-byte chunk
        int tl = 0;
        for (int w = blockIdx.x; w < a.work; w += gridDim.x, ++tl) {
            const int rg = a.row_major ? w / a.n_tt : w % a.n_rg, tt = a.row_major ? w % a.n_tt : w / a.n_rg;
            const int n0 = tt * NT;
            const int acc = NACC == 2 ? (tl & 1) : 0;
            mbar_wait(&tmem_full[acc], (NACC == 2 ? (tl >> 1) : tl) & 1);
            tc_fence_after();
            if constexpr (NACC == 1 && RT == 1) {
                if (a.y_bf16 && !(ABL(a) & 3)) {
                    // one accumulator: drain the warp's whole 32 x NT block into packed bf16 registers and release
                    // the accumulator BEFORE the stores (the next tile's MMAs no longer wait for the epilogue)
                    constexpr int kC = NT / 64;
                    uint32_t pk[kC][32];
#pragma unroll
                    for (int c = 0; c < kC; ++c)
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem + ((32 * qd) << 16) + 64 * c + 16 * hh, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                __nv_bfloat162 b2 =
                                    __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                                pk[c][8 * hh + k] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                        }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tmem_empty[acc]);
                    const int rt = rg;
                    if (rt < a.n_rt) {
#pragma unroll
                        for (int c = 0; c < kC; ++c) {
                            if (n0 + 64 * c >= a.T) break;
                            if (lane == 0) bulk_wait_read0();  // the previous store has read the buffer
                            __syncwarp();
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                                 buf_row + (((k ^ lane) & 7) << 4)),
                                             "r"(pk[c][4 * k]), "r"(pk[c][4 * k + 1]), "r"(pk[c][4 * k + 2]),
                                             "r"(pk[c][4 * k + 3])
                                             : "memory");
                            fence_proxy_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                tma_store_2d(&tmap_y, n0 + 64 * c, rt * 128 + 32 * qd, buf);
                                bulk_commit();
                            }
                        }
                    }
                    continue;
                }
            }
#pragma unroll 1
            for (int j = 0; j < RT; ++j) {
                const int rt = rg * RT + j;
                if (rt >= a.n_rt || (ABL(a) & 1)) break;
#pragma unroll 1
                for (int c = 0; c < NT && n0 + c < a.T; c += cw) {
                    uint32_t pk[32];
                    if (a.y_bf16) {
#pragma unroll
                        for (int hh = 0; hh < 4; ++hh) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem + ((32 * qd) << 16) + (acc * RT + j) * NT + c + 16 * hh, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                __nv_bfloat162 b2 =
                                    __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                                pk[8 * hh + k] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                        }
                    } else {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tmem + ((32 * qd) << 16) + (acc * RT + j) * NT + c + 16 * hh, v);
                            tmem_wait_ld();
#pragma unroll
                            for (int k = 0; k < 16; ++k) pk[16 * hh + k] = v[k];
                        }
                    }
                    if (ABL(a) & 2) continue;
                    if (lane == 0) bulk_wait_read0();  // the previous store has read the buffer
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         buf_row + (((k ^ lane) & 7) << 4)),
                                     "r"(pk[4 * k]), "r"(pk[4 * k + 1]), "r"(pk[4 * k + 2]), "r"(pk[4 * k + 3])
                                     : "memory");
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tmap_y, n0 + c, rt * 128 + 32 * qd, buf);
                        bulk_commit();
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[acc]);
        }
        if (lane == 0) bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

bool encode(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t bi,
            uint32_t bo) {
    return encode_2d(tm, base, inner, outer, row_bytes, bi, bo);
}

template <int NT, int RT>
int launch_cfg(const SpmmLaunch& L, TcArgs a, cudaStream_t stream) {
    constexpr int kChunks = NT / 64;
    const vnm_geom& g = L.P->g;
    a.n_tt = (L.T + NT - 1) / NT;
    // rows one stage's windows touch: window form block 15 (15M .. 15M+7); window-16 form block 7 (7M .. 7M+15)
    a.rows_stage = g.M == 4 ? 128 : g.M > 8 ? 8 * g.M : 16 * g.M;
    const int need = g.M == 4 ? 128 : g.M > 8 ? 7 * g.M + 16 : 15 * g.M + 8;
    a.rb = (need + 7) / 8 * 8;
    a.b_stage_bytes = static_cast<uint32_t>(kChunks * a.rb * 128);
    a.stage_bytes = RT * (kABytes + kEBytes) + a.b_stage_bytes;
    a.stage_bytes = (a.stage_bytes + 1023) / 1024 * 1024;
    a.stages = static_cast<int>((224u * 1024u - 4 * kYBytes) / a.stage_bytes);
    if (a.stages > 4) a.stages = 4;
    if (a.stages < 2) return kLaunchUnsupported;
    a.n_rg = (a.n_rt + RT - 1) / RT;
    a.work = a.n_rg * a.n_tt;
    CUtensorMap ta, tb;
    const int ld_tc = 16 * a.n_mma;
    const int rows_w = a.n_rt * 128;
    if (!encode(&ta, L.P->values_tc, static_cast<uint64_t>(ld_tc), static_cast<uint64_t>(rows_w),
                static_cast<uint64_t>(ld_tc) * 2, 64, 128))
        return kLaunchCudaError;
    if (!encode(&tb, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), static_cast<uint64_t>(L.ldx) * 2,
                64, static_cast<uint32_t>(a.rb)))
        return kLaunchCudaError;
    // Y^T [rows][ldy]: box 128 B of tokens x 32 rows, 128B swizzle (the epilogue staging layout)
    CUtensorMap ty;
    const bool bf = L.y_dtype == VNM_BF16;
    if (!encode_2d(&ty, L.YT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.rows),
                   static_cast<uint64_t>(L.ldy) * (bf ? 2 : 4), bf ? 64 : 32, 32,
                   bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32))
        return kLaunchCudaError;
    const size_t smem = static_cast<size_t>(a.stages) * a.stage_bytes + 4 * kYBytes + 1024 + 256;
    auto k = vnm_spmm_tc_kernel<NT, RT>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return kLaunchCudaError;
    const int grid = a.work < num_sms() ? a.work : num_sms();
    a.abl = VNM_ABLATION_FLAGS();
    // opt-in (VNM_TC_PF): the 1-CTA kernel alone gained 11 % on DeiT-B fc2-sized K, but whole steps got slower
    // (DeiT-B 0.519 -> 0.554 ms: profiles/r01f_experiments.md)
    a.pf = VNM_ENV_INT("VNM_TC_PF", 0);
    cudaError_t e = launch_pdl(false, k, dim3(grid), dim3(kThreads), smem, stream, ta, tb, ty, a);
    count_launch();
    return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

int launch_spmm_tc(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    // window form (M <= 8) / window-16 form (8 < M < 16): rows independent of V
    if (g.V < 32 || g.V > 128 || g.M > 15) return kLaunchUnsupported;
    TcArgs a;
    a.meta_tc = L.P->meta_tc;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.T = L.T;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.M = g.M;
    a.n_mma = g.M > 8 ? g.nb_pad / 2 : g.nb_pad / (g.M == 4 ? 8 : 4);
    a.n_stage = (a.n_mma + 3) / 4;
    a.n_rt = (g.rows_p + 127) / 128;
    // Plan (measured, profiles/r01_*): long K (many stages per tile) -> NT = 256, one accumulator (the
    // epilogue is amortised over the K loop); short K -> NT = 192 with double-buffered accumulators so the
    // epilogue overlaps the next tile.  RT = 2 (two row tiles sharing each X^T tile) measured no faster.
    // VNM_TC_CFG_NT / VNM_TC_CFG_RT override (tuning experiments).
    // Tile order: the larger operand is the one to keep hot in L2 across the tiles resident at a time —
    // row-tile-major when the window-form weights outweigh X^T (Llama), token-tile-major otherwise (DeiT).
    a.row_major = static_cast<int64_t>(a.n_rt) * 128 * 16 * a.n_mma > static_cast<int64_t>(g.cols) * L.T ? 1 : 0;
    // (3 or fewer row tiles: 256-token tiles quantise evenly over the SMs, measured faster for DeiT proj)
    int nt = (a.n_stage >= 12 || a.n_rt <= 3) ? 256 : 192, rt = 1;
    if (const int v = VNM_ENV_INT("VNM_TC_CFG_NT", 0)) nt = v;
    if (const int v = VNM_ENV_INT("VNM_TC_CFG_RT", 0)) rt = v;
    if (nt == 256 && rt == 1) return launch_cfg<256, 1>(L, a, stream);
    if (nt == 128 && rt == 1) return launch_cfg<128, 1>(L, a, stream);
    if (nt == 128 && rt == 2) return launch_cfg<128, 2>(L, a, stream);
    if (nt == 192 && rt == 2) return launch_cfg<192, 2>(L, a, stream);
    return launch_cfg<192, 1>(L, a, stream);
}

}  // namespace vnm
