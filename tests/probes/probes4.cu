// probes4.cu — test-only microbenchmark (round 2): back-to-back tcgen05.mma(.sp) issued by a CONVERGED warp
// (elect.sync inside the asm, descriptors in uniform registers), with the A operand from shared memory (SS)
// or from TMEM (TS), on single CTAs (M = 128) and CTA pairs (cta_group::2, M = 256): which operand path bounds
// the sparse MMA rate the window-form SpMM kernels see.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"

namespace vnm {
namespace {

template <int CG>
__device__ __forceinline__ void issue(uint32_t d, uint64_t ad, uint32_t at, uint64_t bd, uint32_t e, uint32_t idesc,
                                      uint32_t acc, int ts, int sparse) {
    if constexpr (CG == 1) {
        if (sparse && ts)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %5, 0, p;\n\t"
                         "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %4, q;\n\t}" ::"r"(d),
                         "r"(at), "l"(bd), "r"(e), "r"(idesc), "r"(acc)
                         : "memory");
        else if (sparse)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %5, 0, p;\n\t"
                         "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, q;\n\t}" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(e), "r"(idesc), "r"(acc)
                         : "memory");
        else if (ts)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %4, 0, p;\n\t"
                         "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d), "r"(at),
                         "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
        else
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %4, 0, p;\n\t"
                         "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d), "l"(ad),
                         "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
    } else {
        if (sparse && ts)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %5, 0, p;\n\t"
                         "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%3], %4, q;\n\t}" ::"r"(d),
                         "r"(at), "l"(bd), "r"(e), "r"(idesc), "r"(acc)
                         : "memory");
        else if (sparse)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %5, 0, p;\n\t"
                         "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, q;\n\t}" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(e), "r"(idesc), "r"(acc)
                         : "memory");
        else if (ts)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %4, 0, p;\n\t"
                         "@p tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d), "r"(at),
                         "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
        else
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|p, 0xffffffff;\n\tsetp.ne.and.b32 q, %4, 0, p;\n\t"
                         "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(d), "l"(ad),
                         "l"(bd), "r"(idesc), "r"(acc)
                         : "memory");
    }
}

// TMEM: D columns [0, n), A (TS) columns 256.., metadata column 384 (0x4444 pattern: positions 0, 1)
template <int CG>
__global__ void __launch_bounds__(128, 1) bench_mma4_kernel(uint32_t n, int ts, int sparse, uint32_t iters,
                                                            unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    for (uint32_t i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        if constexpr (CG == 2) tmem_alloc_pair(&tmem_base, 512);
        else tmem_alloc(&tmem_base, 512);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base;
    // metadata pattern and zero A in TMEM (each warp its 32 lanes)
    for (int c = 0; c < 128; c += 4)
        tmem_st_32x32b_x4(tb + ((warp * 32) << 16) + 256 + c, 0, 0, 0, 0);
    tmem_st_32x32b_x4(tb + ((warp * 32) << 16) + 384, 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    tmem_wait_st();
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    if (warp == 0 && rank == 0) {
        const uint64_t ad = sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(smem + 16384), 8192, 1024, kLayoutSW128);
        const uint32_t idesc = idesc_bf16(CG == 2 ? 256 : 128, n, sparse != 0, 0, true);
        const unsigned long long t0 = clock64();
        for (uint32_t i = 0; i < iters; ++i) issue<CG>(tb, ad, tb + 256, bd, tb + 384, idesc, i > 0 ? 1u : 0u, ts, sparse);
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p tcgen05.commit.cta_group::%1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)), "n"(CG) : "memory");
        mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        if (tid == 0) cycles[blockIdx.x / CG] = t1 - t0;
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_pair(tb, 512);
        else tmem_dealloc(tb, 512);
    }
}

}  // namespace
}  // namespace vnm

// cycles[i] per CTA (CG = 1) or pair (CG = 2) for `iters` back-to-back MMAs
extern "C" int vnm_probe_bench_mma4(int cg, uint32_t n, int ts, int sparse, uint32_t iters, int nunits,
                                    unsigned long long* cycles) {
    using namespace vnm;
    const size_t smem = 65536 + 1024;
    if (cg == 1) {
        auto k = bench_mma4_kernel<1>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
            return 2;
        k<<<nunits, 128, smem>>>(n, ts, sparse, iters, cycles);
    } else {
        auto k = bench_mma4_kernel<2>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
            return 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * nunits);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k, n, ts, sparse, iters, cycles) != cudaSuccess) return 3;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    return 0;
}

// ---- TMA streaming of a [rows][cols] bf16 matrix in units of box_h rows x box_w values (SWIZZLE_128B when the
// box is 128 B wide), CTA c takes the contiguous unit range [c U / G, (c+1) U / G) of the (row group, K tile) list
// (the small-T plan's stream-K order), `stages` units in flight; optional second tensor streamed alongside with a
// box of [box_h rows][extra_w u32] per unit (the A_i2 rows of a unit).  Elapsed ns of the whole grid.
namespace vnm {
namespace {
__device__ unsigned long long g_p4_t[2];
__global__ void __launch_bounds__(288, 1) stream_units_kernel(const __grid_constant__ CUtensorMap tm,
                                                             const __grid_constant__ CUtensorMap tm2, int32_t ngr,
                                                             int32_t nk, int32_t box_h, int32_t box_w, int32_t stages,
                                                             uint32_t box_bytes, uint32_t extra_bytes, int32_t extra_w) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x >= 32) {  // spinning observer warps (like the small-T plan's consumers waiting on full[])
        const long long U = static_cast<long long>(ngr) * nk;
        const int n = static_cast<int>((blockIdx.x + 1) * U / gridDim.x - blockIdx.x * U / gridDim.x);
        for (int q = 0; q < n; ++q) mbar_wait(&bar[q % stages], (q / stages) & 1);
        return;
    }
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (blockIdx.x == 0) g_p4_t[0] = t0;
    const long long U = static_cast<long long>(ngr) * nk;
    const int u0 = static_cast<int>(blockIdx.x * U / gridDim.x), u1 = static_cast<int>((blockIdx.x + 1) * U / gridDim.x);
    const uint32_t slot = (box_bytes + extra_bytes + 1023) / 1024 * 1024;
    int q = 0;
    for (int u = u0; u < u1; ++u, ++q) {
        const int s = q % stages, gr = u / nk, k = u % nk;
        if (q >= stages) mbar_wait(&bar[s], ((q / stages) - 1) & 1);
        mbar_arrive_expect_tx(&bar[s], box_bytes + extra_bytes);
        tma_load_2d(smem + s * slot, &tm, k * box_w, gr * box_h, &bar[s]);
        if (extra_bytes) tma_load_2d(smem + s * slot + box_bytes, &tm2, k * extra_w, gr * box_h, &bar[s]);
    }
    for (int i = (q > stages ? q - stages : 0); i < q; ++i) mbar_wait(&bar[i % stages], (i / stages) & 1);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    atomicMax(&g_p4_t[1], t1);
}
}  // namespace
}  // namespace vnm

extern "C" int vnm_probe_stream_units(const uint16_t* A, int32_t rows, int32_t cols, int32_t box_h, int32_t box_w,
                                      int32_t stages, int32_t grid, const uint32_t* E, int32_t e_cols, int32_t extra_w,
                                      int32_t swz, int32_t spin_warps, unsigned long long* ns) {
    using namespace vnm;
    CUtensorMap tm, tm2;
    const CUtensorMapSwizzle sw = (swz && box_w * 2 == 128) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (!encode_2d(&tm, A, cols, rows, static_cast<uint64_t>(cols) * 2, box_w, box_h, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sw))
        return 2;
    tm2 = tm;
    if (extra_w && !encode_2d(&tm2, E, e_cols, rows, static_cast<uint64_t>(e_cols) * 4, extra_w, box_h,
                              CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return 2;
    const uint32_t box_bytes = box_h * box_w * 2, extra_bytes = extra_w ? box_h * extra_w * 4 : 0;
    const size_t smem = static_cast<size_t>(stages) * ((box_bytes + extra_bytes + 1023) / 1024 * 1024);
    if (stages > 16 || smem > 227 * 1024) return 5;
    if (cudaFuncSetAttribute(stream_units_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 3;
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_p4_t, z, sizeof(z));
    const int ngr = rows / box_h, nk = cols / box_w;
    stream_units_kernel<<<grid, 32 * (1 + spin_warps), smem>>>(tm, tm2, ngr, nk, box_h, box_w, stages, box_bytes, extra_bytes, extra_w);
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    unsigned long long h[2];
    cudaMemcpyFromSymbol(h, g_p4_t, sizeof(h));
    *ns = h[1] - h[0];
    return 0;
}

// ---- the window-form pair kernel's MMA issue pattern (spmm_tc3.cu), operands resident: per "stage" one
// mma_sp_stage<2> (4 sparse MMAs, B K-group stride sbo, B advanced by b_step per MMA, metadata column pair e / e+2)
// and a tcgen05.commit (multicast to both CTAs) on a per-slot mbarrier, slots cycling through `ring` B regions
// (start offsets stage_rows * 128 B apart, not 1024-aligned when stage_rows % 8 != 0); no waits on the commits.
namespace vnm {
namespace {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    bench_stage_pair_kernel(uint32_t n, uint32_t sbo, uint32_t b_step, uint32_t stage_rows, uint32_t ring,
                            uint32_t stages, int commit, unsigned long long* cycles, uint32_t lbo) {
    // commit == 2: the tc3 producer / MMA handshake: a producer thread waits empty[s] and arrives on full[s] (no
    // loads), the MMA warp waits full[s] before each stage and commits to empty[s] (both CTAs)
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[8], fullb[8], tfull[2], tempty[2];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32;
    const uint32_t rank = cluster_ctarank();
    for (uint32_t i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;  // (B ring + A)
    fence_proxy_async_smem();
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) {
            mbar_init(&bar[i], 1);
            mbar_init(&fullb[i], 1);
        }
        mbar_init(&done, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 2 * 8);  // 8 "epilogue" warps x 2 CTAs
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_pair(&tmem_base, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tb = tmem_base;
    if (warp < 4) {
        for (int c = 480; c < 512; c += 4)
            tmem_st_32x32b_x4(tb + ((warp * 32) << 16) + c, 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
        tmem_wait_st();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1 && rank == 0) {
        const uint32_t idesc0 = idesc_bf16(256, n, true, 0, true), idesc1 = idesc_bf16(256, n, true, 1, true);
        const uint64_t a0 = sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
        const unsigned long long t0 = clock64();
        for (uint32_t q = 0; q < stages; ++q) {
            const uint32_t s = q % ring;
            if (commit >= 4 && q % 5 == 0) {  // tile start: its accumulator is free (two tiles ago drained)
                const uint32_t tl = q / 5;
                mbar_wait(&tempty[tl & 1], ((tl >> 1) & 1) ^ 1);
                tc_fence_after();
            }
            if (commit >= 2) {
                mbar_wait(&fullb[s], (q / ring) & 1);
                if (commit == 5 && q % 5 != 4) mbar_wait(&fullb[(q + 1) % ring], ((q + 1) / ring) & 1);  // tc3's peek
                tc_fence_after();
            }
            const uint64_t bd = sdesc(smem_u32(smem + 81920 + s * stage_rows * 128), lbo, sbo, kLayoutSW128);
            const uint64_t ad = a0 + ((q % 5) * 16384 >> 4);
            mma_sp_stage<2>(tb + (q / 5 % 2) * 224 * (n <= 224), ad, bd, b_step >> 4, tb + 480 + 4 * (q % 5), idesc0, idesc1,
                            q % 5 ? 1u : 0u, 4);
            if (commit) mma_commit_pair_elect(&bar[s], 0x3);
            if (commit >= 4 && q % 5 == 4) mma_commit_pair_elect(&tfull[(q / 5) & 1], 0x3);
        }
        mma_commit_pair_elect(&done, 0x3);
        if ((threadIdx.x & 31) == 0) mbar_wait(&done, 0);
        __syncwarp();
        const unsigned long long t1 = clock64();
        if (tid == 32) cycles[blockIdx.x / 2] = t1 - t0;
    } else if (warp >= 2 && commit >= 4) {
        // commit == 4: 8 "epilogue" warps per CTA take every tile's accumulator (tmem_full) and release it at once
        for (uint32_t tl = 0; tl < stages / 5; ++tl) {
            mbar_wait(&tfull[tl & 1], (tl >> 1) & 1);
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                if (rank == 0) mbar_arrive(&tempty[tl & 1]);
                else mbar_arrive_remote(&tempty[tl & 1], 0);
            }
        }
    } else if (warp >= 2 && commit >= 3) {
        // commit == 3: 8 extra warps spin-wait (mbarrier try_wait loop) on a barrier that completes only at the end,
        // like the window kernels' epilogue warps waiting for an accumulator
        mbar_wait(&done, 0);
    } else if (warp == 0 && commit >= 2 && (threadIdx.x & 31) == 0 && rank == 0) {
        if (commit == 6) {  // a short stall before each arrival (the producer's TMA issue)
        }
        for (uint32_t q = 0; q < stages; ++q) {
            const uint32_t s = q % ring;
            mbar_wait(&bar[s], ((q / ring) & 1) ^ 1);
            mbar_arrive(&fullb[s]);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_pair(tb, 512);
    }
}
}  // namespace
}  // namespace vnm

extern "C" int vnm_probe_bench_stage_pair(uint32_t n, uint32_t sbo, uint32_t b_step, uint32_t stage_rows, uint32_t ring,
                                          uint32_t stages, int commit, int pairs, unsigned long long* cycles) {
    using namespace vnm;
    const size_t smem = 200 * 1024;
    if (cudaFuncSetAttribute(bench_stage_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 2;
    bench_stage_pair_kernel<<<2 * pairs, commit >= 3 ? 320 : 128, smem>>>(n, sbo, b_step, stage_rows, ring, stages, commit, cycles,
                                                                          16384u);
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    return 0;
}
// the same with the B operand's chunk stride (UMMA LBO) given: tc3 uses the ring's whole region (ring_rows * 128 B)
extern "C" int vnm_probe_bench_stage_pair_lbo(uint32_t n, uint32_t sbo, uint32_t b_step, uint32_t stage_rows, uint32_t ring,
                                              uint32_t stages, int commit, int pairs, unsigned long long* cycles, uint32_t lbo) {
    using namespace vnm;
    const size_t smem = 220 * 1024;
    if (cudaFuncSetAttribute(bench_stage_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 2;
    bench_stage_pair_kernel<<<2 * pairs, commit >= 3 ? 320 : 128, smem>>>(n, sbo, b_step, stage_rows, ring, stages, commit, cycles,
                                                                          lbo);
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    return 0;
}
