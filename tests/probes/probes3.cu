// probes3.cu — test-only microbenchmark (round 1b): back-to-back tcgen05.mma(.sp) on CTA PAIRS
// (cta_group::2, M = 256) from resident shared memory, optionally with a concurrent TMA stream into the
// same shared memory (the window SpMM's load traffic), to find the MMA ceiling of spmm_tc2.cu.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"

namespace vnm {
namespace {

// smem: A 16 KB | B 4 chunks x 4 KB x ... (48 KB window region) | TMA sink 96 KB
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    bench_mma_pair_kernel(const __grid_constant__ CUtensorMap tm, uint32_t n_mma, uint32_t sparse, uint32_t sbo,
                          uint32_t iters, uint32_t tma_kb_per_mma, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar, tbar[2];
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32;
    const uint32_t rank = cluster_ctarank();
    for (uint32_t i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&tbar[0], 1);
        mbar_init(&tbar[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_pair(&tmem_base, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + 256, 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    tmem_wait_st();
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (tid == 0 && rank == 0) {
        const uint64_t ad = sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(smem + 16384), 8192, sbo, kLayoutSW128);
        const uint32_t idesc = idesc_bf16(256, n_mma, sparse != 0, 0, true);
        unsigned long long t0 = clock64();
        for (uint32_t i = 0; i < iters; ++i) {
            if (sparse)
                mma_sp_bf16_pair(tbase, ad, bd, tbase + 256, idesc, i > 0);
            else
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(i > 0 ? 1u : 0u)
                    : "memory");
        }
        mma_commit_pair(&bar, 0x3);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        cycles[blockIdx.x / 2] = t1 - t0;
    } else if (tid == 32 && tma_kb_per_mma) {
        // concurrent TMA stream: tma_kb_per_mma KB per MMA-equivalent, 16 KB boxes (64 x 128 rows) into a
        // 96 KB sink, two in flight
        const uint32_t nbox = (iters * tma_kb_per_mma) / 48;  // groups of 3 boxes
        for (uint32_t i = 0; i < nbox; ++i) {
            const int s = i & 1;
            if (i >= 2) mbar_wait(&tbar[s], ((i / 2) - 1) & 1);
            mbar_arrive_expect_tx(&tbar[s], 16384 * 3);
            for (int j = 0; j < 3; ++j)
                tma_load_2d(smem + 65536 + (s * 3 + j) * 16384, &tm, 0, ((blockIdx.x * 7 + i * 3 + j) * 128) % 8192, &tbar[s]);
        }
        if (nbox >= 1) mbar_wait(&tbar[(nbox - 1) & 1], ((nbox - 1) / 2) & 1);
        if (nbox >= 2) mbar_wait(&tbar[(nbox - 2) & 1], ((nbox - 2) / 2) & 1);
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_pair(tbase, 512);
    }
}

}  // namespace
}  // namespace vnm

// X: bf16 [8192][64] (1 MB, L2-resident) feeds the concurrent TMA stream.  cycles: one per pair.
extern "C" int vnm_probe_bench_mma_pair(const uint16_t* X, uint32_t n_mma, uint32_t sparse, uint32_t sbo,
                                        uint32_t iters, uint32_t tma_kb_per_mma, int pairs, unsigned long long* cycles) {
    using namespace vnm;
    CUtensorMap tm;
    if (!encode_2d(&tm, X, 64, 8192, 128, 64, 128)) return 2;
    const size_t smem = 65536 + 96 * 1024 + 1024;
    if (cudaFuncSetAttribute(bench_mma_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 3;
    bench_mma_pair_kernel<<<2 * pairs, 128, smem>>>(tm, n_mma, sparse, sbo, iters, tma_kb_per_mma, cycles);
    if (cudaGetLastError() != cudaSuccess) return 4;
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 5;
}

// ---- DRAM access pattern probe: stream a [rows][ld] bf16 matrix with TMA boxes of box_h rows x box_w
// values; CTA c takes row groups c, c + grid, ... and walks each group's K tiles in order (the decode
// kernels' pattern), `stages` boxes in flight.  Returns elapsed ns (globaltimer) of the whole grid.
namespace vnm {
namespace {
__device__ unsigned long long g_p3_t[2];
__global__ void __launch_bounds__(32, 1) stream_boxes_kernel(const __grid_constant__ CUtensorMap tm, int32_t rows,
                                                              int32_t cols, int32_t box_h, int32_t box_w, int32_t stages,
                                                              uint32_t box_bytes) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t bar[8];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (blockIdx.x == 0) g_p3_t[0] = t0;
    const int ngr = (rows + box_h - 1) / box_h, nk = (cols + box_w - 1) / box_w;
    int q = 0;
    for (int gr = blockIdx.x; gr < ngr; gr += gridDim.x)
        for (int k = 0; k < nk; ++k, ++q) {
            const int s = q % stages;
            if (q >= stages) mbar_wait(&bar[s], ((q / stages) - 1) & 1);
            mbar_arrive_expect_tx(&bar[s], box_bytes);
            tma_load_2d(smem + s * box_bytes, &tm, k * box_w, gr * box_h, &bar[s]);
        }
    for (int i = (q > stages ? q - stages : 0); i < q; ++i) mbar_wait(&bar[i % stages], (i / stages) & 1);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    atomicMax(&g_p3_t[1], t1);
}
}  // namespace
}  // namespace vnm

extern "C" int vnm_probe_stream_boxes(const uint16_t* A, int32_t rows, int32_t cols, int64_t ld, int32_t box_h,
                                      int32_t box_w, int32_t stages, int32_t grid, unsigned long long* ns) {
    using namespace vnm;
    CUtensorMap tm;
    if (!encode_2d(&tm, A, cols, rows, ld * 2, box_w, box_h, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_NONE))
        return 2;
    const uint32_t box_bytes = box_h * box_w * 2;
    const size_t smem = static_cast<size_t>(stages) * box_bytes + 128;
    if (cudaFuncSetAttribute(stream_boxes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return 3;
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_p3_t, z, sizeof(z));
    stream_boxes_kernel<<<grid, 32, smem>>>(tm, rows, cols, box_h, box_w, stages, box_bytes);
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    unsigned long long h[2];
    cudaMemcpyFromSymbol(h, g_p3_t, sizeof(h));
    *ns = h[1] - h[0];
    return 0;
}

// ---- legacy warp-level sparse MMA rate: every warp issues `iters` x 4 independent mma.sp m16n8k32 (bf16)
namespace vnm {
namespace {
__global__ void __launch_bounds__(512) bench_mma_sync_sp_kernel(uint32_t iters, float* sink) {
    float d[4][4] = {};
    uint32_t a[4] = {0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u}, b[4] = {0x3f803f80u, 0, 0, 0};
    const uint32_t e = 0x44444444u;
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile(
                "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, "
                "%6, %7}, {%8, %9, %10, %11}, {%0, %1, %2, %3}, %12, 0x0;"
                : "+f"(d[k][0]), "+f"(d[k][1]), "+f"(d[k][2]), "+f"(d[k][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(e));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    if (s == 12345.f) sink[threadIdx.x] = s;
}
}  // namespace
}  // namespace vnm

// returns ns for grid x warps_per_cta warps each issuing iters x 4 MMAs
extern "C" int vnm_probe_mma_sync_sp(uint32_t iters, int grid, int warps, float* sink, unsigned long long* ns) {
    using namespace vnm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench_mma_sync_sp_kernel<<<grid, 32 * warps>>>(16, sink);
    cudaEventRecord(e0);
    bench_mma_sync_sp_kernel<<<grid, 32 * warps>>>(iters, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return 4;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ns = static_cast<unsigned long long>(ms * 1e6);
    return 0;
}

// ---------------------------------------------------------------- PDL ordering check (tests/test_gpu_spmm.py)
// One CTA: lets its programmatic dependents launch at once (griddepcontrol.launch_dependents), then spins for
// `delay` cycles and only then copies src -> dst.  A dependent kernel launched right after it with programmatic
// stream serialization (e.g. the small-T vnm_spmm) overlaps the spin; only its griddepcontrol.wait keeps it from
// reading dst before the copy — so a missing wait shows as wrong results, not as a narrow race.
namespace vnm {
namespace {
__global__ void delayed_copy_kernel(uint4* dst, const uint4* src, size_t n16, long long delay) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long t0 = clock64();
    while (clock64() - t0 < delay) {
    }
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
}
}  // namespace
}  // namespace vnm

extern "C" int vnm_probe_delayed_copy(void* dst, const void* src, size_t bytes, long long delay_cycles, void* stream) {
    vnm::delayed_copy_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint4*>(dst), static_cast<const uint4*>(src), bytes / 16, delay_cycles);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
