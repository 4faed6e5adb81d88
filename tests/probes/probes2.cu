// probes2.cu — TEST-ONLY round-2 probes (built into libvnm_probe.so with probes.cu):
//   MB1b  interleaved M=64 accumulator (D address lane offset 16) and metadata lane offset
//   MB2b  sparse MMA throughput with independent accumulators
//   MB3a  TMA tile::gather4 placement into a 128B-swizzled atom
//   MB3b  L2/HBM -> SMEM throughput: gather4 (random 128 B rows) vs 2D tiles
//   CP    tcgen05.cp.128x128b placement (smem [128][16 B] -> TMEM lanes x 4 columns)
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace vnm;

namespace {

constexpr uint32_t kMetaCol2 = 256;

__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, int32_t col, int32_t r0, int32_t r1,
                                            int32_t r2, int32_t r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t d) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}

__global__ void __launch_bounds__(128, 1)
    probe_interleave_kernel(const uint16_t* __restrict__ A_in, const uint16_t* __restrict__ B_in,
                            const uint32_t* __restrict__ E_in, float* __restrict__ D_out, uint32_t d_lane,
                            uint32_t e_lane) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[4 * 1024];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (uint32_t i = tid; i < sizeof(sA) / 4; i += 128) reinterpret_cast<uint32_t*>(sA)[i] = 0;
    for (uint32_t i = tid; i < sizeof(sB) / 4; i += 128) reinterpret_cast<uint32_t*>(sB)[i] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < 128 * 16; i += 128) {
        uint32_t m = i / 16, j = i % 16;
        *reinterpret_cast<uint16_t*>(sA + (m / 8) * 1024 + sw128_offset(m % 8, 2 * j)) = A_in[i];
    }
    for (uint32_t i = tid; i < 32 * 64; i += 128) {
        uint32_t k = i / 64, n = i % 64;
        *reinterpret_cast<uint16_t*>(sB + (k / 8) * 1024 + sw128_offset(k % 8, 2 * n)) = B_in[i];
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    for (uint32_t c = 0; c < 64; c += 4) tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + c, 0, 0, 0, 0);
    {
        const uint32_t* e = E_in + (warp * 32 + lane) * 4;
        tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + kMetaCol2, e[0], e[1], e[2], e[3]);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(sB), 16384, 1024, kLayoutSW128);
        mma_sp_bf16(tbase + (d_lane << 16), ad, bd, tbase + (e_lane << 16) + kMetaCol2,
                    idesc_bf16(64, 64, true, 0, true), 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (uint32_t c = 0; c < 64; c += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tbase + ((warp * 32) << 16) + c, r);
        tmem_wait_ld();
        for (int i = 0; i < 16; ++i) D_out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(r[i]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

// mode 0: accumulators at column offsets a*n; mode 1: M=64 interleave (accumulator a at lane offset 16a)
__global__ void __launch_bounds__(128, 1) bench_mma_multi_kernel(uint32_t m_mma, uint32_t n_mma, uint32_t iters,
                                                                  uint32_t nacc, uint32_t mode,
                                                                  unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32;
    for (uint32_t i = tid; i < 32768 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + 448, 0x44444444u, 0x44444444u, 0x44444444u, 0x44444444u);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(smem + 16384), 4096, 1024, kLayoutSW128);
        const uint32_t idesc = idesc_bf16(m_mma, n_mma, true, 0, true);
        unsigned long long t0 = clock64();
        for (uint32_t i = 0; i < iters; ++i) {
            const uint32_t a = i % nacc;
            const uint32_t d = mode == 0 ? tbase + a * n_mma : tbase + ((a * 16u) << 16);
            mma_sp_bf16(d, ad, bd, tbase + 448, idesc, i >= nacc ? 1u : 0u);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

__global__ void probe_gather4_kernel(const __grid_constant__ CUtensorMap tm, const int32_t* rows, int32_t col,
                                     uint8_t* out) {
    __shared__ __align__(1024) uint8_t s[1024];
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0xEE;
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 1024);
        tma_gather4(s, &tm, col, rows[0], rows[1], rows[2], rows[3], &bar);
        tma_gather4(s + 512, &tm, col, rows[4], rows[5], rows[6], rows[7], &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = s[i];
}

// MB3b: each CTA streams `iters` stages of 16 KB into a 4-stage ring.  gather: 32 gather4 per stage issued by
// `lanes` threads (rows from a precomputed random table, 64-col chunk from a cheap hash); else one 2D tile.
__global__ void __launch_bounds__(32, 1) bench_tma_kernel(const __grid_constant__ CUtensorMap tm, int32_t nrows,
                                                          int32_t ncolchunks, int32_t iters, int32_t gather,
                                                          int32_t lanes, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[4];
    __shared__ int32_t table[4096];
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int lane = threadIdx.x;
    for (int i = lane; i < 4096; i += 32) {
        uint32_t h = (i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        table[i] = static_cast<int32_t>(h % static_cast<uint32_t>(nrows));
    }
    if (lane == 0) {
        for (int s = 0; s < 4; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint32_t cmask = static_cast<uint32_t>(ncolchunks - 1);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int s = it % 4;
        if (it >= 4) mbar_wait(&bars[s], ((it / 4) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&bars[s], 16384);
        __syncwarp();
        uint8_t* dst = buf + s * 16384;
        if (gather) {
            for (int g = lane; lane < lanes && g < 32; g += lanes) {
                const int b = (it * 32 + g) * 4;
                const int32_t col = static_cast<int32_t>(((it * 7 + g * 13) & cmask) * 64);
                tma_gather4(dst + g * 512, &tm, col, table[b & 4095], table[(b + 1) & 4095], table[(b + 2) & 4095],
                            table[(b + 3) & 4095], &bars[s]);
            }
        } else if (lane == 0) {
            const int32_t r0 = static_cast<int32_t>(((it * 2654435761u + blockIdx.x * 97u) >> 7) % static_cast<uint32_t>(nrows / 128)) * 128;
            const int32_t col = static_cast<int32_t>(((it * 7 + blockIdx.x) & cmask) * 64);
            tma_load_2d(dst, &tm, col, r0, &bars[s]);
        }
        __syncwarp();
    }
    for (int it = iters > 4 ? iters - 4 : 0; it < iters; ++it) mbar_wait(&bars[it % 4], (it / 4) & 1);
    if (lane == 0) cycles[blockIdx.x] = clock64() - t0;
}

__global__ void __launch_bounds__(128, 1) probe_tmem_cp_kernel(uint32_t lbo, uint32_t sbo, uint32_t* out) {
    __shared__ __align__(1024) uint32_t s[128 * 4 * 2];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (uint32_t i = tid; i < 128 * 8; i += 128) s[i] = i;
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    if (tid == 0) {
        tmem_cp_128x128b(tbase + kMetaCol2, sdesc(smem_u32(s), lbo, sbo, 0));
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t r[16];
    tmem_ld_32x32b_x16(tbase + ((warp * 32) << 16) + kMetaCol2, r);
    tmem_wait_ld();
    for (int i = 0; i < 4; ++i) out[(warp * 32 + lane) * 4 + i] = r[i];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn probe_encode() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<EncodeFn>(p);
}

int make_map(CUtensorMap* tm, const void* base, uint64_t rows, uint64_t cols, uint32_t box_c, uint32_t box_r) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    return static_cast<int>(probe_encode()(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

}  // namespace

extern "C" int vnm_probe_interleave(const uint16_t* A_in, const uint16_t* B_in, const uint32_t* E_in, float* D_out,
                                    uint32_t d_lane, uint32_t e_lane) {
    probe_interleave_kernel<<<1, 128>>>(A_in, B_in, E_in, D_out, d_lane, e_lane);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int vnm_probe_bench_mma_multi(uint32_t m, uint32_t n, uint32_t iters, uint32_t nacc, uint32_t mode,
                                         uint32_t nblocks, unsigned long long* cycles) {
    cudaFuncSetAttribute(bench_mma_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    bench_mma_multi_kernel<<<nblocks, 128, 32768>>>(m, n, iters, nacc, mode, cycles);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int vnm_probe_gather4(const uint16_t* X, int64_t rows, int64_t cols, uint32_t box_rows,
                                 const int32_t* row_idx, int32_t col, uint8_t* out) {
    CUtensorMap tm;
    int e = make_map(&tm, X, rows, cols, 64, box_rows);
    if (e) return 1000 + e;
    probe_gather4_kernel<<<1, 128>>>(tm, row_idx, col, out);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int vnm_probe_bench_tma(const uint16_t* X, int64_t rows, int64_t cols, int32_t iters, int32_t gather,
                                   int32_t lanes, uint32_t nblocks, unsigned long long* cycles) {
    CUtensorMap tm;
    int e = make_map(&tm, X, rows, cols, 64, gather ? 1 : 128);
    if (e) return 1000 + e;
    cudaFuncSetAttribute(bench_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 1024);
    bench_tma_kernel<<<nblocks, 32, 4 * 16384 + 1024>>>(tm, static_cast<int32_t>(rows),
                                                        static_cast<int32_t>(cols / 64), iters, gather, lanes, cycles);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int vnm_probe_tmem_cp(uint32_t lbo, uint32_t sbo, uint32_t* out) {
    probe_tmem_cp_kernel<<<1, 128>>>(lbo, sbo, out);
    return static_cast<int>(cudaGetLastError());
}

// =====================================================================================================
// Window probe: one sparse MMA (M = m_mma, N = 64) whose B descriptor walks K-groups of 8 rows with a
// caller-chosen stride: B is a dense [krows x 64] tile (MN-major), either 128B-swizzled with the swizzle
// phase taken from the ABSOLUTE row (as a TMA tile load writes it; layout 2, K-group stride = sbo) or
// unswizzled core matrices [8-token chunk][k-row][16 B] (layout 0, K-group stride = lbo).
// =====================================================================================================
namespace {
__global__ void __launch_bounds__(128, 1)
    probe_window_kernel(const uint16_t* __restrict__ A_in,  // [128][16]
                        const uint16_t* __restrict__ B_in,  // [krows][64]
                        const uint32_t* __restrict__ E_in,  // [128][4]
                        float* __restrict__ D_out,          // [128][64]
                        uint32_t m_mma, uint32_t krows, uint32_t layout, uint32_t lbo, uint32_t sbo,
                        uint32_t base_off, uint32_t start_row) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (uint32_t i = tid; i < sizeof(sA) / 4; i += 128) reinterpret_cast<uint32_t*>(sA)[i] = 0;
    for (uint32_t i = tid; i < sizeof(sB) / 4; i += 128) reinterpret_cast<uint32_t*>(sB)[i] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < 128 * 16; i += 128) {
        uint32_t m = i / 16, j = i % 16;
        *reinterpret_cast<uint16_t*>(sA + (m / 8) * 1024 + sw128_offset(m % 8, 2 * j)) = A_in[i];
    }
    for (uint32_t i = tid; i < krows * 64; i += 128) {
        uint32_t k = i / 64, n = i % 64;
        uint32_t off;
        if (layout == 2) off = (k / 8) * 1024 + sw128_offset(k % 8, 2 * n);        // row k at 128*k, phase k%8
        else off = (n / 8) * (krows * 16) + k * 16 + (n % 8) * 2;                  // [chunk][k][8 tokens]
        *reinterpret_cast<uint16_t*>(sB + off) = B_in[i];
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    {
        const uint32_t* e = E_in + (warp * 32 + lane) * 4;
        tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + kMetaCol2, e[0], e[1], e[2], e[3]);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
        uint64_t bd = sdesc(smem_u32(sB) + start_row * (layout == 2 ? 128u : 16u), lbo, sbo, layout);
        bd |= static_cast<uint64_t>(base_off & 7u) << 49;
        mma_sp_bf16(tbase, ad, bd, tbase + kMetaCol2, idesc_bf16(m_mma, 64, true, 0, true), 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (uint32_t c = 0; c < 64; c += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tbase + ((warp * 32) << 16) + c, r);
        tmem_wait_ld();
        for (int i = 0; i < 16; ++i) D_out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(r[i]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}
}  // namespace

extern "C" int vnm_probe_window(const uint16_t* A_in, const uint16_t* B_in, const uint32_t* E_in, float* D_out,
                                uint32_t m_mma, uint32_t krows, uint32_t layout, uint32_t lbo, uint32_t sbo,
                                uint32_t base_off, uint32_t start_row) {
    probe_window_kernel<<<1, 128>>>(A_in, B_in, E_in, D_out, m_mma, krows, layout, lbo, sbo, base_off, start_row);
    return static_cast<int>(cudaGetLastError());
}
