// probes.cu — TEST-ONLY hardware probes and microbenchmarks, built into a
// separate libvnm_probe.so that the product never loads.
//
// MB1 probe_sparse_mma: one CTA runs ONE tcgen05.mma.sp.cta_group::1.kind::f16 with caller-chosen
//     A (compressed, K-major, 128B swizzle), B (32 x 64, MN-major, 128B swizzle), metadata words
//     written into TMEM lanes 0..127 x 4 columns, and dumps all 128 lanes x 64 columns of D.  The host
//     (tests/probe_layouts.py) decodes which metadata bits steer which row / K-group and where each row
//     of D lands in TMEM.
// MB2 bench_mma: back-to-back MMAs from smem on every SM, to compare sparse M=64 / M=128 and dense.
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace vnm;

namespace {

constexpr uint32_t kMetaCol = 256;

__global__ void __launch_bounds__(128, 1)
    probe_sparse_mma_kernel(const uint16_t* __restrict__ A_in,   // [128][16] compressed values (bf16 bits)
                            const uint16_t* __restrict__ B_in,   // [32][64] dense B (bf16 bits), row k, col n
                            const uint32_t* __restrict__ E_in,   // [128][4] TMEM metadata words (lane, col)
                            float* __restrict__ D_out,           // [128][64] all TMEM lanes, columns 0..63
                            uint32_t m_mma, uint32_t id2, uint32_t e_col_off, uint32_t sparse) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];  // 16 atoms of 8 rows x 128 B
    __shared__ __align__(1024) uint8_t sB[4 * 1024];   // 4 K-groups of 8 rows x 128 B (64 n)
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;

    for (uint32_t i = tid; i < sizeof(sA) / 4; i += 128) reinterpret_cast<uint32_t*>(sA)[i] = 0;
    for (uint32_t i = tid; i < sizeof(sB) / 4; i += 128) reinterpret_cast<uint32_t*>(sB)[i] = 0;
    __syncthreads();
    // A: row m, value j (0..15) -> atom m/8, row m%8, byte 2j   (K-major SW128)
    for (uint32_t i = tid; i < 128 * 16; i += 128) {
        uint32_t m = i / 16, j = i % 16;
        *reinterpret_cast<uint16_t*>(sA + (m / 8) * 1024 + sw128_offset(m % 8, 2 * j)) = A_in[i];
    }
    // B: row k, column n -> K-group k/8, row k%8, byte 2n   (MN-major SW128, one 64-wide N chunk)
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

    // metadata: warp w writes lanes 32w..32w+31, columns kMetaCol..kMetaCol+3
    {
        const uint32_t* e = E_in + (warp * 32 + lane) * 4;
        tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + kMetaCol, e[0], e[1], e[2], e[3]);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(sB), 16384, 1024, kLayoutSW128);
        if (sparse) {
            const uint32_t idesc = idesc_bf16(m_mma, 64, true, id2, true);
            mma_sp_bf16(tbase, ad, bd, tbase + kMetaCol + e_col_off, idesc, 0);
        } else {
            const uint32_t idesc = idesc_bf16(m_mma, 64, false, 0, true);
            mma_bf16(tbase, ad, bd, idesc, 0);
        }
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

// MB2: every CTA issues `iters` MMAs of the given shape on resident operands, one commit at the end.
__global__ void __launch_bounds__(128, 1) bench_mma_kernel(uint32_t m_mma, uint32_t n_mma, uint32_t sparse,
                                                            uint32_t iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const uint32_t tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    // operands: A 128 rows x 128 B (16 KB), B 4 K-groups x up to 4 N-chunks (16 KB); zeros are fine
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
    tmem_st_32x32b_x4(tbase + ((warp * 32) << 16) + kMetaCol, 0x44444444u, 0x44444444u, 0x44444444u,
                      0x44444444u);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(smem), 16, 1024, kLayoutSW128);
        const uint64_t bd = sdesc(smem_u32(smem + 16384), 4096, 1024, kLayoutSW128);
        const uint32_t idesc = idesc_bf16(m_mma, n_mma, sparse != 0, 0, true);
        unsigned long long t0 = clock64();
        for (uint32_t i = 0; i < iters; ++i) {
            if (sparse)
                mma_sp_bf16(tbase, ad, bd, tbase + kMetaCol, idesc, i > 0);
            else
                mma_bf16(tbase, ad, bd, idesc, i > 0);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tbase, 512);
    (void)lane;
}

}  // namespace

extern "C" int vnm_probe_sparse_mma(const uint16_t* A_in, const uint16_t* B_in, const uint32_t* E_in,
                                    float* D_out, uint32_t m_mma, uint32_t id2, uint32_t e_col_off,
                                    uint32_t sparse, cudaStream_t stream) {
    probe_sparse_mma_kernel<<<1, 128, 0, stream>>>(A_in, B_in, E_in, D_out, m_mma, id2, e_col_off, sparse);
    return static_cast<int>(cudaGetLastError());
}

extern "C" int vnm_probe_bench_mma(uint32_t m_mma, uint32_t n_mma, uint32_t sparse, uint32_t iters,
                                   uint32_t nblocks, unsigned long long* cycles, cudaStream_t stream) {
    cudaFuncSetAttribute(bench_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    bench_mma_kernel<<<nblocks, 128, 32768, stream>>>(m_mma, n_mma, sparse, iters, cycles);
    return static_cast<int>(cudaGetLastError());
}
