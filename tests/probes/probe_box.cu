// TEST-ONLY probe: smem layout TMA produces for a 2-D box whose inner extent (32 / 48 bf16 = 64 / 96 B) is
// narrower than the 128-byte swizzle span.  Prints, for each box row r and 16-byte chunk c, the smem byte
// offset where it landed.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2410_16135_b200/csrc/tmap.h"
#include "../../paper_2410_16135_b200/csrc/ptx.cuh"
using namespace vnm;
__global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t* out) {
    __shared__ __align__(1024) uint16_t s[4096];
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0xFFFF;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, 0);  // placeholder, real count below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_load_2d(s, &tm, 0, 0, &bar);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = s[i];
}
__global__ void k2(const __grid_constant__ CUtensorMap tm, uint16_t* out, uint32_t bytes) {
    __shared__ __align__(1024) uint16_t s[4096];
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0xFFFF;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    __syncthreads();
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, bytes);
        tma_load_2d(s, &tm, 0, 0, &bar);
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = s[i];
}
int main() {
    const int R = 16, C = 128;
    uint16_t h[R * C];
    for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
    uint16_t *d, *o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8192);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int bi : {64, 32, 48, 56}) {
        CUtensorMap tm;
        if (!encode_2d(&tm, d, C, R, C * 2, bi, 8)) { printf("box %d: encode failed\n", bi); continue; }
        cudaMemset(o, 0, 8192);
        k2<<<1, 128>>>(tm, o, bi * 8 * 2);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("box %d: %s\n", bi, cudaGetErrorString(e)); return 1; }
        uint16_t s[4096]; cudaMemcpy(s, o, 8192, cudaMemcpyDeviceToHost);
        printf("box inner %d bf16 (%d B): element (r, c) -> smem byte offset\n", bi, bi * 2);
        for (int r = 0; r < 8; ++r) {
            printf("  r%d:", r);
            for (int c = 0; c < bi; c += 8) {
                int off = -1;
                for (int i = 0; i < 4096; ++i) if (s[i] == (uint16_t)(r * 256 + c)) { off = 2 * i; break; }
                printf(" c%d@%d", c, off);
            }
            printf("\n");
        }
    }
    return 0;
}
