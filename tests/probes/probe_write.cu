// TEST-ONLY probe: HBM write bandwidth for write-only streams (the DeiT SpMM's traffic is ~80% Y^T writes).
// (1) cudaMemsetAsync, (2) st.global.v4 grid-stride, (3) st.global.v4 with .cs (evict-first),
// (4) TMA bulk stores (cp.async.bulk.global.shared::cta) of 16 KB from shared memory, 148 x k CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void st_v4(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(1, 2, 3, 4);
}
__global__ void st_v4_cs(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        __stcs(p + i, make_uint4(1, 2, 3, 4));
}
__global__ void bulk_store(uint8_t* p, size_t bytes, int chunk) {
    extern __shared__ __align__(128) uint8_t s[];
    for (int i = threadIdx.x; i < chunk / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(5, 6, 7, 8);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (size_t off = (size_t)blockIdx.x * chunk; off < bytes; off += (size_t)gridDim.x * chunk) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off),
                         "r"((uint32_t)__cvta_generic_to_shared(s)), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
int main() {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (size_t mb : {155, 310, 1024}) {
        size_t bytes = mb << 20; uint8_t* p; cudaMalloc(&p, bytes);
        auto run = [&](const char* name, auto f) {
            for (int i = 0; i < 3; ++i) f();
            float best = 1e9;
            for (int i = 0; i < 10; ++i) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
            printf("%5zu MB %-28s %8.1f us %7.0f GB/s\n", mb, name, best * 1e3, bytes / (best * 1e-3) / 1e9);
        };
        run("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 0, bytes); });
        for (int g : {148 * 4, 148 * 8, 148 * 16}) {
            char nm[64]; snprintf(nm, 64, "st.v4 grid %d", g);
            run(nm, [&] { st_v4<<<g, 256>>>((uint4*)p, bytes / 16); });
            snprintf(nm, 64, "st.v4.cs grid %d", g);
            run(nm, [&] { st_v4_cs<<<g, 256>>>((uint4*)p, bytes / 16); });
        }
        cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        for (int chunk : {4096, 16384, 65536}) for (int g : {148, 296}) {
            char nm[64]; snprintf(nm, 64, "bulk store %dKB grid %d", chunk / 1024, g);
            run(nm, [&] { bulk_store<<<g, 128, chunk>>>(p, bytes, chunk); });
        }
        cudaFree(p);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
