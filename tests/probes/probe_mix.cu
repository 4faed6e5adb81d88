// TEST-ONLY probe: what HBM throughput the DeiT window-form SpMM's traffic pattern can reach, with no MMA at all.
// The tc3 kernel (csrc/spmm_tc3.cu) writes Y^T [rows][T] bf16 in tiles of 128 rows x NT tokens per CTA (CTA pairs
// share a token tile, row pair rp = cid % n_rp, token tiles cid / n_rp + i * rp_per: the resident-A order) with
// st.global.v4 of 8 rows x 64 B per warp instruction, and reads its X^T half-slab [K][NT/2] per tile.  Here the
// same CTAs, tile order and store instruction pattern run with the MMA and TMEM removed:
//   mode 0  Y^T writes only (the epilogue pattern: 8 warps, 2 per 32-row quadrant, alternate 64-token chunks)
//   mode 1  X^T reads only (2 reader warps per CTA, ld.global.nc.v4 of whole 128-byte lines)
//   mode 2  both at once (the kernel's DRAM traffic mix)
//   mode 3  Y^T writes with each warp writing whole 128-byte lines (4 rows x 128 B per instruction)
// and for comparison a linear copy with the same read:write byte ratio.  Prints GB/s of (reads + writes).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct P {
    uint16_t* Y;
    const uint16_t* X;
    int rows, K, T, NT, n_rp, n_tt, rp_per, mode;
    unsigned* sink;
};

__global__ void __launch_bounds__(384, 1) tile_traffic(P p) {
    const int cid = blockIdx.x / 2, rank = blockIdx.x % 2;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_rt = (p.rows + 127) / 128;
    unsigned acc = 0;
    for (int i = 0;; ++i) {
        const int rp = cid % p.n_rp, tt = cid / p.n_rp + i * p.rp_per;
        if (tt >= p.n_tt) break;
        const int rt = 2 * rp + rank;
        if (warp < 8 && p.mode != 1) {
            if (rt >= n_rt) continue;
            const int qd = warp % 4, half = warp / 4;
            const int nch = (p.NT + 63) / 64;
            for (int c = half; c < nch; c += 2) {
                const int t0 = tt * p.NT + c * 64;
                const int t_end = min(p.T, min(tt * p.NT + p.NT, t0 + 64));
                if (p.mode == 4 || p.mode == 5) {
                    // straight from the TMEM 32x32b layout: lane = row, 16 consecutive tokens (32 B) per lane;
                    // mode 4 one 256-bit store per lane, mode 5 two 128-bit stores
                    const int grow = rt * 128 + 32 * qd + lane;
                    for (int k = 0; k < 4; ++k) {
                        const int tok = t0 + 16 * k;
                        if (grow < p.rows && tok + 16 <= t_end) {
                            uint16_t* dst = p.Y + static_cast<int64_t>(grow) * p.T + tok;
                            if (p.mode == 4) {
                                asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(grow),
                                             "r"(tok), "r"(1), "r"(2), "r"(3), "r"(4), "r"(5), "r"(6) : "memory");
                            } else {
                                reinterpret_cast<uint4*>(dst)[0] = make_uint4(grow, tok, 1, 2);
                                reinterpret_cast<uint4*>(dst)[1] = make_uint4(grow, tok, 3, 4);
                            }
                        }
                    }
                } else if (p.mode == 3) {
                    // 4 rows x 128 B per instruction (8 lanes per row)
                    for (int j = 0; j < 8; ++j) {
                        const int r = 4 * j + lane / 8, tok = t0 + (lane % 8) * 8;
                        const int grow = rt * 128 + 32 * qd + r;
                        if (grow < p.rows && tok + 8 <= t_end) {
                            uint4 v = make_uint4(grow, tok, 1, 2);
                            *reinterpret_cast<uint4*>(p.Y + static_cast<int64_t>(grow) * p.T + tok) = v;
                        }
                    }
                } else {
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const int th = t0 + h2 * 32;
                        for (int j = 0; j < 4; ++j) {
                            const int r = 8 * j + lane / 4, tok = th + (lane % 4) * 8;
                            const int grow = rt * 128 + 32 * qd + r;
                            if (grow < p.rows && tok + 8 <= t_end) {
                                uint4 v = make_uint4(grow, tok, 1, 2);
                                *reinterpret_cast<uint4*>(p.Y + static_cast<int64_t>(grow) * p.T + tok) = v;
                            }
                        }
                    }
                }
            }
        } else if (warp >= 8 && (p.mode == 1 || p.mode == 2)) {
            // X^T half-slab [K][NT/2] of this CTA: rows of NT/2 * 2 bytes; 4 warps, 16 loads of 16 B in flight each
            const int nh = p.NT / 2, x0 = tt * p.NT + nh * rank;
            const int per_row = nh * 2 / 16;  // 16-byte pieces per row
            const int tot = p.K * per_row;
            for (int e0 = (warp - 8) * 32 + lane; e0 < tot; e0 += 128 * 16) {
                uint4 v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int e = e0 + u * 128;
                    const int k = e / per_row, pc = e % per_row;
                    const int tok = x0 + pc * 8;
                    v[u] = make_uint4(0, 0, 0, 0);
                    if (e < tot && tok + 8 <= p.T)
                        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                     : "l"(p.X + static_cast<int64_t>(k) * p.T + tok));
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) acc ^= v[u].x ^ v[u].w;
            }
        }
    }
    if (acc == 0x9e3779b9u) p.sink[0] = acc;
}

__global__ void lin_copy(const uint4* x, uint4* y, size_t nx16, int ratio) {
    // reads nx16 x 16 B, writes ratio times as many bytes (each read chunk stored ratio times, to distinct places)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nx16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = x[i];
        for (int r = 0; r < ratio; ++r) y[r * nx16 + i] = v;
    }
}

int main() {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int T = 50432;
    uint16_t *Y, *X;
    unsigned* sink;
    cudaMalloc(&Y, (size_t)1536 * T * 2);
    cudaMalloc(&X, (size_t)1540 * T * 2);
    cudaMalloc(&sink, 64);
    cudaMemset(Y, 0, (size_t)1536 * T * 2);
    cudaMemset(X, 0, (size_t)1540 * T * 2);
    uint8_t* flush;
    const size_t fl = 512ull << 20;
    cudaMalloc(&flush, fl);
    auto timeit = [&](auto f) {
        float best = 1e9;
        for (int it = 0; it < 8; ++it) {
            cudaMemsetAsync(flush, it, fl);  // L2 flushed (and its write-back forced by a later read below)
            cudaMemsetAsync(flush, it + 1, fl / 2);
            cudaEventRecord(a);
            f();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it >= 2 && ms < best) best = ms;
        }
        return best * 1e3;
    };
    struct Shape { const char* name; int rows, K, NT; };
    for (Shape s : {Shape{"qkv 1152x385 NT224", 1152, 385, 224}, Shape{"fc1 1536x385 NT224", 1536, 385, 224},
                    Shape{"proj 384x385 NT256", 384, 385, 256}, Shape{"fc2 384x1540 NT256", 384, 1540, 256},
                    Shape{"fc1 1536x385 NT448", 1536, 385, 448}}) {
        P p;
        p.Y = Y; p.X = X; p.rows = s.rows; p.K = s.K; p.T = T; p.NT = s.NT; p.sink = sink;
        const int n_rt = (s.rows + 127) / 128;
        p.n_rp = (n_rt + 1) / 2;
        p.n_tt = (T + s.NT - 1) / s.NT;
        const int pairs = 74 / p.n_rp * p.n_rp;
        p.rp_per = pairs / p.n_rp;
        const double yb = (double)s.rows * T * 2, xb = (double)s.K * T * 2;
        for (int mode : {0, 3, 4, 5}) {
            p.mode = mode;
            const double us = timeit([&] { tile_traffic<<<2 * pairs, 384>>>(p); });
            const double by = (mode == 0 || mode >= 3 ? yb : 0) + (mode == 1 ? xb : 0) + (mode == 2 ? xb + yb : 0);
            printf("%-22s mode %d  %8.1f us  %7.0f GB/s  (%.1f MB)\n", s.name, mode, us, by / (us * 1e-6) / 1e9, by / 1e6);
        }
    }
    // linear streams with the same ratios
    for (int ratio : {1, 3, 4}) {
        const size_t nx = (size_t)384 * T * 2 / 16;
        const double us = timeit([&] { lin_copy<<<148 * 8, 256>>>((const uint4*)X, (uint4*)Y, nx, ratio); });
        const double by = (double)nx * 16 * (1 + ratio);
        printf("linear read:write 1:%d %8.1f us  %7.0f GB/s  (%.1f MB)\n", ratio, us, by / (us * 1e-6) / 1e9, by / 1e6);
    }
    {
        const size_t nx = (size_t)1536 * T * 2 / 16 / 4;
        const double us = timeit([&] { lin_copy<<<148 * 8, 256>>>((const uint4*)X, (uint4*)Y, nx, 1); });
        printf("linear copy 1:1 (%zu MB) %8.1f us  %7.0f GB/s\n", nx * 32 >> 20, us, nx * 32.0 / (us * 1e-6) / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
