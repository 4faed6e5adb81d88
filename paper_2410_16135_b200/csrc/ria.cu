// ria.cu — RIA importance scores: the score pre-pass of the V:N:M mask for the TS1 /
// TS3 settings, feeding vnm_prune / vnm_prune_compress through their `score` argument.
//
//   Eq. (1):  RIA_ij = ( |W_ij| / sum_r |W_rj| + |W_ij| / sum_c |W_ic| ) * ( ||X_j||_2 )^a
// Readings (Q16, Q21): the activation norm is indexed by the input channel j; a zero sum
// makes its fraction 0; fp32 arithmetic (the paper fixes no precision).
//
// Three memory-bound passes over W (bf16, row-major [rows][ldw]):
//   1. partial sums: tile = 64 rows x 512 columns, one thread per column pair: column partials over the
//      tile's rows (in-thread, row order) and row partials over the tile's columns (warp shuffles, then the
//      8 warps in order) -> workspace;
//   2. finish: row sums over column tiles and column sums over row tiles, in tile order (deterministic);
//   3. scores: elementwise, 8 weights per thread (16-byte loads, 2 x 16-byte stores).
// vnm_act_norms: ||X_j||_2 over the T tokens of X^T [cols][ldx] (feature-major: one contiguous row per
// channel), one warp per channel.
#include <cstdint>
#include <cuda_runtime.h>

#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kTR = 64;   // rows per tile
constexpr int kTC = 512;  // columns per tile (256 threads x 2)

__device__ __forceinline__ float absbf(uint32_t h) { return __uint_as_float((h & 0x7FFFu) << 16); }

__global__ void __launch_bounds__(256) ria_partial_kernel(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols,
                                                          float* colpart, float* rowpart) {
    const int ct = blockIdx.x, rt = blockIdx.y;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int c0 = ct * kTC + 2 * threadIdx.x;
    __shared__ float sRow[8][kTR];
    float cs0 = 0.f, cs1 = 0.f;
    for (int r = 0; r < kTR; ++r) {
        const int i = rt * kTR + r;
        float e0 = 0.f, e1 = 0.f;
        if (i < rows) {
            const uint16_t* wr = W + static_cast<int64_t>(i) * ldw;
            if (c0 + 1 < cols) {
                const uint32_t w2 = *reinterpret_cast<const uint32_t*>(wr + c0);
                e0 = absbf(w2);
                e1 = absbf(w2 >> 16);
            } else if (c0 < cols) {
                e0 = absbf(wr[c0]);
            }
        }
        cs0 += e0;
        cs1 += e1;
        float rs = e0 + e1;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, s);
        if (lane == 0) sRow[warp][r] = rs;
    }
    if (c0 < cols) colpart[static_cast<int64_t>(rt) * cols + c0] = cs0;
    if (c0 + 1 < cols) colpart[static_cast<int64_t>(rt) * cols + c0 + 1] = cs1;
    __syncthreads();
    if (threadIdx.x < kTR && rt * kTR + threadIdx.x < rows) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += sRow[w][threadIdx.x];
        rowpart[static_cast<int64_t>(ct) * rows + rt * kTR + threadIdx.x] = v;
    }
}

__global__ void ria_finish_kernel(const float* colpart, const float* rowpart, int32_t rows, int32_t cols, int32_t nrt,
                                  int32_t nct, const float* act, float a, float* colsum, float* rowsum, float* actp) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx < cols) {
        float s = 0.f;
        for (int t = 0; t < nrt; ++t) s += colpart[static_cast<int64_t>(t) * cols + idx];
        colsum[idx] = s;
        actp[idx] = act ? powf(act[idx], a) : 1.f;
    } else if (idx < static_cast<int64_t>(cols) + rows) {
        const int64_t i = idx - cols;
        float s = 0.f;
        for (int t = 0; t < nct; ++t) s += rowpart[static_cast<int64_t>(t) * rows + i];
        rowsum[i] = s;
    }
}

// 8 consecutive weights of one row per thread
__global__ void __launch_bounds__(256) ria_score_kernel(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols,
                                                        const float* colsum, const float* rowsum, const float* actp,
                                                        float* score, int64_t lds) {
    const int c8 = (cols + 7) / 8;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(rows) * c8) return;
    const int i = static_cast<int>(idx / c8), j0 = static_cast<int>(idx % c8) * 8;
    const uint16_t* wr = W + static_cast<int64_t>(i) * ldw + j0;
    uint16_t w[8];
    if (j0 + 8 <= cols) {
        const uint4 v = *reinterpret_cast<const uint4*>(wr);
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[2 * k] = static_cast<uint16_t>(u[k]);
            w[2 * k + 1] = static_cast<uint16_t>(u[k] >> 16);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = j0 + k < cols ? wr[k] : 0;
    }
    const float R = rowsum[i];
    float o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int j = j0 + k < cols ? j0 + k : cols - 1;
        const float e = absbf(w[k]), C = colsum[j];
        const float f1 = C > 0.f ? e / C : 0.f, f2 = R > 0.f ? e / R : 0.f;
        o[k] = (f1 + f2) * actp[j];
    }
    float* sr = score + static_cast<int64_t>(i) * lds + j0;
    if (j0 + 8 <= cols) {
        *reinterpret_cast<float4*>(sr) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(sr + 4) = make_float4(o[4], o[5], o[6], o[7]);
    } else {
        for (int k = 0; k < 8 && j0 + k < cols; ++k) sr[k] = o[k];
    }
}

__global__ void act_norms_kernel(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, float* norms) {
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (j >= cols) return;
    const uint16_t* xr = XT + static_cast<int64_t>(j) * ldx;
    float s = 0.f;
    for (int t = lane; t < T; t += 32) {
        const float x = __uint_as_float(static_cast<uint32_t>(xr[t]) << 16);
        s = fmaf(x, x, s);
    }
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) s += __shfl_xor_sync(0xffffffffu, s, k);
    if (lane == 0) norms[j] = sqrtf(s);
}

}  // namespace

size_t ria_workspace_bytes(int32_t rows, int32_t cols) {
    const size_t nrt = (static_cast<size_t>(rows) + kTR - 1) / kTR, nct = (static_cast<size_t>(cols) + kTC - 1) / kTC;
    return (nrt * cols + nct * rows + 2 * static_cast<size_t>(cols) + rows) * 4;
}

int launch_ria(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, const float* act, float a, float* score,
               int64_t lds, void* ws, cudaStream_t st) {
    const int nrt = (rows + kTR - 1) / kTR, nct = (cols + kTC - 1) / kTC;
    float* colpart = static_cast<float*>(ws);
    float* rowpart = colpart + static_cast<int64_t>(nrt) * cols;
    float* colsum = rowpart + static_cast<int64_t>(nct) * rows;
    float* actp = colsum + cols;
    float* rowsum = actp + cols;
    ria_partial_kernel<<<dim3(nct, nrt), 256, 0, st>>>(W, ldw, rows, cols, colpart, rowpart);
    count_launch();
    const int64_t nf = static_cast<int64_t>(cols) + rows;
    ria_finish_kernel<<<static_cast<unsigned>((nf + 255) / 256), 256, 0, st>>>(colpart, rowpart, rows, cols, nrt, nct, act,
                                                                                a, colsum, rowsum, actp);
    count_launch();
    const int64_t n8 = static_cast<int64_t>(rows) * ((cols + 7) / 8);
    ria_score_kernel<<<static_cast<unsigned>((n8 + 255) / 256), 256, 0, st>>>(W, ldw, rows, cols, colsum, rowsum, actp,
                                                                               score, lds);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

int launch_act_norms(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, float* norms, cudaStream_t st) {
    act_norms_kernel<<<(cols + 7) / 8, 256, 0, st>>>(XT, ldx, cols, T, norms);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
