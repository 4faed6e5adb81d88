// permute.cu — V:N:M-specific channel-permutation gain scores: the cost matrix of the
// linear sum assignment that approximates the input-permutation step of the paper's channel permutation,
// Eq. (7) `eq:admm1` (§4.2; "approximately modeled as the traditional linear sum assignment
// problem").  The Hungarian solve itself stays on the host (sequential).
//
//   cost[j][b*M + s] = sum over V-row stripes of the retained score channel j contributes when it replaces
//   the occupant of slot s of column block b (every other column frozen) and the block is re-pruned by
//   S_{V:N:M}: column L1 top-4 (ties -> smaller position) then per-row top-2 of the kept 4.
//   Contribution = sum of e_j over the rows that keep slot s (reading Q22).
//
// The decisions need no re-pruning per candidate: with the other M-1 columns fixed,
//   * slot s is kept  <=>  (L_j, s) beats the 4th best of the others (always when M = 4);
//   * if kept, the other 3 kept columns are the top 3 of the others, so row r keeps slot s <=> (e_j[r], s)
//     beats the 2nd best of those 3 in that row.
// Both thresholds depend only on (stripe, block, slot, row) and are built once per stripe and shared by every
// candidate j.  Column L1s use the canonical stride-halving tree (Q3), so every decision equals
// the oracle's; sums are fp32 in stripe order (deterministic).
#include <cstdint>
#include <cuda_runtime.h>

#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kBC = 4;     // blocks per CTA
constexpr int kCand = 256; // candidate channels per CTA (one per thread)

// colL1[vb][c] = stride-halving tree of |score| over the V rows of stripe vb (zero outside rows x cols)
template <int V>
__global__ void __launch_bounds__(256) colsum_tree_kernel(const float* score, int64_t lds, int32_t rows, int32_t cols,
                                                           int32_t cols_p, float* colL1) {
    const int c = blockIdx.x * 256 + threadIdx.x, vb = blockIdx.y;
    if (c >= cols_p) return;
    auto e = [&](int r) -> float {
        const int gr = vb * V + r;
        return (gr < rows && c < cols) ? fabsf(score[static_cast<int64_t>(gr) * lds + c]) : 0.f;
    };
    if constexpr (V == 1) {
        colL1[static_cast<int64_t>(vb) * cols_p + c] = e(0);
        return;
    }
    float s[V / 2 > 0 ? V / 2 : 1];
#pragma unroll
    for (int i = 0; i < V / 2; ++i) s[i] = e(i) + e(i + V / 2);
#pragma unroll
    for (int st = V / 4; st >= 1; st >>= 1)
#pragma unroll
        for (int i = 0; i < st; ++i) s[i] = s[i] + s[i + st];
    colL1[static_cast<int64_t>(vb) * cols_p + c] = s[0];
}

// key order of both decisions: larger value first, then the smaller block position
__device__ __forceinline__ bool beats(float va, int pa, float vb, int pb) { return va > vb || (va == vb && pa < pb); }

// MMAX: block width bound (8, 16, 32); KBC: column blocks per CTA (4 for M <= 8, else 1 to bound shared memory)
template <int V, int MMAX, int KBC>
__global__ void __launch_bounds__(256) permute_gain_kernel(const float* score, int64_t lds, int32_t rows, int32_t cols,
                                                           int32_t M, int32_t cols_p, int32_t nb, int32_t nvb,
                                                           const float* colL1, float* cost, int64_t ldc) {
    constexpr int kBC = KBC;
    __shared__ float sL4[kBC][MMAX];             // 4th-best L1 of the others (per block, slot)
    __shared__ int sC4[kBC][MMAX];               // ... its position (-1: M = 4, always kept)
    __shared__ float sThrE[kBC][MMAX][V];        // 2nd-best e of the top-3 others, per row
    __shared__ int8_t sThrC[kBC][MMAX][V];       // ... its position
    __shared__ int8_t sTop3[kBC][MMAX][3];       // the 3 best others (positions)
    const int b0 = blockIdx.x * kBC, j = blockIdx.y * kCand + threadIdx.x;
    const int nbl = min(kBC, nb - b0);
    float acc[kBC][MMAX];
#pragma unroll
    for (int b = 0; b < kBC; ++b)
#pragma unroll
        for (int s = 0; s < MMAX; ++s) acc[b][s] = 0.f;

    for (int vb = 0; vb < nvb; ++vb) {
        const float* Lrow = colL1 + static_cast<int64_t>(vb) * cols_p;
        // ---- per (block, slot): rank the other M-1 columns by (L1 desc, position asc)
        __syncthreads();
        if (threadIdx.x < kBC * MMAX) {
            const int b = threadIdx.x / MMAX, s = threadIdx.x % MMAX;
            if (b < nbl && s < M) {
                float tv[4] = {-1.f, -1.f, -1.f, -1.f};
                int ti[4] = {-1, -1, -1, -1};
                for (int c = 0; c < M; ++c) {  // running top-4 of the others
                    if (c == s) continue;
                    const float L = Lrow[(b0 + b) * M + c];
                    int k = 4;
                    while (k > 0 && beats(L, c, tv[k - 1], ti[k - 1] < 0 ? 64 : ti[k - 1])) --k;
                    if (k < 4) {
                        for (int q = 3; q > k; --q) { tv[q] = tv[q - 1]; ti[q] = ti[q - 1]; }
                        tv[k] = L;
                        ti[k] = c;
                    }
                }
                sL4[b][s] = tv[3];
                sC4[b][s] = ti[3];
                for (int q = 0; q < 3; ++q) sTop3[b][s][q] = static_cast<int8_t>(ti[q]);
            }
        }
        __syncthreads();
        // ---- per (block, slot, row): the 2nd best of the top-3 others by (e desc, position asc)
        for (int idx = threadIdx.x; idx < kBC * MMAX * V; idx += 256) {
            const int b = idx / (MMAX * V), s = (idx / V) % MMAX, r = idx % V;
            if (b >= nbl || s >= M) continue;
            const int gr = vb * V + r;
            int ti[3];
            float ev[3];
            for (int q = 0; q < 3; ++q) {
                ti[q] = sTop3[b][s][q];
                const int gc = (b0 + b) * M + ti[q];
                ev[q] = (gr < rows && gc < cols) ? fabsf(score[static_cast<int64_t>(gr) * lds + gc]) : 0.f;
            }
            int o0 = 0, o1 = 1, o2 = 2;
            if (beats(ev[o1], ti[o1], ev[o0], ti[o0])) { int t = o0; o0 = o1; o1 = t; }
            if (beats(ev[o2], ti[o2], ev[o1], ti[o1])) { int t = o1; o1 = o2; o2 = t; }
            if (beats(ev[o1], ti[o1], ev[o0], ti[o0])) { int t = o0; o0 = o1; o1 = t; }
            sThrE[b][s][r] = ev[o1];
            sThrC[b][s][r] = static_cast<int8_t>(ti[o1]);
        }
        __syncthreads();
        if (j >= cols_p) continue;
        // ---- candidate j: its L1 and its values in this stripe
        const float Lj = Lrow[j];
        float ej[V];
#pragma unroll
        for (int r = 0; r < V; ++r) {
            const int gr = vb * V + r;
            ej[r] = (gr < rows && j < cols) ? fabsf(score[static_cast<int64_t>(gr) * lds + j]) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < kBC; ++b)
#pragma unroll
            for (int s = 0; s < MMAX; ++s) {
                const int c4 = sC4[b][s];
                // slot s must exist and be kept in this stripe (compile-time b, s: acc stays in registers)
                if (b < nbl && s < M && (c4 < 0 || beats(Lj, s, sL4[b][s], c4))) {
                    float part = 0.f;
#pragma unroll
                    for (int r = 0; r < V; ++r)  // fully unrolled: ej[] stays in registers
                        if (beats(ej[r], s, sThrE[b][s][r], sThrC[b][s][r])) part += ej[r];
                    acc[b][s] += part;
                }
            }
    }
    if (j >= cols_p) return;
#pragma unroll
    for (int b = 0; b < kBC; ++b)
#pragma unroll
        for (int s = 0; s < MMAX; ++s)
            if (b < nbl && s < M) cost[static_cast<int64_t>(j) * ldc + (b0 + b) * M + s] = acc[b][s];
}

template <int V, int MMAX, int KBC>
int launch_vm(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, float* colL1,
              cudaStream_t st) {
    const int nvb = g.rows_p / V;
    colsum_tree_kernel<V><<<dim3((g.cols_p + 255) / 256, nvb), 256, 0, st>>>(score, lds, g.rows, g.cols, g.cols_p, colL1);
    count_launch();
    permute_gain_kernel<V, MMAX, KBC><<<dim3((g.nb + KBC - 1) / KBC, (g.cols_p + kCand - 1) / kCand), 256, 0, st>>>(
        score, lds, g.rows, g.cols, g.M, g.cols_p, g.nb, nvb, colL1, cost, ldc);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

template <int V>
int launch_v(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, float* colL1,
             cudaStream_t st) {
    if (g.M <= 8) return launch_vm<V, 8, (V <= 64 ? kBC : 1)>(score, lds, g, cost, ldc, colL1, st);
    if (g.M <= 16) return launch_vm<V, 16, 1>(score, lds, g, cost, ldc, colL1, st);
    return launch_vm<V, 32, 1>(score, lds, g, cost, ldc, colL1, st);
}

}  // namespace

size_t permute_gain_workspace_bytes(const vnm_geom& g) {
    return static_cast<size_t>(g.rows_p / (g.V > 0 ? g.V : 1)) * g.cols_p * 4;
}

int launch_permute_gain(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, void* ws,
                        cudaStream_t st) {
    float* colL1 = static_cast<float*>(ws);
    switch (g.V) {
        case 1: return launch_v<1>(score, lds, g, cost, ldc, colL1, st);
        case 2: return launch_v<2>(score, lds, g, cost, ldc, colL1, st);
        case 4: return launch_v<4>(score, lds, g, cost, ldc, colL1, st);
        case 8: return launch_v<8>(score, lds, g, cost, ldc, colL1, st);
        case 16: return launch_v<16>(score, lds, g, cost, ldc, colL1, st);
        case 32: return launch_v<32>(score, lds, g, cost, ldc, colL1, st);
        case 64: return launch_v<64>(score, lds, g, cost, ldc, colL1, st);
        case 128: return launch_v<128>(score, lds, g, cost, ldc, colL1, st);
        default: return kLaunchUnsupported;
    }
}

}  // namespace vnm
