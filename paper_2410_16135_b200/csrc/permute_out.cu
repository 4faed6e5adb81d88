// permute_out.cu — the OUTPUT-channel half of the V:N:M-specific channel permutation:
// the cost matrix of the linear sum assignment that approximates Eq. (8) `eq:admm2` (§4.2 P:211-213,
// "approximately modeled as the traditional linear sum assignment problem"; "V:N:M sparsity allows both
// input and output CP to affect the retained norm").  The Hungarian solve stays with the caller.
//
//   cost[i][g*V + s] = the retained score row i contributes when it replaces the occupant of slot s of V-row
//   stripe g (every other row frozen) and the stripe is re-pruned by S_{V:N:M}: in each column block
//   the 4 columns of largest L1 over the stripe — now with row i at position s — are kept (ties -> smaller
//   column), then row i keeps its 2 largest e among them (ties -> smaller position); summed over the blocks
//   (reading Q23).  With every row in its own slot the costs add up to the retained score.
//
// Every column L1 of a candidate's hypothetical block changes (row i enters every column), so it is recomputed
// per candidate — but without re-summing the stripe: the canonical stride-halving tree (Q3) of each
// column is built once per (stripe, block) in shared memory, and the tree with leaf s replaced by x is
// x + sibling_1 + sibling_2 + ... (log2 V adds along the leaf's path; fp32 addition is commutative, so this is
// bit-identical to re-running the tree) — every keep decision equals the oracle's.  Contributions are summed in
// fp32 in block order (deterministic).
#include <cstdint>
#include <cuda_runtime.h>

#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kCand = 128;  // candidate rows per CTA (one per thread)
constexpr int kSlots = 32;  // slots per CTA (accumulators per thread)

// key order of both decisions: larger value first, then the smaller position
__device__ __forceinline__ bool beats(float va, int pa, float vb, int pb) { return va > vb || (va == vb && pa < pb); }

// P = V rounded up to a power of two (zero rows added exactly); tree levels 0 .. log2(P)-1 stored per column:
// level 0 = the P leaves, level k = P >> k node values; offsets lvl_off(k) = 2P - (2P >> k)
template <int P, int MMAX>
__global__ void __launch_bounds__(kCand) permute_gain_out_kernel(const float* score, int64_t lds, int32_t rows,
                                                                 int32_t cols, int32_t V, int32_t M, int32_t nb,
                                                                 int32_t rows_p, float* cost, int64_t ldc) {
    constexpr int kLv = (P > 1) ? 2 * P - 2 : 1;  // stored tree values per column (levels 0 .. log2 P - 1)
    __shared__ float tree[MMAX][kLv];
    const int vb = blockIdx.y, s0 = blockIdx.z * kSlots;
    const int i = blockIdx.x * kCand + threadIdx.x;  // candidate row
    const bool live = i < rows_p;
    float acc[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.f;
    auto e_at = [&](int r, int c) -> float {  // |score| zero-padded to rows_p x cols_p
        return (r < rows && c < cols) ? fabsf(score[static_cast<int64_t>(r) * lds + c]) : 0.f;
    };
    for (int b = 0; b < nb; ++b) {
        // ---- the stripe's block: leaves, then the stride-halving levels, for every column
        __syncthreads();
        for (int t = threadIdx.x; t < M * P; t += kCand) {
            const int c = t / P, r = t % P;
            tree[c][r] = r < V ? e_at(vb * V + r, b * M + c) : 0.f;
        }
        __syncthreads();
        if constexpr (P > 1) {
            int off_prev = 0, off = P;
            for (int st = P / 2; st >= 2; st >>= 1) {  // level k (st = P >> k) from level k-1
                for (int t = threadIdx.x; t < M * st; t += kCand) {
                    const int c = t / st, r = t % st;
                    tree[c][off + r] = tree[c][off_prev + r] + tree[c][off_prev + r + st];
                }
                __syncthreads();
                off_prev = off;
                off += st;
            }
        }
        // ---- the candidate's own values in this block
        float ei[MMAX];
#pragma unroll
        for (int c = 0; c < MMAX; ++c) ei[c] = (live && c < M) ? e_at(i, b * M + c) : 0.f;
        // ---- every slot of the chunk
#pragma unroll 1
        for (int k = 0; k < kSlots; ++k) {
            const int s = s0 + k;
            if (s >= V) break;
            // L1 of every column with leaf s := e_i (the leaf's path through the stored levels)
            float L[MMAX];
#pragma unroll
            for (int c = 0; c < MMAX; ++c) {
                if (c >= M) break;
                float v = ei[c];
                if constexpr (P > 1) {
                    int off = 0, span = P;  // level k-1 holds `span` nodes starting at `off`
                    for (int st = P / 2; st >= 1; st >>= 1) {
                        const int node = s & (span - 1);  // this leaf's node at level k-1
                        v = v + tree[c][off + (node ^ st)];
                        off += span;
                        span = st;
                    }
                }
                L[c] = v;
            }
            // top-4 columns (ties -> smaller column), as ascending column positions
            int kept[4];
            unsigned used = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int best = -1;
#pragma unroll
                for (int c = 0; c < MMAX; ++c) {
                    if (c >= M) break;
                    if (used & (1u << c)) continue;
                    if (best < 0 || L[c] > L[best]) best = c;
                }
                used |= 1u << best;
                kept[q] = best;
            }
            // ascending order of the kept columns (the block positions of the 2:4 decision)
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
                for (int b2 = 0; b2 < 3 - a2; ++b2)
                    if (kept[b2] > kept[b2 + 1]) {
                        const int t = kept[b2];
                        kept[b2] = kept[b2 + 1];
                        kept[b2 + 1] = t;
                    }
            float e4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float v = 0.f;
#pragma unroll
                for (int c = 0; c < MMAX; ++c)
                    if (c == kept[q]) v = ei[c];
                e4[q] = v;
            }
            // row i's top-2 among the kept 4 (ties -> smaller position), added lower position first
            int first = 0;
#pragma unroll
            for (int q = 1; q < 4; ++q)
                if (beats(e4[q], q, e4[first], first)) first = q;
            int second = first == 0 ? 1 : 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q != first && beats(e4[q], q, e4[second], second)) second = q;
            const int lo = first < second ? first : second, hi = first < second ? second : first;
            acc[k] = acc[k] + e4[lo];
            acc[k] = acc[k] + e4[hi];
        }
    }
    if (!live) return;
#pragma unroll
    for (int k = 0; k < kSlots; ++k)
        if (s0 + k < V) cost[static_cast<int64_t>(i) * ldc + vb * V + s0 + k] = acc[k];
}

template <int P, int MMAX>
int launch_pm(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, cudaStream_t st) {
    const dim3 grid((g.rows_p + kCand - 1) / kCand, g.rows_p / g.V, (g.V + kSlots - 1) / kSlots);
    permute_gain_out_kernel<P, MMAX><<<grid, kCand, 0, st>>>(score, lds, g.rows, g.cols, g.V, g.M, g.nb, g.rows_p, cost, ldc);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

template <int P>
int launch_p(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, cudaStream_t st) {
    if (g.M <= 8) return launch_pm<P, 8>(score, lds, g, cost, ldc, st);
    if (g.M <= 16) return launch_pm<P, 16>(score, lds, g, cost, ldc, st);
    return launch_pm<P, 32>(score, lds, g, cost, ldc, st);
}

}  // namespace

int launch_permute_gain_out(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc,
                            cudaStream_t st) {
    switch (g.V) {
        case 1: return launch_p<1>(score, lds, g, cost, ldc, st);
        case 2: return launch_p<2>(score, lds, g, cost, ldc, st);
        case 4: return launch_p<4>(score, lds, g, cost, ldc, st);
        case 8: return launch_p<8>(score, lds, g, cost, ldc, st);
        case 16: return launch_p<16>(score, lds, g, cost, ldc, st);
        case 32: return launch_p<32>(score, lds, g, cost, ldc, st);
        case 64: return launch_p<64>(score, lds, g, cost, ldc, st);
        case 128: return launch_p<128>(score, lds, g, cost, ldc, st);
        default: return kLaunchUnsupported;
    }
}

}  // namespace vnm
