// prune2.cu — the V:N:M mask + compression pass, instruction-lean form for
// 32 <= V <= 128 and M <= 8 (the paper's configurations: V in {32, 64, 128}; M <= 8 in
// every BJ config).  Same outputs, byte for byte, as prune.cu, which stays for the other shapes and for
// vnm_compress from a given mask.
//
// S_{V:N:M} (§3 "Pruning of V:N:M sparsity"): importance e = |score| (ABS: |W|);
// per V x M block keep the 4 columns of largest column L1; per row keep the 2 largest e of those 4
// (P:84); then the compressed form A_n / A_i1 / A_i2 (App. A).
//
// prune.cu is instruction-bound (profiles/r01_ncu_prune_*: ~36 instructions per weight, 75% SM
// throughput, 21% of HBM), so this kernel is organised around the instruction count:
//   load     a tile = V rows x 32 column blocks, ONE 2D TMA (zero fill outside rows x cols = the implicit
//            padding of P:107-108) — no per-thread address arithmetic; persistent CTAs walk the tiles with
//            the next tile's TMA in flight (double buffer) while the current one is processed;
//   columns  2 lanes per column pair (two bf16 in one 32-bit word), lane q owns rows q, q+2, ...; the
//            canonical stride-halving tree (Q3) runs in registers for strides V/2 .. 2 and ends
//            with one xor-shuffle (stride 1) — the oracle's additions in the oracle's order;
//   top-4    one lane per block (ties -> smaller column); the window-form encoding of every kept
//            column pair (byte-permute selectors, tc_form.cuh) is a 64-entry table built once per CTA;
//   rows     lane = block, warps over rows: 4 shared loads at per-lane fixed offsets, the top-2 by a
//            branch-free max/min network on keys (e, 3 - pos); pad blocks need no special case (their
//            columns are TMA zero fill, which prunes to exactly the pad encoding: values 0, nibble 0x4);
//   store    A_n, window-form values and A_i2 words are staged in shared memory and leave as one TMA tensor
//            store each per tile (no per-row address arithmetic; the store clips at the tensor edge);
//            A_i2 nibbles are packed 8 per word by byte permutes;
//   A_i1     the columns that carry nonzeros (OR over the block's rows), completed with the lowest free
//            columns (Q19); when that differs from the kept 4 (rare) the nibbles are re-based.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tc_form.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

// NW warps per CTA: 8 (3 CTAs per SM, large weights) or 16 (one tile per CTA for small weights: the per-tile
// latency halves, the row pass being the longest phase)
constexpr int kCB = 32;  // column blocks per tile (one per lane in the row pass) for M <= 8
// 8 < M <= 16: 16 blocks per tile (tile columns 16M <= 256, one TMA box; the row pass runs 2 rows per warp step)
__host__ __device__ constexpr int kcb_of(int M) { return M > 8 ? 16 : 32; }

struct Prune2Args {
    uint32_t* mask_out;  // may be null
    uint8_t* col_idx;
    uint32_t* meta;      // A_i2 (row padding words only; the rest leaves by TMA)
    uint32_t* meta_tc;   // optional window form, see tc_form.cuh (values_tc leaves by TMA)
    int32_t has_values, has_tc, n_stage_tc, n_mma;
    int32_t M, rows_p, nb, nb_pad, ld_mask, ld_meta;
    int32_t has_score;
    int32_t trace;  // VNM_PRUNE_TRACE: %globaltimer at the phase boundaries of CTA 0's first tile
};

__device__ unsigned long long g_prune2_t[8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PTRACE(k)                                                                \
    if (a.trace) {  /* uniform: no timer read (or its predicated issue) when off */ \
        if (blockIdx.x == 0 && it == 0 && threadIdx.x == 0) g_prune2_t[k] = gtime(); \
    }

__device__ __forceinline__ float bf16_to_f32_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_to_f32_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// byte-permute selector placing one window-form slot: 1 -> v_lo (bytes 0,1 of vals), 2 -> v_hi (2,3),
// 0 -> zero (bytes 4,5 of the zero second operand)
__device__ __forceinline__ uint32_t slot_sel(uint16_t v) { return v == 1 ? 0x10u : (v == 2 ? 0x32u : 0x54u); }

struct Maps {
    CUtensorMap w, s;          // loads: W [rows][cols] bf16, score [rows][cols] fp32
    CUtensorMap val, tcv, met; // stores: A_n [rows_p][ld_val], values_tc [rows_w][ld_tc], A_i2 [rows_p][ld_meta]
};

// Several weights of the same (V, M) in one launch (vnm_prune_compress_batched): tiles are numbered across the
// problems (tile0 = prefix sums of the per-problem tile counts) and each tile reads its own problem's maps and
// arguments; the shared-memory layout is sized for the largest problem.
constexpr int kMaxBatch = 8;
struct Batch {
    int32_t n;
    int32_t tile0[kMaxBatch + 1];
    int32_t any_score, any_mask, any_tc;
    Maps tm[kMaxBatch];
    Prune2Args a[kMaxBatch];
};

// MINB: CTAs per SM the register budget is sized for (8-warp CTAs: 3, or 4 when no window form is written —
// the window-form staging is then not allocated and 4 CTAs fit in shared memory)
// LEAN = 1: no score, no mask, no tensor-core form anywhere in the batch (the decode / deployment case); LEAN = 2: no
// score, no mask, the tensor-core form as the batch asks (the prefill case): those paths
// compile out of the per-row loop (fewer branches and parameter loads per weight; the kernel is issue-bound)
template <int V, int M, int NW, int MINB, int LEAN>
__global__ void __launch_bounds__(32 * NW, MINB) prune2_kernel(const __grid_constant__ Batch B) {
    constexpr int kWarps = NW, kThreads = 32 * NW;
    constexpr int kCB = kcb_of(M);  // column blocks per tile (shadows the namespace constant)
    constexpr int RI = 32 / kCB;    // rows per warp step in the row pass (lane = block + kCB * row)
    constexpr int TC = kCB * M;     // tile columns (<= 256)
    // window-16 form (8 < M < 16, M % 4 != 0; include/vnm.h): 8 values per block, 4 group nibbles (u16)
    constexpr bool kW16 = M > 8 && M % 4 != 0;
    // natural 2:4 form at M = 16 (include/vnm.h): a block is 4 whole groups, 2 values each (= the window-16 group
    // encoding of a block that fills its window); a 16-block tile is 64 groups = 8 MMAs = 2 stages
    constexpr bool kN16 = M == 16;
    constexpr int kTcvWords = (kW16 || kN16) ? 4 : 2;  // 32-bit words of tensor-core values per block
    constexpr int P = TC / 2;    // words per W row in shared memory
    constexpr int RPW = V / kWarps;
    constexpr uint32_t kWBytes = V * TC * 2, kSBytes = V * TC * 4;
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    // two tile buffers (W [+ score]) for the TMA double buffer, the output staging, then the scratch
    const uint32_t buf_bytes = kWBytes + (B.any_score ? kSBytes : 0);
    uint32_t* sVal = reinterpret_cast<uint32_t*>(smem + 2 * buf_bytes);    // [V][kCB] A_n pairs
    uint2* sTcv = reinterpret_cast<uint2*>(sVal + V * kCB);                 // [V][kCB] window values (M > 4; any_tc)
    uint32_t* sMet = reinterpret_cast<uint32_t*>(sTcv) + (B.any_tc ? V * kCB * kTcvWords : 0);  // [V][4] A_i2 words
    float* sL = reinterpret_cast<float*>(sMet + V * 4);                     // [TC] column L1
    uint32_t* sKp = reinterpret_cast<uint32_t*>(sL + 256);                  // [kCB] kept columns, 8 bits each
    uint32_t* sUni = sKp + kCB;                                             // [kCB] kept positions carrying bits
    uint2* sTab = reinterpret_cast<uint2*>(sUni + kCB);                     // [8 * 8] window-form encodings
    uint32_t* sBits = reinterpret_cast<uint32_t*>(sTab + 64);               // [V][kCB] (mask_out)
    uint8_t* sNib = reinterpret_cast<uint8_t*>(sBits + (B.any_mask ? V * kCB : 0));  // [V][kCB] A_i2 nibbles
    uint8_t* sTcn = sNib + V * kCB;  // [V][kCB] window nibbles (u16 for the window-16 form)
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int3 sInfo[2];  // (problem, column tile, row tile) of the tile in each buffer, set by its issuer

    const int ntiles = B.tile0[B.n];
    auto problem = [&](int tile) {
        int p = 0;
        while (p + 1 < B.n && tile >= B.tile0[p + 1]) ++p;
        return p;
    };
    // one thread decodes the tile (problem lookup, 2-D split) for everyone: it writes sInfo[bi] before its
    // arrive on bar[bi], and the other threads read it after their wait on bar[bi] (release / acquire)
    auto issue = [&](int tile, int bi) {
        const int p = problem(tile), lt = tile - B.tile0[p];
        const Prune2Args& ap = B.a[p];
        const int ntx = (ap.nb_pad + kCB - 1) / kCB, bx = lt % ntx, by = lt / ntx;
        sInfo[bi] = make_int3(p, bx, by);
        uint8_t* dst = smem + bi * buf_bytes;
        mbar_arrive_expect_tx(&bar[bi], kWBytes + (ap.has_score ? kSBytes : 0));
        tma_load_2d(dst, &B.tm[p].w, bx * kCB * M, by * V, &bar[bi]);
        if (ap.has_score) tma_load_2d(dst + kWBytes, &B.tm[p].s, bx * kCB * M, by * V, &bar[bi]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
    }
    if (threadIdx.x < kCB) sUni[threadIdx.x] = 0u;
    if (M > 4 && threadIdx.x < 64) {
        // window-form encoding of the kept pair (cl, ch) = (t / 8, t % 8), cl < ch (tc_form.cuh): byte-permute
        // selectors placing v_lo / v_hi / 0 in the 4 slots, and the two group nibbles
        const int cl = threadIdx.x / 8, ch = threadIdx.x % 8;
        const TcBlock t = cl < ch ? tc_encode_block(cl, ch, 1, 2) : tc_encode_block(0, 1, 1, 2);
        uint2 e;
        e.x = (slot_sel(t.val[0]) | (slot_sel(t.val[1]) << 8)) | ((slot_sel(t.val[2]) | (slot_sel(t.val[3]) << 8)) << 16);
        e.y = t.nibs;
        sTab[threadIdx.x] = e;
    }
    __syncthreads();

    int it = 0;
    {
        const Prune2Args& a = B.a[0];
        PTRACE(0)
    }
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int bi = it & 1;
        // prefetch the next tile into the other buffer (its previous contents were consumed last iteration)
        if (threadIdx.x == 0 && tile + static_cast<int>(gridDim.x) < ntiles) issue(tile + gridDim.x, bi ^ 1);
        mbar_wait(&bar[bi], (it >> 1) & 1);
        const int3 info = sInfo[bi];
        const int p = info.x, bx = info.y, by = info.z;
        const Prune2Args& a = B.a[p];
        const Maps& tm = B.tm[p];
        const bool has_score = LEAN == 0 && a.has_score, tc = (M <= 8 || kW16 || kN16) && LEAN != 1 && a.has_tc;
        uint32_t* const mask_out = LEAN ? nullptr : a.mask_out;
        const int b0 = bx * kCB, r0 = by * V;
        PTRACE(1)
        const uint32_t* sW = reinterpret_cast<const uint32_t*>(smem + bi * buf_bytes);
        const float* sS = reinterpret_cast<const float*>(smem + bi * buf_bytes + kWBytes);

        // ---- column L1: lane q = lane & 1 owns rows q + 2i; strides V/2 .. 2 in registers, 1 by shuffle
#pragma unroll 1
        for (int cp = warp * 16 + (lane >> 1); cp < (P + 16 * NW - 1) / (16 * NW) * (16 * NW); cp += 16 * NW) {
            const int q = lane & 1;
            float lo = 0.f, hi = 0.f;
            if (cp < P) {
                float s0[V / 4], s1[V / 4];  // level 1 (row stride V/2) folded into the loads
                if (has_score) {
#pragma unroll
                    for (int i = 0; i < V / 4; ++i) {
                        const float2 x = *reinterpret_cast<const float2*>(sS + (q + 2 * i) * TC + 2 * cp);
                        const float2 y = *reinterpret_cast<const float2*>(sS + (q + 2 * i + V / 2) * TC + 2 * cp);
                        s0[i] = fabsf(x.x) + fabsf(y.x);
                        s1[i] = fabsf(x.y) + fabsf(y.y);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < V / 4; ++i) {
                        const uint32_t x = sW[(q + 2 * i) * P + cp], y = sW[(q + 2 * i + V / 2) * P + cp];
                        s0[i] = fabsf(bf16_to_f32_lo(x)) + fabsf(bf16_to_f32_lo(y));
                        s1[i] = fabsf(bf16_to_f32_hi(x)) + fabsf(bf16_to_f32_hi(y));
                    }
                }
#pragma unroll
                for (int st = V / 8; st >= 1; st >>= 1)  // row strides V/4 .. 2
#pragma unroll
                    for (int i = 0; i < st; ++i) {
                        s0[i] = s0[i] + s0[i + st];
                        s1[i] = s1[i] + s1[i + st];
                    }
                lo = s0[0];
                hi = s1[0];
            }
            lo = lo + __shfl_xor_sync(0xffffffffu, lo, 1);  // row stride 1 (rows 0 and 1)
            hi = hi + __shfl_xor_sync(0xffffffffu, hi, 1);
            if (q == 0 && cp < P) {
                sL[2 * cp] = lo;
                sL[2 * cp + 1] = hi;
            }
        }
        // the previous tile's TMA stores must have read the staging buffers before they are rewritten
        if (threadIdx.x == 0) bulk_wait_read0();
        __syncthreads();
        PTRACE(2)

        // ---- top-4 columns per block (lane = block; ties -> smaller column)
        if (warp == 0 && lane < kCB) {
            const int b = lane;
            float tv[4] = {-1.f, -1.f, -1.f, -1.f};
            int ti[4] = {0, 1, 2, 3};
#pragma unroll
            for (int c = 0; c < M; ++c) {
                const float L = sL[b * M + c];
                if (L > tv[3]) {
                    if (L > tv[2]) {
                        tv[3] = tv[2]; ti[3] = ti[2];
                        if (L > tv[1]) {
                            tv[2] = tv[1]; ti[2] = ti[1];
                            if (L > tv[0]) { tv[1] = tv[0]; ti[1] = ti[0]; tv[0] = L; ti[0] = c; }
                            else { tv[1] = L; ti[1] = c; }
                        } else { tv[2] = L; ti[2] = c; }
                    } else { tv[3] = L; ti[3] = c; }
                }
            }
            uint32_t km = (1u << ti[0]) | (1u << ti[1]) | (1u << ti[2]) | (1u << ti[3]);
            int kc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { kc[q] = __ffs(km) - 1; km &= km - 1; }
            sKp[b] = static_cast<uint32_t>(kc[0]) | (kc[1] << 8) | (kc[2] << 16) | (kc[3] << 24);
        }
        __syncthreads();
        PTRACE(3)

        // ---- rows: lane = block b, this warp's rows r = warp + 8 i.  Pad blocks (b >= nb) hold zero fill
        // and come out as the pad encoding by themselves (kept {0,1,2,3}, rows keep positions 0,1, values 0).
        // (kCB = 16, M > 8: lanes 16-31 take the next row of the warp's pair: r = warp + kWarps (2 i + lane / 16))
        const int b = lane % kCB, rs = lane / kCB;
        const uint32_t kp = sKp[b];
        const int k0 = kp & 0xFF, k1 = (kp >> 8) & 0xFF, k2 = (kp >> 16) & 0xFF, k3 = kp >> 24;
        const uint16_t* wcol = reinterpret_cast<const uint16_t*>(sW) + b * M + (warp + kWarps * rs) * TC;
        const float* scol = sS + b * M + (warp + kWarps * rs) * TC;
        uint32_t upos = 0;  // kept positions chosen by some row
#pragma unroll
        for (int i = 0; i < RPW / RI; ++i) {
            const int r = warp + kWarps * (RI * i + rs);
            const uint16_t* wr = wcol + kWarps * RI * i * TC;
            const uint32_t w0 = wr[k0], w1 = wr[k1], w2 = wr[k2], w3 = wr[k3];
            uint32_t t1, t2;
            if (has_score) {
                const float* sr = scol + kWarps * RI * i * TC;
                const unsigned long long q0 = (static_cast<unsigned long long>(__float_as_uint(fabsf(sr[k0]))) << 2) | 3u;
                const unsigned long long q1 = (static_cast<unsigned long long>(__float_as_uint(fabsf(sr[k1]))) << 2) | 2u;
                const unsigned long long q2 = (static_cast<unsigned long long>(__float_as_uint(fabsf(sr[k2]))) << 2) | 1u;
                const unsigned long long q3 = (static_cast<unsigned long long>(__float_as_uint(fabsf(sr[k3]))) << 2);
                const unsigned long long m01 = q0 > q1 ? q0 : q1, n01 = q0 > q1 ? q1 : q0;
                const unsigned long long m23 = q2 > q3 ? q2 : q3, n23 = q2 > q3 ? q3 : q2;
                const unsigned long long u1 = m01 > m23 ? m01 : m23;
                const unsigned long long lo2 = m01 > m23 ? m23 : m01, hi2 = n01 > n23 ? n01 : n23;
                t1 = static_cast<uint32_t>(u1);
                t2 = static_cast<uint32_t>(lo2 > hi2 ? lo2 : hi2);
            } else {
                // key = |w| (the bf16 shifted up by 17 drops the sign bit) above the position tie-break
                const uint32_t q0 = w0 * 0x20000u + 3u, q1 = w1 * 0x20000u + 2u;
                const uint32_t q2 = w2 * 0x20000u + 1u, q3 = w3 * 0x20000u;
                const uint32_t m01 = max(q0, q1), n01 = min(q0, q1), m23 = max(q2, q3), n23 = min(q2, q3);
                t1 = max(m01, m23);
                t2 = max(min(m01, m23), max(n01, n23));
            }
            // positions (0..3 among the kept 4) of the two largest: 3 - (key & 3)
            const uint32_t f = 3u - (t1 & 3u), sc = 3u - (t2 & 3u);
            const uint32_t plo = min(f, sc), phi = max(f, sc);
            // v_lo | v_hi << 16 by one byte permute of the 4 kept values
            const uint32_t p01 = __byte_perm(w0, w1, 0x5410), p23 = __byte_perm(w2, w3, 0x5410);
            const uint32_t vals = __byte_perm(p01, p23, (plo * 0x22u + 0x10u) | ((phi * 0x22u + 0x10u) << 8));
            upos |= (1u << plo) | (1u << phi);
            sVal[r * kCB + b] = vals;
            sNib[r * kCB + b] = static_cast<uint8_t>(plo | (phi << 2));
            if (kN16 && tc) {
                // natural 2:4 form, M = 16: groups 4b .. 4b+3 of the row -> values 8b .. 8b+7 of the tile's row
                const int cl = static_cast<int>(__byte_perm(kp, 0u, 0x4440u | plo));
                const int ch = static_cast<int>(__byte_perm(kp, 0u, 0x4440u | phi));
                const TcBlock16 t = tc_encode_block16(cl, ch, static_cast<uint16_t>(vals & 0xFFFFu),
                                                      static_cast<uint16_t>(vals >> 16));
                *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sTcv) + r * (8 * kCB) + 8 * b) =
                    make_uint4(t.val[0] | (static_cast<uint32_t>(t.val[1]) << 16), t.val[2] | (static_cast<uint32_t>(t.val[3]) << 16),
                               t.val[4] | (static_cast<uint32_t>(t.val[5]) << 16), t.val[6] | (static_cast<uint32_t>(t.val[7]) << 16));
                reinterpret_cast<uint16_t*>(sTcn)[r * kCB + b] = static_cast<uint16_t>(t.nibs);
            } else if (kW16 && tc) {
                // window-16 form: half h of block b -> MMA 2 (b/4) + h, slots 4 (b%4) .. +3 of its 16 (the tile's
                // values_tc row is [8 MMAs][16 values]); the 4 group nibbles as one u16
                const int cl = static_cast<int>(__byte_perm(kp, 0u, 0x4440u | plo));
                const int ch = static_cast<int>(__byte_perm(kp, 0u, 0x4440u | phi));
                const TcBlock16 t = tc_encode_block16(cl, ch, static_cast<uint16_t>(vals & 0xFFFFu),
                                                      static_cast<uint16_t>(vals >> 16));
                uint16_t* dst = reinterpret_cast<uint16_t*>(sTcv) + r * (8 * kCB) + 32 * (b / 4) + 4 * (b % 4);
                *reinterpret_cast<uint2*>(dst) = make_uint2(t.val[0] | (static_cast<uint32_t>(t.val[1]) << 16),
                                                            t.val[2] | (static_cast<uint32_t>(t.val[3]) << 16));
                *reinterpret_cast<uint2*>(dst + 16) = make_uint2(t.val[4] | (static_cast<uint32_t>(t.val[5]) << 16),
                                                                 t.val[6] | (static_cast<uint32_t>(t.val[7]) << 16));
                reinterpret_cast<uint16_t*>(sTcn)[r * kCB + b] = static_cast<uint16_t>(t.nibs);
            } else if (M > 4 && M <= 8 && tc) {
                const uint32_t cl = __byte_perm(kp, 0u, 0x4440u | plo), ch = __byte_perm(kp, 0u, 0x4440u | phi);
                const uint2 e = sTab[cl * 8 + ch];
                uint2 pk;
                pk.x = __byte_perm(vals, 0u, e.x & 0xFFFFu);
                pk.y = __byte_perm(vals, 0u, e.x >> 16);
                sTcv[r * kCB + b] = pk;
                sTcn[r * kCB + b] = static_cast<uint8_t>(e.y);
            }
            if (mask_out) {  // mask bits of pad blocks (columns >= cols_p) stay 0
                const uint32_t cl = __byte_perm(kp, 0u, 0x4440u | plo), ch = __byte_perm(kp, 0u, 0x4440u | phi);
                sBits[r * kCB + b] = b0 + b < a.nb ? (1u << cl) | (1u << ch) : 0u;
            }
        }
        atomicOr(&sUni[b], upos);
        __syncthreads();
        PTRACE(4)

        // ---- A_i1 = the columns carrying bits, completed with the lowest free columns (Q19)
        const uint32_t up = sUni[b];
        const uint32_t kept = (1u << k0) | (1u << k1) | (1u << k2) | (1u << k3);
        uint32_t ci = ((up & 1u) << k0) | (((up >> 1) & 1u) << k1) | (((up >> 2) & 1u) << k2) | (((up >> 3) & 1u) << k3);
        constexpr uint32_t colmask = (1u << M) - 1u;
        for (int need = 4 - __popc(ci); need > 0; --need) ci |= 1u << (__ffs(~ci & colmask) - 1);
        if (a.has_values && warp == 0 && lane < kCB && b0 + b < a.nb_pad) {
            uint32_t word = 0, m = ci;
#pragma unroll
            for (int q = 0; q < 4; ++q) { word |= static_cast<uint32_t>(__ffs(m) - 1) << (8 * q); m &= m - 1; }
            reinterpret_cast<uint32_t*>(a.col_idx)[static_cast<int64_t>(by) * a.nb_pad + b0 + b] = word;
        }
        // a kept column carries no nonzero (tiny V, degenerate rows): the nibbles index A_i1 -> re-base them
        if (__syncthreads_or(ci != kept)) {
            if (ci != kept) {
                const int kc[4] = {k0, k1, k2, k3};
                int pos[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) pos[q] = __popc(ci & ((1u << kc[q]) - 1u));
                for (int i = 0; i < RPW / RI; ++i) {
                    const int r = warp + kWarps * (RI * i + rs);
                    const uint32_t n = sNib[r * kCB + b];
                    const int lo = n & 3, hi = n >> 2;
                    const int plo = lo == 0 ? pos[0] : (lo == 1 ? pos[1] : (lo == 2 ? pos[2] : pos[3]));
                    const int phi = hi == 0 ? pos[0] : (hi == 1 ? pos[1] : (hi == 2 ? pos[2] : pos[3]));
                    sNib[r * kCB + b] = static_cast<uint8_t>(plo | (phi << 2));
                }
            }
            __syncthreads();
        }
        if (threadIdx.x < kCB) sUni[threadIdx.x] = 0u;  // next tile (every read of it is above)

        // ---- A_i2 words: 8 nibble bytes -> one word (byte permutes)
        constexpr int kMW = kCB / 8;  // A_i2 words per row of the tile
        for (int t = threadIdx.x; t < V * kMW; t += kThreads) {
            const uint2 x = *reinterpret_cast<const uint2*>(sNib + (t / kMW) * kCB + 8 * (t % kMW));
            const uint32_t lo = x.x | (x.x >> 4), hi = x.y | (x.y >> 4);
            const uint32_t word = __byte_perm(lo, hi, 0x6420);
            if constexpr (kCB == 32) {
                sMet[t] = word;
            } else if (a.has_values && b0 / 8 + t % kMW < a.nb_pad / 8) {  // 16-block tiles: straight to A_i2
                a.meta[static_cast<int64_t>(r0 + t / kMW) * a.ld_meta + b0 / 8 + t % kMW] = word;
            }
        }
        const int cbv = min(kCB, a.nb_pad - b0);  // blocks of this tile inside nb_pad (a multiple of 8)
        if (a.has_values && b0 + cbv == a.nb_pad) {  // last column tile: row padding words (Q20)
            const int pw0 = a.nb_pad / 8, npw = a.ld_meta - pw0;
            for (int i = threadIdx.x; i < V * npw; i += kThreads)
                a.meta[static_cast<int64_t>(r0 + i / npw) * a.ld_meta + pw0 + i % npw] = 0x44444444u;
        }
        if (tc) {
            // meta_tc (include/vnm.h): lane L of a 128-row tile holds rows (L%8) + 16(L/16) and +8; h = (L/8)%2
            // selects K-groups 4h..4h+3 of the MMA.  One 16-byte store per (lane, stage) of this tile; MMA
            // slots past the last real MMA get the filler 0x44444444 (as vnm_pack_tc writes).
            const uint8_t* src = M == 4 ? sNib : sTcn;
            const uint16_t* src16 = reinterpret_cast<const uint16_t*>(sTcn);
            constexpr int bpm = M == 4 ? 8 : ((kW16 || kN16) ? 2 : 4);  // blocks per MMA (window-16: 4 per 2 MMAs)
            constexpr int nst = kCB / (4 * bpm);    // stages per tile (1 or 2)
            const int st0 = b0 / (4 * bpm);
            const int t128 = r0 / 128, l0 = r0 % 128;
            for (int i = threadIdx.x; i < nst * V; i += kThreads) {
                const int L = l0 + i % V, sl = i / V;
                const int h = (L / 8) & 1;
                const int ra = (L % 8) + 16 * (L / 16) - l0, rb_ = ra + 8;
                uint32_t w4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int mi = (st0 + sl) * 4 + k;
                    const int bl0 = (mi - st0 * 4) * bpm;  // first tile-local block of MMA mi
                    uint32_t wa = 0, wb = 0;
                    if (kN16) {
                        // MMA mt = groups 8 mt .. 8 mt + 7 = blocks 2 mt, 2 mt + 1; K-groups 4h .. 4h+3 = block 2 mt + h
                        const int bl = 2 * (mi - st0 * 4) + h;
                        wa = src16[ra * kCB + bl];
                        wb = src16[rb_ * kCB + bl];
                    } else if (kW16) {
                        // tile-local MMA mt = 2 j + hm: byte hm of the nibble words of blocks 4j + 2h, 4j + 2h + 1
                        const int mt = mi - st0 * 4, bl = 4 * (mt >> 1) + 2 * h, sh = 8 * (mt & 1);
                        wa = ((src16[ra * kCB + bl] >> sh) & 0xFFu) | (((src16[ra * kCB + bl + 1] >> sh) & 0xFFu) << 8);
                        wb = ((src16[rb_ * kCB + bl] >> sh) & 0xFFu) | (((src16[rb_ * kCB + bl + 1] >> sh) & 0xFFu) << 8);
                    } else if (M == 4) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            wa |= static_cast<uint32_t>(src[ra * kCB + bl0 + 4 * h + q]) << (4 * q);
                            wb |= static_cast<uint32_t>(src[rb_ * kCB + bl0 + 4 * h + q]) << (4 * q);
                        }
                    } else {
                        const int bl = bl0 + 2 * h;
                        wa = static_cast<uint32_t>(src[ra * kCB + bl]) | (static_cast<uint32_t>(src[ra * kCB + bl + 1]) << 8);
                        wb = static_cast<uint32_t>(src[rb_ * kCB + bl]) | (static_cast<uint32_t>(src[rb_ * kCB + bl + 1]) << 8);
                    }
                    w4[k] = mi < a.n_mma ? (wa | (wb << 16)) : 0x44444444u;
                }
                if (st0 + sl < a.n_stage_tc)
                    *reinterpret_cast<uint4*>(a.meta_tc + ((static_cast<int64_t>(t128) * a.n_stage_tc + st0 + sl) * 128 + L) * 4) =
                        make_uint4(w4[0], w4[1], w4[2], w4[3]);
            }
        }
        if (mask_out) {
            const int w0 = b0 * M / 32;
            constexpr int mwords = TC / 32;
            const int nw = min(mwords, a.ld_mask - w0);
            for (int i = threadIdx.x; i < V * nw; i += kThreads) {
                const int r = i / nw, w = i % nw;
                const int lo_col = 32 * w, hi_col = lo_col + 31;  // tile-local columns of this word
                uint32_t word = 0;
                for (int bl = lo_col / M; bl <= hi_col / M && bl < kCB; ++bl) {
                    const uint32_t bits = sBits[r * kCB + bl];
                    const int sh = bl * M - lo_col;
                    word |= sh >= 0 ? (sh < 32 ? bits << sh : 0u) : bits >> (-sh);
                }
                mask_out[static_cast<int64_t>(r0 + r) * a.ld_mask + w0 + w] = word;
            }
        }
        // ---- TMA tensor stores of the staged tile (clipped at nb_pad / rows by the tensor maps)
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            if (a.has_values) {
                tma_store_2d(&tm.val, 2 * b0, r0, sVal);
                if constexpr (kCB == 32) tma_store_2d(&tm.met, b0 / 8, r0, sMet);
            }
            if (tc) tma_store_2d(&tm.tcv, (M == 4 ? 2 : ((kW16 || kN16) ? 8 : 4)) * b0, r0, M == 4 ? static_cast<const void*>(sVal) : sTcv);
            bulk_commit();
        }
        PTRACE(5)
    }
    if (threadIdx.x == 0) bulk_wait0();
}

template <int V, int M, int NW, int MINB, int LEAN = 0>
cudaError_t launch2(const Batch& B, size_t smem, cudaStream_t st) {
    constexpr int kThreads = 32 * NW;
    auto k = prune2_kernel<V, M, NW, MINB, LEAN>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int ntiles = B.tile0[B.n];
    int grid = num_sms() * per_sm;
    if (grid > ntiles) grid = ntiles;
    k<<<grid, kThreads, smem, st>>>(B);
    count_launch();
    if (B.a[0].trace) {
        unsigned long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_prune2_t, sizeof(h));
        fprintf(stderr, "prune2 V=%d M=%d grid %d tiles %d per_sm %d: tma %llu cols %llu top4 %llu rows %llu out %llu ns\n",
                V, M, grid, ntiles, per_sm, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4]);
    }
    return cudaGetLastError();
}

template <int V, int NW, int MINB, int LEAN = 0>
cudaError_t launch_m(int M, const Batch& B, size_t smem, cudaStream_t st) {
    switch (M) {
        case 4: return launch2<V, 4, NW, MINB, LEAN>(B, smem, st);
        case 5: return launch2<V, 5, NW, MINB, LEAN>(B, smem, st);
        case 6: return launch2<V, 6, NW, MINB, LEAN>(B, smem, st);
        case 7: return launch2<V, 7, NW, MINB, LEAN>(B, smem, st);
        case 8: return launch2<V, 8, NW, MINB, LEAN>(B, smem, st);
        case 9: return launch2<V, 9, NW, MINB, LEAN>(B, smem, st);
        case 10: return launch2<V, 10, NW, MINB, LEAN>(B, smem, st);
        case 11: return launch2<V, 11, NW, MINB, LEAN>(B, smem, st);
        case 12: return launch2<V, 12, NW, MINB, LEAN>(B, smem, st);
        case 13: return launch2<V, 13, NW, MINB, LEAN>(B, smem, st);
        case 14: return launch2<V, 14, NW, MINB, LEAN>(B, smem, st);
        case 15: return launch2<V, 15, NW, MINB, LEAN>(B, smem, st);
        case 16: return launch2<V, 16, NW, MINB, LEAN>(B, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int V>
cudaError_t launch_v2(int M, const Batch& B, size_t smem, cudaStream_t st) {
    // fewer tiles than SMs: one tile per CTA, 16 warps (latency); else 8-warp CTAs, 3 per SM (throughput)
    if (V <= 64 && B.tile0[B.n] < num_sms()) return launch_m<V, 16, 1>(M, B, smem, st);
    // V = 128: the tile + staging take most of the shared memory, so one CTA per SM — of 16 warps (VNM_PRUNE_NW=8: 8)
    // (no score and no mask: those paths compile out of the per-row loop, LEAN = 2, or 1 without a tensor-core form)
    const bool nsm = !B.any_score && !B.any_mask && VNM_ENV_INT("VNM_PRUNE_LEAN2", 1);
    if (V == 128 && VNM_ENV_INT("VNM_PRUNE_NW", 16) == 16) {
        if (nsm) return B.any_tc ? launch_m<V, 16, 1, 2>(M, B, smem, st) : launch_m<V, 16, 1, 1>(M, B, smem, st);
        return launch_m<V, 16, 1>(M, B, smem, st);
    }
    if constexpr (V <= 64) {
        if (!B.any_tc && nsm) return launch_m<V, 8, 4, 1>(M, B, smem, st);
        if (!B.any_tc) return launch_m<V, 8, 4>(M, B, smem, st);  // no window form: 4 CTAs per SM (measured faster)
    }
    if (nsm) return launch_m<V, 8, 3, 2>(M, B, smem, st);
    return launch_m<V, 8, 3>(M, B, smem, st);
}

}  // namespace

static bool L_unsupported(const PruneLaunch& L) {
    const vnm_geom& g = *L.g;
    // M > 8: 16-block tiles, canonical outputs only (the window-16 / natural 2:4 forms are packed after the pass;
    // a 32-bit mask word can straddle two 16M-column tiles, so a mask output takes prune.cu)
    return L.mask_in || g.V < 32 || g.V > 128 || g.M > 16 || g.rows == 0 || g.cols == 0 ||
           (L.values_tc && (!L.meta_tc || !L.values)) ||
           (g.M > 8 && (L.mask_out || (L.values_tc && g.M % 4 == 0 && g.M != 16)));
}

// Per-problem tensor maps and arguments (+ the pad-row memsets of the window form); false: not applicable.
static bool setup_problem(const PruneLaunch& L, Maps& tm, Prune2Args& a, cudaStream_t stream) {
    const vnm_geom& g = *L.g;
    if (L_unsupported(L)) return false;
    const int kCB = kcb_of(g.M);
    const bool has_score = L.score != nullptr, tc = L.values_tc != nullptr, vals = L.values != nullptr;
    if (tc && (!L.meta_tc || !vals)) return false;
    const int tile_cols = kCB * g.M;
    if (!encode_2d(&tm.w, L.W, static_cast<uint64_t>(g.cols), static_cast<uint64_t>(g.rows),
                   static_cast<uint64_t>(L.ldw) * 2, tile_cols, g.V, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   CU_TENSOR_MAP_SWIZZLE_NONE))
        return false;
    tm.s = tm.w;
    if (has_score && !encode_2d(&tm.s, L.score, static_cast<uint64_t>(g.cols), static_cast<uint64_t>(g.rows),
                                static_cast<uint64_t>(L.lds) * 4, tile_cols, g.V, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                CU_TENSOR_MAP_SWIZZLE_NONE))
        return false;
    tm.val = tm.tcv = tm.met = tm.w;
    int n_mma = 0, ld_tc = 0;
    if (vals) {
        if (!encode_2d(&tm.val, L.values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                       static_cast<uint64_t>(g.ld_val) * 2, 2 * kCB, g.V, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                       CU_TENSOR_MAP_SWIZZLE_NONE) ||
            (kCB == 32 &&  // 16-block tiles: 8-byte A_i2 rows, below the TMA box minimum -> stored by the threads
             !encode_2d(&tm.met, L.meta, static_cast<uint64_t>(g.nb_pad / 8), static_cast<uint64_t>(g.rows_p),
                        static_cast<uint64_t>(g.ld_meta) * 4, kCB / 8, g.V, CU_TENSOR_MAP_DATA_TYPE_UINT32,
                        CU_TENSOR_MAP_SWIZZLE_NONE)))
            return false;
    }
    if (tc) {
        const bool w16 = g.M > 8;
        // natural 2:4 form (M = 16): MMAs of 8 groups over ceil8(cols_p / 4) groups; window-16: 2 MMAs per 4 blocks
        n_mma = g.M == 16 ? (g.cols_p / 4 + 7) / 8 : w16 ? g.nb_pad / 2 : g.nb_pad / (g.M == 4 ? 8 : 4);
        ld_tc = 16 * n_mma;
        const int vpb = g.M == 4 ? 2 : (w16 ? 8 : 4);  // window-form values per block
        if (!encode_2d(&tm.tcv, L.values_tc, static_cast<uint64_t>(ld_tc), static_cast<uint64_t>(g.rows_p),
                       static_cast<uint64_t>(ld_tc) * 2, vpb * kCB, g.V, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                       CU_TENSOR_MAP_SWIZZLE_NONE))
            return false;
    }
    a.mask_out = L.mask_out; a.col_idx = L.col_idx; a.meta = L.meta; a.meta_tc = L.meta_tc;
    a.ld_meta = g.ld_meta;
    a.has_values = vals ? 1 : 0; a.has_tc = tc ? 1 : 0;
    a.M = g.M; a.rows_p = g.rows_p; a.nb = g.nb; a.nb_pad = g.nb_pad; a.ld_mask = g.ld_mask;
    a.has_score = has_score ? 1 : 0;
    a.trace = VNM_ENV_INT("VNM_PRUNE_TRACE", 0) ? 1 : 0;
    a.n_mma = n_mma;
    a.n_stage_tc = (n_mma + 3) / 4;
    if (tc) {
        const int rows_w = (g.rows_p + 127) / 128 * 128;  // rows of the last 128-row tile beyond rows_p
        if (rows_w > g.rows_p) {
            cudaMemsetAsync(L.values_tc + static_cast<int64_t>(g.rows_p) * ld_tc, 0,
                            static_cast<size_t>(rows_w - g.rows_p) * ld_tc * 2, stream);
            const int l0 = g.rows_p % 128;  // lanes l0.. of the last tile hold only rows >= rows_p
            cudaMemset2DAsync(L.meta_tc + (static_cast<int64_t>(rows_w / 128 - 1) * a.n_stage_tc * 128 + l0) * 4, 2048,
                              0x44, static_cast<size_t>(128 - l0) * 16, a.n_stage_tc, stream);
        }
    }
    return true;
}

// n problems of one (V, M) in one launch.  kLaunchUnsupported when this kernel does not apply to all of them
// (the caller then falls back to one launch per problem).
int launch_prune2_batch(const PruneLaunch* Ls, int n, cudaStream_t stream) {
    if (n < 1 || n > kMaxBatch) return kLaunchUnsupported;
    const int V = Ls[0].g->V, M = Ls[0].g->M;
    for (int i = 0; i < n; ++i) {
        const vnm_geom& g = *Ls[i].g;
        if (g.V != V || g.M != M || L_unsupported(Ls[i])) return kLaunchUnsupported;
    }
    Batch B;  // host staging of the kernel parameters (copied into the launch; per call: thread-safe)
    B.n = n;
    B.tile0[0] = 0;
    B.any_score = B.any_mask = B.any_tc = 0;
    for (int i = 0; i < n; ++i) {
        if (!setup_problem(Ls[i], B.tm[i], B.a[i], stream)) return kLaunchUnsupported;
        const vnm_geom& g = *Ls[i].g;
        B.tile0[i + 1] = B.tile0[i] + ((g.nb_pad + kcb_of(M) - 1) / kcb_of(M)) * (g.rows_p / V);
        B.any_score |= B.a[i].has_score;
        B.any_mask |= Ls[i].mask_out != nullptr;
        B.any_tc |= B.a[i].has_tc;
    }
    const int kCB = kcb_of(M);
    const int tile_cols = kCB * M;
    const size_t buf = static_cast<size_t>(V) * tile_cols * 2 + (B.any_score ? static_cast<size_t>(V) * tile_cols * 4 : 0);
    const bool w16 = M > 8 && (M % 4 != 0 || M == 16);  // 8 tensor-core values per block
    const size_t smem = 2 * buf + static_cast<size_t>(V) * kCB * (B.any_tc ? 4 + (w16 ? 16 : 8) : 4) +
                        static_cast<size_t>(V) * 16 + 256 * 4 + 2 * kCB * 4 + 64 * 8 +
                        (B.any_mask ? static_cast<size_t>(V) * kCB * 4 : 0) +
                        (B.any_tc ? (w16 ? 3 : 2) : 1) * static_cast<size_t>(V) * kCB;
    if (smem > kMaxSmem) return kLaunchUnsupported;
    cudaError_t e;
    switch (V) {
        case 32: e = launch_v2<32>(M, B, smem, stream); break;
        case 64: e = launch_v2<64>(M, B, smem, stream); break;
        case 128: e = launch_v2<128>(M, B, smem, stream); break;
        default: return kLaunchUnsupported;
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

// Returns kLaunchUnsupported when this kernel does not apply (the caller falls back to prune.cu).
int launch_prune2(const PruneLaunch& L, cudaStream_t stream) { return launch_prune2_batch(&L, 1, stream); }

}  // namespace vnm
