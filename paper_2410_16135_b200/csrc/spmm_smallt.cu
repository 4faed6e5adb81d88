// spmm_smallt.cu — the small-T plan of the V:N:M SpMM (decode-sized token counts, 1 <= T <= 32, any M, V >= 16),
// SURVEY §8(a) rows a6-a8 and §8(d) config 4b; §3 "Acceleration of V:N:M sparsity" P:106-109, App. A
// P:547-548 ("retrieve the retained weights and the corresponding tiles of B").
//
// At T <= 32 the product is a stream of the canonical packed weights — A_n (2 values per block and row), A_i2
// (one 2:4 nibble per block and row) and A_i1 (4 column indices per block and V-block) — with a few MACs per
// weight, so the kernel is a TMA stream with light tensor work on top, and it reads nothing but those arrays and
// a dense slice of X^T:
//   * unit of work = 128 rows x 32 column blocks (4 k-steps of logical K = 32), staged in a ring of S slots by
//     one producer warp: the A_n box [128 rows][64 values] (128-byte swizzle) by ONE TMA; the A_i2 words
//     [128 rows][4], the A_i1 words of the unit's V-block(s) and the dense X^T slice of the 32 blocks
//     [32 M channels][TP tokens] by 16-byte cp.async from all 32 lanes, completing on the same mbarrier
//     (cp.async.mbarrier.arrive).  Measured (profiles/r02_decode.md): the TMA engine spends about the same time
//     on every box row whatever its width, and the 16-B A_i2 rows / 32-B X^T rows of a unit were 2/3 of its
//     rows — boxes of them capped a CTA at ~1 unit per 450 ns.  The X^T slice is L2-resident (every row group
//     re-reads it), written swizzled (conflict-free for the gather below) and shared by the unit's two
//     V-blocks (V = 64);
//   * warp-level sparse MMA (mma.sp::ordered_metadata m16n8k32, bf16 in, fp32 accumulate): A_n IS the
//     2:4-compressed operand of the gathered product (the block's 2 kept values = one group of 4 gathered
//     channels) and its A_i2 word is the operand's metadata; the A fragments come from the swizzled A_n box by
//     ldmatrix (conflict-free); the B fragments are GATHERED by ldmatrix.trans itself: lane i supplies the
//     shared-memory address of gathered K-row i of the k-step, i.e. X^T channel (block i/4, A_i1 position i%4)
//     of the slice — no gather copy, no B tile, no metadata repacking;
//   * 8 consumer warps: half h = w % 2 (64 rows = 4 m16 tiles = one V-block at V = 64), phase p = w / 2 (units
//     p, p + 4, ... of the CTA's share); the slot ring size S is a multiple of the phases in use (4, or S itself
//     when only 2-3 slots fit), so every slot is read by one phase only, whose warps wait on its uses in order;
//   * persistent CTAs take equal contiguous shares of the (row group, stage) list (stream-K); at the end of a
//     piece (the row group changes or the share ends) the 4 phases are added in phase order through shared
//     memory; a row group cut between CTAs is finished by the LAST CTA to arrive (ticket), which adds the fp32
//     pieces in CTA order — deterministic, no second kernel, no CTA ever waits for another.
// Why not tcgen05 here: an M = 64/128 sparse tcgen05.mma costs >= 104 cycles whatever N <= 128
// (profiles/r01_probes.md MB2) and needs the gathered B tile in shared memory plus the metadata repacked into
// TMEM each stage — per-stage work the previous small-T plan measured at ~1 us per stage (0.24 of HBM); here the
// tensor work per unit is 64 warp MMAs that hide under the stream.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kRowsU = 128;        // rows per unit (two 64-row halves)
constexpr int kKS = 4;             // k-steps (8 blocks = logical K 32) per unit
constexpr int kBlkU = 8 * kKS;     // 32 column blocks per unit
constexpr int kCons = 8;           // consumer warps
constexpr int kPhases = kCons / 2;
constexpr int kProd = kCons;       // producer warp index
constexpr int kFix = kCons + 1;    // fix-up warp: finishes every piece but the share's last, off the consumers' path
constexpr int kThreads = 32 * (kCons + 2);
constexpr uint32_t kABytes = kRowsU * 128;   // A_n box [128 rows][64 bf16], SW128
constexpr uint32_t kTicketWords = kWsTicketBytes / 4;  // fixed ticket region at the start of the workspace
constexpr int kMBoxUnits = 8;                // units per A_i2 box: [128 rows][8 units x 4 words] = 128 B per row
constexpr uint32_t kMBoxBytes = kRowsU * 128;
#ifndef VNM_ST_MB
#define VNM_ST_MB 2
#endif
constexpr int kMB = VNM_ST_MB;                       // A_i2 box ring slots
constexpr uint32_t kCRow = kBlkU * 4;        // A_i1 words of one V-block and unit (128 B)

// VNM_SPMM_TRACE: %globaltimer per CTA — entry, after the prologue, first unit landed, consumers done, exit
__device__ unsigned long long g_st_t[9][1024];  // [4..8]: last piece: reduced, ticket checked, published, folded, stored
__device__ unsigned long long g_st_u[160][32][4];  // VNM_SPMM_TRACE=2: per unit: slot free, landed, consumed, issued
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kMaxProb = 4;  // problems per launch (vnm_spmm_batched)

// one problem of the launch (its own weights, X^T, Y^T; the same T, y dtype and V class as the others)
struct StProb {
    void* YT;
    int64_t ldy;
    int32_t rows, rows_p, V, M, n_st, n_rp;
    int32_t c_rows;      // A_i1 rows (V-blocks) per unit: max(1, 128 / V)
    int32_t x_pack;      // > 1: X^T viewed as 128-byte lines of x_pack = 64 / ldx channels (SW128); 1: one row per channel
    int32_t x_l8;        // ldx / 8 (16-byte chunks per channel in the packed view)
    int32_t x_pack_log2;
    int32_t x_box, x_nbox;  // rows of the view per TMA box (<= 256), boxes per slice
    uint32_t x_box_bytes;   // shared-memory bytes per box
    uint32_t tx_bytes, c_bytes;
};

// the problems' tensor maps: [problem][A_n, X^T, A_i2, A_i1]
struct StMaps {
    CUtensorMap m[kMaxProb][4];
};

struct StArgs {
    float* ws;           // partials [row groups][maxseg][128][TP] fp32 (after the ticket region)
    uint32_t* tickets;   // [kTicketWords] per row group (all problems), zero at launch; every launch leaves them zero
    int32_t T, units, grid, maxseg, n_rg;
    int32_t n_prob;
    int32_t ub[kMaxProb + 1];  // first unit of problem i (ub[n_prob] = units); units are problem-major
    int32_t gb[kMaxProb + 1];  // first row group of problem i in the launch-wide numbering (tickets, partials)
    int32_t S;           // ring slots
    int32_t nph;         // consumer phases in use (4, 3 or 2; S is a multiple of nph)
    int32_t rg_mode;     // 1: shares are whole row groups (no workspace: no piece is ever cut between CTAs)
    int32_t wready;      // VNM_SPMM_WEIGHTS_READY: weight TMAs of the first ring fill before griddepcontrol.wait
    uint32_t x_bytes;    // X^T slice bytes per slot (the largest problem's, rounded to 1 KB)
    uint32_t slot_bytes;
    int32_t trace;
    int32_t abl;  // VNM_ABL timing ablations (-DVNM_ABLATIONS builds only; results invalid): 1 consumers skip the
                  // MMA work, 2 no X^T slice loads, 8 no A_i2 / A_i1 loads
    StProb pr[kMaxProb];
};

__device__ __forceinline__ int prob_of(const StArgs& a, int u) {  // problem holding (launch-wide) unit u
    int i = 0;
#pragma unroll
    for (int k = 1; k < kMaxProb; ++k)
        if (k < a.n_prob && u >= a.ub[k]) i = k;
    return i;
}
// (32-bit unsigned arithmetic: the host keeps units x grid and row groups x grid below 2^32; a 64-bit division is a
// ~0.3 us software routine on the tail's critical path)
__device__ __forceinline__ int unit_owner(const StArgs& a, int u) {  // CTA whose share contains unit u
    return static_cast<int>((static_cast<uint32_t>(u + 1) * static_cast<uint32_t>(a.grid) - 1u) / static_cast<uint32_t>(a.units));
}
__device__ __forceinline__ int share_begin(const StArgs& a, int b) {  // first unit of CTA b's share
    if (a.rg_mode) {  // whole row groups: the first unit of launch-wide row group G
        const int G = static_cast<int>(static_cast<uint32_t>(b) * static_cast<uint32_t>(a.n_rg) / static_cast<uint32_t>(a.grid));
        int i = 0;
#pragma unroll
        for (int k = 1; k < kMaxProb; ++k)
            if (k < a.n_prob && G >= a.gb[k]) i = k;
        return G >= a.n_rg ? a.units : a.ub[i] + (G - a.gb[i]) * a.pr[i].n_st;
    }
    return static_cast<int>(static_cast<uint32_t>(b) * static_cast<uint32_t>(a.units) / static_cast<uint32_t>(a.grid));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
// D (16 x 8, fp32) += A (16 x 32, 2:4-compressed bf16, metadata e) * B (32 x 8 bf16)
__device__ __forceinline__ void mma_sp_16832(float (&d)[4], const uint32_t (&A)[4], const uint32_t (&B)[4], uint32_t e) {
    asm volatile(
        "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
        "{%8, %9, %10, %11}, {%0, %1, %2, %3}, %12, 0x0;"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(B[0]), "r"(B[1]), "r"(B[2]), "r"(B[3]), "r"(e));
}

// byte offset of 16-byte token chunk n of X^T slice row r: rows of TP*2 bytes, TMA swizzle none (TP = 8),
// 32B (TP = 16) or 64B (TP = 32) — Swizzle<log2(TP/8),4,3>: chunk bits [4, ..) ^= row-address bits [7, ..)
template <int TP>
__device__ __forceinline__ uint32_t xoff(int r, int n) {
    if constexpr (TP == 8) return 16u * r;
    else if constexpr (TP == 16) return 32u * r + 16u * (n ^ ((r >> 2) & 1));
    else return 64u * r + 16u * (n ^ ((r >> 1) & 3));
}

// Finish piece [pu0, pu1) of row group rp whose sum is in redb [128][TP] fp32: a whole row group goes straight to
// Y^T; a row group cut between CTAs is published to the workspace and the LAST CTA to arrive adds the pieces in CTA
// order (deterministic) — the CUTLASS semaphore pattern: the pieces' stores, a barrier, ONE acq_rel atomic by
// thread 0 (release: cumulative over the group's stores through the barrier; acquire: the reads that follow the
// next barrier).  t_early: the ticket read (acquire) when the share's last piece began, or ~0u (the fix-up warp's
// pieces: straight to publishing).
// Called by the 256 consumer threads (cons: named barrier 1) for the share's last piece, and by the fix-up warp
// (__syncwarp) for the others.
template <int TP, bool kBf16, int kNthr>
__device__ __forceinline__ void finish_piece(const StArgs& a, int pi, int rp, int pu0, int pu1, float* redb, int tid,
                                             uint32_t t_early, uint32_t& flag) {
    auto sync = [&] {
        if constexpr (kNthr == 32) __syncwarp();
        else asm volatile("bar.sync 1, %0;" ::"n"(kNthr) : "memory");
    };
    constexpr int kN4 = kRowsU * TP / 4;  // float4 groups of a piece
    const bool tr = kNthr > 32 && a.trace && tid == 0 && blockIdx.x < 1024;
    if (tr) g_st_t[4][blockIdx.x] = gtime();
    const StProb& pp = a.pr[pi];
    const int row0 = rp * kRowsU;
    const int rg_u0 = a.ub[pi] + rp * pp.n_st;  // the row group's first (launch-wide) unit
    const int G = a.gb[pi] + rp;                // its launch-wide index (ticket, partials)
    float4* red4 = reinterpret_cast<float4*>(redb);
    const bool whole = pu0 == rg_u0 && pu1 == rg_u0 + pp.n_st;
    if (!whole) {
        const int own0 = unit_owner(a, rg_u0);
        const int nseg = unit_owner(a, rg_u0 + pp.n_st - 1) - own0 + 1;
        const int me = static_cast<int>(blockIdx.x) - own0;
        float* wsr = a.ws + static_cast<int64_t>(G) * a.maxseg * kRowsU * TP;
        // were all the other pieces in already when this piece began (t_early, an acquire read then)?  Then this
        // CTA is the last one and finishes without publishing its own piece; otherwise publish + count.  (No second
        // read at the end: measured, that L2 round trip (~0.7 us) cost more on the publishing path than it saved.)
        if (tid == 0) flag = t_early == static_cast<uint32_t>(nseg - 1) ? 1u : 0u;
        sync();
        if (tr) g_st_t[5][blockIdx.x] = gtime();
        if (!flag) {
            float4* mine = reinterpret_cast<float4*>(wsr + static_cast<int64_t>(me) * kRowsU * TP);
            for (int i = tid; i < kN4; i += kNthr) __stcg(mine + i, red4[i]);
            sync();
            if (tid == 0) {
                uint32_t old;
                asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.tickets + G) : "memory");
                flag = old == static_cast<uint32_t>(nseg - 1) ? 1u : 0u;
            }
            sync();
            if (tr) g_st_t[6][blockIdx.x] = gtime();
            if (!flag) return;  // an other CTA finishes the row group
        }
        // the last one: every piece, in the canonical order p_0 + (p_1 + (... + p_{nseg-1})) (this CTA's own from
        // shared memory)
        constexpr int kU = kN4 / kNthr < 2 ? (kN4 / kNthr > 0 ? kN4 / kNthr : 1) : 2;
        constexpr int kJ = 4;  // pieces whose loads are all issued before the fold (one round trip)
        for (int i0 = tid; i0 < kN4; i0 += kNthr * kU) {
            float4 sum[kU];
            if (nseg <= kJ) {
                float4 v[kJ][kU];
#pragma unroll
                for (int j = 0; j < kJ; ++j)
#pragma unroll
                    for (int k = 0; k < kU; ++k) {
                        const int i = i0 + k * kNthr;
                        if (j < nseg && i < kN4)
                            v[j][k] = j == me ? red4[i]
                                              : __ldcg(reinterpret_cast<const float4*>(wsr + static_cast<int64_t>(j) * kRowsU * TP) + i);
                    }
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    sum[k] = v[kJ - 1][k];
#pragma unroll
                    for (int j = kJ - 1; j >= 0; --j) {
                        if (j == nseg - 1) sum[k] = v[j][k];
                        else if (j < nseg - 1)
                            sum[k] = make_float4(v[j][k].x + sum[k].x, v[j][k].y + sum[k].y, v[j][k].z + sum[k].z,
                                                 v[j][k].w + sum[k].w);
                    }
                }
            } else {
                for (int j = nseg - 1; j >= 0; --j) {
                    const float4* src = reinterpret_cast<const float4*>(wsr + static_cast<int64_t>(j) * kRowsU * TP);
#pragma unroll
                    for (int k = 0; k < kU; ++k) {
                        const int i = i0 + k * kNthr;
                        if (i < kN4) {
                            const float4 v = j == me ? red4[i] : __ldcg(src + i);
                            sum[k] = j == nseg - 1 ? v : make_float4(v.x + sum[k].x, v.y + sum[k].y, v.z + sum[k].z, v.w + sum[k].w);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kU; ++k)
                if (i0 + k * kNthr < kN4) red4[i0 + k * kNthr] = sum[k];
        }
        sync();
        if (tr) g_st_t[7][blockIdx.x] = gtime();
        if (tid == 0) a.tickets[G] = 0u;  // ready for the next launch (stream order)
    }
    // Y^T rows row0 .. +127, tokens [0, T): one 16-byte group (8 bf16 / 4 fp32 tokens) per thread and step
    constexpr int kEl = kBf16 ? 8 : 4;
    constexpr int kGroups = TP / kEl;
    for (int i = tid; i < kRowsU * kGroups; i += kNthr) {
        const int r = i / kGroups, t0 = (i % kGroups) * kEl;
        const int grow = row0 + r;
        if (grow >= pp.rows || t0 >= a.T) continue;
        const float* v = redb + r * TP + t0;
        uint8_t* dst = static_cast<uint8_t*>(pp.YT) + (static_cast<int64_t>(grow) * pp.ldy + t0) * (kBf16 ? 2 : 4);
        if (t0 + kEl <= a.T) {
            uint32_t w[4];
            if constexpr (kBf16) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
                    w[e] = *reinterpret_cast<uint32_t*>(&b2);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(v[e]);
            }
            asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
        } else {
            for (int e = 0; e < a.T - t0; ++e) {
                if constexpr (kBf16)
                    reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(v[e]);
                else
                    reinterpret_cast<float*>(dst)[e] = v[e];
            }
        }
    }
}

// NT8: token tiles of 8 computed (T <= 8 NT8); VSET: V-blocks per 64-row half (64 / V for V <= 64, else 1)
template <int NT8, int VSET, bool kBf16>
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_smallt_kernel(const __grid_constant__ StMaps maps, const __grid_constant__ StArgs a) {
    constexpr int TP = NT8 == 1 ? 8 : (NT8 == 2 ? 16 : 32);  // tokens per X^T slice row in shared memory
    extern __shared__ __align__(1024) uint8_t smem[];
    // [A_i2 box ring: kMB x 16 KB][slot s: A_n 16 KB | X^T slice x_bytes | A_i1 c_rows x 128 B]
    // [red: 2 x [128][TP] fp32 (piece sums, double-buffered)][barriers]
    uint8_t* mbox = smem;
    uint8_t* slots = smem + kMB * kMBoxBytes;
    float* red = reinterpret_cast<float*>(slots + a.S * a.slot_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * kRowsU * TP);
    uint64_t* empty = full + a.S;
    uint64_t* mfull = empty + a.S;
    uint64_t* mempty = mfull + kMB;
    uint64_t* pfull = mempty + kMB;   // [2] piece j's sum is in red[j % 2] (consumers -> fix-up warp)
    uint64_t* pempty = pfull + 2;     // [2] red[j % 2] is free again (fix-up warp -> consumers)
    uint32_t* flags = reinterpret_cast<uint32_t*>(pempty + 2);  // broadcast words: [0] consumers, [1] fix-up warp

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int u0 = share_begin(a, blockIdx.x), u1 = share_begin(a, blockIdx.x + 1);
    const bool tr = a.trace && blockIdx.x < 1024 && threadIdx.x == 0;
    if (tr) g_st_t[0][blockIdx.x] = gtime();
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);   // the producer's expect_tx arrival (+ the TMA bytes)
            mbar_init(&empty[s], 2);  // the two half warps of the phase that consumes the slot
        }
        for (int k = 0; k < kMB; ++k) {
            mbar_init(&mfull[k], 1);
            mbar_init(&mempty[k], 2 * a.nph);  // every consumer warp of a phase in use releases every box once
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&pfull[k], 1);
            mbar_init(&pempty[k], 1);
        }

        fence_mbar_init();
    }
    if (warp == kProd && lane == 0) {
        for (int i = 0; i < a.n_prob; ++i)
            for (int j = 0; j < 4; ++j) tma_prefetch_desc(&maps.m[i][j]);
    }
    __syncthreads();
    // the previous kernel's outputs (this layer's X^T, packed weights, the workspace) are visible; with
    // weights_ready the producer waits later, after issuing the weights of its first units (below)
    if (!(warp == kProd && a.wready)) grid_dep_wait();
    grid_dep_launch();  // the next kernel may take SMs as this grid's CTAs exit
    if (tr) g_st_t[1][blockIdx.x] = gtime();

    if (warp == kProd) {
        // ------------------------------------------------------------ producer: lane 0 issues the TMAs (A_n box +
        // X^T slice boxes).  (L2 prefetches of the A_i2 / A_i1 lines from the other lanes measured slower.)
        if (lane == 0) {
            // A_i2 words: a few long TMA rows per row group instead of a 16-byte row per unit — boxes
            // [128 rows][8 units x 4 words] (128-byte swizzle) from the first unit of each piece (row group of the
            // share) on, in a ring of kMB boxes; box k is issued with the first unit that reads it
            int k = 0, pend = u0;  // next box; first unit past the last issued box
            int pi = prob_of(a, u0);
            const CUtensorMap* tm = maps.m[pi];
            // the problem's fields in registers (re-read only at a problem switch: param-space loads through a
            // dynamic index are on the issue path of every unit otherwise)
            int n_st, n_rp, M, xpl2, x_nbox, x_box, V, ub;
            uint32_t tx, c_bytes, xbb;
            auto load_prob = [&](int i) {
                const StProb& q = a.pr[i];
                n_st = q.n_st; n_rp = q.n_rp; M = q.M; xpl2 = q.x_pack_log2; x_nbox = q.x_nbox; x_box = q.x_box;
                V = q.V; tx = q.tx_bytes; c_bytes = q.c_bytes; xbb = q.x_box_bytes; ub = a.ub[i];
            };
            load_prob(pi);
            int rp = (u0 - ub) / n_st, st = u0 - ub - rp * n_st, s = 0, par = 0;  // (incremental)
            // weights_ready (vnm_spmm_batched flag): the packed weights were written before the previous kernel
            // began, so the first ring fill's weight boxes (A_n, A_i2, A_i1) are issued BEFORE waiting for that
            // kernel (they stream in during its tail); their X^T slices follow the wait
            int npre = a.wready ? min(a.S, u1 - u0) : 0;
            int dx_s[16], dx_y0[16], dx_pi[16];
            auto flush_pre = [&](int n) {  // wait for the previous kernel, then the X^T slices of units [0, n)
                grid_dep_wait();
                for (int j = 0; j < n; ++j) {
                    const StProb& pj = a.pr[dx_pi[j]];
                    uint8_t* bj = slots + dx_s[j] * a.slot_bytes;
                    for (int b = 0; b < ((a.abl & 2) ? 0 : pj.x_nbox); ++b)
                        tma_load_2d(bj + kABytes + b * pj.x_box_bytes, &maps.m[dx_pi[j]][1], 0, dx_y0[j] + b * pj.x_box,
                                    &full[dx_s[j]]);
                }
            };
            for (int u = u0, q = 0; u < u1; ++u, ++q) {
                // a third A_i2 box needs a ring slot the consumers release only after units that need X^T: end
                // the pre-wait phase first (short row groups)
                if (q < npre && u == pend && k >= kMB) {
                    flush_pre(q);
                    npre = q;
                }
                if (u == pend) {
                    const int pu1 = min(u1, ub + (rp + 1) * n_st);
                    const int ms = k % kMB;
                    mbar_wait(&mempty[ms], ((k / kMB) & 1) ^ 1);
                    mbar_arrive_expect_tx(&mfull[ms], kMBoxBytes);
                    tma_load_2d(mbox + ms * kMBoxBytes, &tm[2], kKS * st, rp * kRowsU, &mfull[ms]);
                    pend = min(pu1, u + kMBoxUnits);
                    ++k;
                }
                mbar_wait(&empty[s], par ^ 1);
                if (a.trace == 2 && blockIdx.x < 160 && q < 32) g_st_u[blockIdx.x][q][0] = gtime();
                uint8_t* base = slots + s * a.slot_bytes;
                mbar_arrive_expect_tx(&full[s], (a.abl & 2) ? kABytes + c_bytes : tx);
                tma_load_2d(base, &tm[0], st * 2 * kBlkU, rp * kRowsU, &full[s]);
                tma_load_2d(base + kABytes + a.x_bytes, &tm[3], st * kBlkU, (rp * kRowsU) / V, &full[s]);
                const int y0 = (st * kBlkU * M) >> xpl2;  // first row of the slice in the X^T view
                if (q < npre) {  // X^T after the wait
                    dx_s[q] = s;
                    dx_y0[q] = y0;
                    dx_pi[q] = pi;
                    if (q == npre - 1) flush_pre(npre);
                } else {
                    for (int b = 0; b < ((a.abl & 2) ? 0 : x_nbox); ++b)
                        tma_load_2d(base + kABytes + b * xbb, &tm[1], 0, y0 + b * x_box, &full[s]);
                }
                if (a.trace == 2 && blockIdx.x < 160 && q < 32) g_st_u[blockIdx.x][q][3] = gtime();
                if (++s == a.S) {
                    s = 0;
                    par ^= 1;
                }
                if (++st == n_st) {
                    st = 0;
                    if (++rp == n_rp && u + 1 < u1) {  // next problem
                        rp = 0;
                        ++pi;
                        load_prob(pi);
                        tm = maps.m[pi];
                    }
                }
            }
        }
        return;
    }

    if (warp == kFix) {
        // ------------------------------------------------------------ fix-up warp: every piece but the last
        int jp = 0;
        for (int pu0 = u0; pu0 < u1; ++jp) {
            const int pi = prob_of(a, pu0), rp = (pu0 - a.ub[pi]) / a.pr[pi].n_st;
            const int pu1 = min(u1, a.ub[pi] + (rp + 1) * a.pr[pi].n_st);
            if (pu1 == u1) break;  // the share's last piece: the consumers finish it
            mbar_wait(&pfull[jp & 1], (jp >> 1) & 1);
            finish_piece<TP, kBf16, 32>(a, pi, rp, pu0, pu1, red + (jp & 1) * (kRowsU * TP), lane, ~0u, flags[1]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&pempty[jp & 1]);
            pu0 = pu1;
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int h = warp & 1, p = warp >> 1;
    const int g = lane >> 2, c = lane & 3;
    const int hsh = 16 * (c & 1);  // metadata half of this thread (selector 0: threads c = 0, 1 of each group)
    const int cons_tid = threadIdx.x;  // 0 .. 255
    float acc[4][NT8][4];
    int k_piece = 0;  // first A_i2 box of the current piece (the producer's order)
    int k_rel = 0;    // first box this warp has not released yet
    // release boxes [k_rel, k_end) (each waited on first: a box is released only after it was (re)issued, so the
    // arrivals of consecutive uses of a ring slot never mix)
    auto release_to = [&](int k_end) {
        for (; k_rel < k_end; ++k_rel) {
            mbar_wait(&mfull[k_rel % kMB], (k_rel / kMB) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&mempty[k_rel % kMB]);
        }
    };

    int jp = 0;  // piece index (the fix-up warp's numbering)
    for (int pu0 = u0; pu0 < u1;) {
        const int pi = prob_of(a, pu0);
        const StProb& pp = a.pr[pi];
        const int rg_u0 = a.ub[pi] + (pu0 - a.ub[pi]) / pp.n_st * pp.n_st;  // the row group's first unit
        const int rp = (rg_u0 - a.ub[pi]) / pp.n_st;
        const int pu1 = min(u1, rg_u0 + pp.n_st);
        // this problem's geometry for the k-step loop
        const int M = pp.M, c_rows = pp.c_rows, x_pack = pp.x_pack, x_pack_log2 = pp.x_pack_log2, x_l8 = pp.x_l8;
        // the share's last piece of a cut row group: read its ticket now (acquire); used when the piece is done
        uint32_t t_early = ~0u;
        if (pu1 == u1 && !(pu0 == rg_u0 && pu1 == rg_u0 + pp.n_st) && cons_tid == 0 && !a.rg_mode)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(t_early) : "l"(a.tickets + a.gb[pi] + rp) : "memory");

#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int n = 0; n < NT8; ++n)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[mt][n][k] = 0.f;
        const bool half_ok = rp * kRowsU + 64 * h < pp.rows_p;
        // this phase's units of the piece: u = u0 + q, q = p (mod nph); phases p >= nph have none
        const int nph = a.nph;
        int u = p < nph ? pu0 + ((p - (pu0 - u0)) % nph + nph) % nph : pu1;
        int s = (u - u0) % a.S, par = ((u - u0) / a.S) & 1;  // slot / phase parity, advanced without divisions
        for (; u < pu1; u += nph) {
            const int q = u - u0;
            const int kb = k_piece + (u - pu0) / kMBoxUnits, ub = (u - pu0) % kMBoxUnits;
            release_to(kb);
            mbar_wait(&mfull[kb % kMB], (kb / kMB) & 1);
            mbar_wait(&full[s], par);
            if (tr && q == 0) g_st_t[2][blockIdx.x] = gtime();
            if (a.trace == 2 && lane == 0 && h == 0 && blockIdx.x < 160 && q < 32) g_st_u[blockIdx.x][q][1] = gtime();
            if (half_ok && !(a.abl & 1)) {
                const uint32_t sA = smem_u32(slots + s * a.slot_bytes);
                const uint32_t sX = sA + kABytes, sC = sX + a.x_bytes;
                const uint32_t sMb = smem_u32(mbox + (kb % kMB) * kMBoxBytes);
                // A_i2 words of this unit for rows g, g + 8 of every m16 tile (4 words = the unit's 4 k-steps):
                // row r of the box holds 8 units x 16 B, 16-byte chunk ub at ub ^ (r % 8) (SW128)
                uint4 w0[4], w1[4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    const int r0 = 64 * h + 16 * mt + g;  // (r0 + 8) % 8 == r0 % 8
                    const uint32_t o = 16u * ((ub ^ r0) & 7);
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(w0[mt].x), "=r"(w0[mt].y), "=r"(w0[mt].z), "=r"(w0[mt].w)
                                 : "r"(sMb + 128u * r0 + o));
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(w1[mt].x), "=r"(w1[mt].y), "=r"(w1[mt].z), "=r"(w1[mt].w)
                                 : "r"(sMb + 128u * (r0 + 8) + o));
                }
                // Manually scheduled (in-order issue; the asm statements keep program order): the A_i1 words of
                // all k-steps first, the gathered B fragments one k-step ahead of their MMAs, the 4 A fragments of
                // a k-step before its MMAs.  K-steps past n_ks are computed too: their A values are zero (TMA
                // zero fill past ld_val) and their metadata the pad pattern, so they add exact zeros.
                const int jm = lane >> 3, rr = lane & 7;
                uint32_t cwv[kKS][VSET];
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks)
#pragma unroll
                    for (int v = 0; v < VSET; ++v) {
                        const int crow = c_rows == 1 ? 0 : h * VSET + v;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cwv[ks][v]) : "r"(sC + crow * kCRow + 4 * (8 * ks + (lane >> 2))));
                    }
                // B of k-step ks: lane i addresses gathered K-row i = block 8 ks + i / 4, A_i1 position i % 4
                auto load_b = [&](int ks, uint32_t (&B)[VSET][NT8][4]) {
#pragma unroll
                    for (int v = 0; v < VSET; ++v) {
                        const int xr = (8 * ks + (lane >> 2)) * M + static_cast<int>((cwv[ks][v] >> (8 * (lane & 3))) & 0xFFu);
#pragma unroll
                        for (int n = 0; n < NT8; ++n) {
                            uint32_t off;
                            if (x_pack > 1) {  // X^T viewed as 128-byte lines of x_pack channels (SW128)
                                const int line = xr >> x_pack_log2;
                                const int ch = (xr & (x_pack - 1)) * x_l8 + n;
                                off = 128u * line + 16u * ((ch ^ line) & 7);
                            } else {
                                off = xoff<TP>(xr, n);
                            }
                            ldsm_x4_t(sX + off, B[v][n]);
                        }
                    }
                };
                uint32_t Bb[2][VSET][NT8][4];
                load_b(0, Bb[0]);
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    if (ks + 1 < kKS) load_b(ks + 1, Bb[(ks + 1) & 1]);
                    uint32_t A[4][4];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        const int row = 64 * h + 16 * mt + rr + 8 * (jm & 1);
                        const int chunk = 2 * ks + (jm >> 1);
                        ldsm_x4(sA + 128 * row + 16 * ((chunk ^ row) & 7), A[mt]);
                    }
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        const uint32_t x0 = ks == 0 ? w0[mt].x : ks == 1 ? w0[mt].y : ks == 2 ? w0[mt].z : w0[mt].w;
                        const uint32_t x1 = ks == 0 ? w1[mt].x : ks == 1 ? w1[mt].y : ks == 2 ? w1[mt].z : w1[mt].w;
                        const uint32_t e = ((x0 >> hsh) & 0xFFFFu) | (((x1 >> hsh) & 0xFFFFu) << 16);
                        const int v = mt / (4 / VSET);
#pragma unroll
                        for (int n = 0; n < NT8; ++n) mma_sp_16832(acc[mt][n], A[mt], Bb[ks & 1][v][n], e);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (a.trace == 2 && lane == 0 && h == 0 && blockIdx.x < 160 && q < 32) g_st_u[blockIdx.x][q][2] = gtime();
            for (s += nph; s >= a.S; s -= a.S) par ^= 1;
        }
        k_piece += (pu1 - pu0 + kMBoxUnits - 1) / kMBoxUnits;
        if (p < a.nph) release_to(k_piece);  // the piece's boxes are done (also those this warp had no unit in)
        // ---- end of the piece: the phases' sums added in phase order, ((p_0 + p_1) + p_2) + p_3, into red[j % 2] by
        // a chain of named barriers — phase r adds its share as soon as its own units are done and phase r - 1 has
        // added its own (the chain mostly overlaps the later phases' last units; one step of it after the last
        // unit, where 4 CTA-wide rounds measured ~0.9 us); every piece but the share's last goes to the fix-up warp
        // (the consumers move on at once), the last one is finished here
        const bool last_piece = pu1 == u1;
        float* redb = red + (jp & 1) * (kRowsU * TP);
        if (p < a.nph) {
            if (p == 0) {
                if (cons_tid == 0) mbar_wait(&pempty[jp & 1], ((jp >> 1) & 1) ^ 1);  // its use two pieces ago is done
                asm volatile("bar.sync 2, 64;" ::: "memory");
            } else {
                asm volatile("bar.sync %0, 128;" ::"r"(2 + p) : "memory");  // phase p - 1 has added its sums
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int n = 0; n < NT8; ++n)
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        float2* d = reinterpret_cast<float2*>(redb + (64 * h + 16 * mt + g + 8 * k2) * TP + 8 * n + 2 * c);
                        float2 v = make_float2(acc[mt][n][2 * k2], acc[mt][n][2 * k2 + 1]);
                        if (p > 0) {
                            const float2 o = *d;
                            v.x = o.x + v.x;
                            v.y = o.y + v.y;
                        }
                        *d = v;
                    }
            if (p + 1 < a.nph) asm volatile("bar.arrive %0, 128;" ::"r"(3 + p) : "memory");  // phase p + 1 may add
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kCons) : "memory");  // the piece's sum is complete
        if (!last_piece) {
            if (cons_tid == 0) mbar_arrive(&pfull[jp & 1]);
        } else {
            finish_piece<TP, kBf16, 32 * kCons>(a, pi, rp, pu0, pu1, redb, cons_tid, t_early, flags[0]);
        }
        ++jp;
        pu0 = pu1;
    }
    if (tr) g_st_t[3][blockIdx.x] = gtime();
}

struct StProbPlan {
    int n_rp, n_st, c_rows, x_pack, x_box, x_nbox;
    uint32_t x_box_bytes, x_bytes;
};

struct StPlan {
    int n, units, n_rg, grid, maxseg, S, nph, tp, c_rows;
    int ub[kMaxProb + 1], gb[kMaxProb + 1];
    StProbPlan pr[kMaxProb];
    uint32_t x_bytes, slot_bytes;
    size_t smem, ws_bytes;
    bool ok;
};

// n problems of one launch (the same T; units problem-major).  ldx[i]: X^T_i's leading dimension (nullptr or 0:
// assume ldx == TP, the dense case; only the X^T view / box shape depend on it)
StPlan make_plan(const vnm_geom* const* gs, const int64_t* ldx, int n, int32_t T) {
    StPlan p{};
    p.n = n;
    p.tp = T <= 8 ? 8 : (T <= 16 ? 16 : 32);
    p.ok = n >= 1 && n <= kMaxProb && T >= 1 && T <= 32;
    if (!p.ok) return p;
    int vset0 = 0;
    for (int i = 0; i < n; ++i) {
        const vnm_geom& g = *gs[i];
        StProbPlan& q = p.pr[i];
        const int vset = g.V >= 64 ? 1 : (g.V > 0 ? 64 / g.V : 0);
        if (g.V < 16 || g.nb_pad == 0 || g.rows_p == 0 || (i > 0 && vset != vset0)) {
            p.ok = false;
            return p;
        }
        vset0 = vset;
        q.n_rp = (g.rows_p + kRowsU - 1) / kRowsU;
        q.n_st = (g.nb_pad / 8 + kKS - 1) / kKS;
        q.c_rows = g.V >= kRowsU ? 1 : kRowsU / g.V;
        // X^T slice by TMA: with a dense X^T (ldx == TP) the slice rows are contiguous, so it is viewed as 128-byte
        // lines of 64 / TP channels (4x fewer, 4x longer TMA rows at TP = 16; SW128); otherwise one row per channel
        const int64_t lx = (ldx && ldx[i]) ? ldx[i] : p.tp;
        q.x_pack = (lx == p.tp && g.cols % (64 / p.tp) == 0) ? 64 / p.tp : 1;
        const int vrows = kBlkU * g.M / q.x_pack;  // rows of the X^T view per slice
        const uint32_t row_bytes = q.x_pack > 1 ? 128u : static_cast<uint32_t>(p.tp * 2);
        q.x_nbox = (vrows + 255) / 256;
        q.x_box = ((vrows + q.x_nbox - 1) / q.x_nbox + 7) / 8 * 8;  // whole 8-row swizzle atoms per box
        q.x_box_bytes = static_cast<uint32_t>(q.x_box) * row_bytes;
        q.x_bytes = (q.x_nbox * q.x_box_bytes + 1023) / 1024 * 1024;
        p.ub[i] = p.units;
        p.gb[i] = p.n_rg;
        p.units += q.n_rp * q.n_st;
        p.n_rg += q.n_rp;
        p.x_bytes = q.x_bytes > p.x_bytes ? q.x_bytes : p.x_bytes;
        p.c_rows = q.c_rows > p.c_rows ? q.c_rows : p.c_rows;
    }
    p.ub[n] = p.units;
    p.gb[n] = p.n_rg;
    p.grid = p.units < num_sms() ? p.units : num_sms();
    p.slot_bytes = (kABytes + p.x_bytes + p.c_rows * kCRow + 1023) / 1024 * 1024;
    const size_t fixed = static_cast<size_t>(kMB) * kMBoxBytes + 2 * static_cast<size_t>(kRowsU) * p.tp * 4 +
                         (2 * 16 + 2 * kMB + 4) * 8 + 64;
    p.S = static_cast<int>((kMaxSmem - fixed) / p.slot_bytes);
    if (p.S > 16) p.S = 16;
    // S a multiple of the phase count nph: slot s is then only ever read by the warps of phase s % nph, which wait
    // on its uses in order.  (Otherwise use j + 2 of a slot can belong to a phase that never waited on use j + 1,
    // and its parity wait passes while use j + 1's TMA is still in flight: a parity wait cannot tell phase j from
    // phase j + 2.  Seen as a rare illegal-instruction trap on the producer's next arrive, S = 9.)
    // The phases in use (4, 3 or 2) are chosen for the deepest ring (the consumers are not the bottleneck: a unit
    // keeps a warp ~0.4 us busy against the producer's ~0.5 us per unit, profiles/r02c_trace_up.txt).
    {
        int best_s = 0, best_n = 1;
        for (int k = kPhases; k >= 2; --k)
            if (p.S - p.S % k > best_s) {
                best_s = p.S - p.S % k;
                best_n = k;
            }
        p.nph = best_n;
        p.S = best_s;
    }
    p.smem = static_cast<size_t>(p.S) * p.slot_bytes + fixed;
    p.maxseg = 1;
    for (int i = 0; i < n; ++i)
        for (int rp = 0; rp < p.pr[i].n_rp; ++rp) {
            const long long x0 = p.ub[i] + static_cast<long long>(rp) * p.pr[i].n_st, x1 = x0 + p.pr[i].n_st - 1;
            const int o0 = static_cast<int>(((x0 + 1) * p.grid - 1) / p.units);
            const int o1 = static_cast<int>(((x1 + 1) * p.grid - 1) / p.units);
            if (o1 - o0 + 1 > p.maxseg) p.maxseg = o1 - o0 + 1;
        }
    p.ws_bytes = kTicketWords * 4 + static_cast<size_t>(p.n_rg) * p.maxseg * kRowsU * p.tp * 4;
    p.ok = p.S >= 2 && p.n_rg <= static_cast<int>(kTicketWords) &&
           static_cast<uint64_t>(p.units + 1) * static_cast<uint64_t>(num_sms() + 1) < (1ull << 32);  // 32-bit share math
    return p;
}

template <int NT8, int VSET>
int launch_nt(vnm_dtype y_dtype, const StPlan& p, const StArgs& a, const StMaps& maps, cudaStream_t st) {
    auto k = y_dtype == VNM_BF16 ? vnm_spmm_smallt_kernel<NT8, VSET, true> : vnm_spmm_smallt_kernel<NT8, VSET, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)) != cudaSuccess)
        return kLaunchCudaError;
    if (a.trace) {  // the last-piece stamps are written only by the CTAs that reach them
        void* sym = nullptr;
        if (cudaGetSymbolAddress(&sym, g_st_t) == cudaSuccess) cudaMemsetAsync(sym, 0, sizeof(unsigned long long) * 9 * 1024, st);
    }
    cudaError_t e = launch_pdl(true, k, dim3(a.grid), dim3(kThreads), p.smem, st, maps, a);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess && a.trace) {
        static unsigned long long h[9][1024];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_st_t, sizeof(h));
        unsigned long long t0 = ~0ull, mx[4] = {0, 0, 0, 0}, mn[4] = {~0ull, ~0ull, ~0ull, ~0ull};
        const int n = a.grid < 1024 ? a.grid : 1024;
        for (int i = 0; i < n; ++i) t0 = h[0][i] < t0 ? h[0][i] : t0;
        for (int j = 0; j < 4; ++j)
            for (int i = 0; i < n; ++i) {
                const unsigned long long v = h[j][i] - t0;
                mx[j] = v > mx[j] ? v : mx[j];
                mn[j] = v < mn[j] ? v : mn[j];
            }
        fprintf(stderr, "smallt grid %d S %d units %d slot %u B: entry %llu..%llu  prologue %llu..%llu  first %llu..%llu  "
                        "done %llu..%llu ns\n", a.grid, p.S, p.units, p.slot_bytes, mn[0], mx[0], mn[1], mx[1], mn[2], mx[2],
                mn[3], mx[3]);
        if (a.trace == 2) {
            static unsigned long long u[160][32][4];
            cudaMemcpyFromSymbol(u, g_st_u, sizeof(u));
            for (int i = 0; i < n && i < 160; ++i) {
                const int nu = static_cast<int>(static_cast<long long>(i + 1) * p.units / a.grid -
                                                static_cast<long long>(i) * p.units / a.grid);
                auto rel = [&](int j) { return h[j][i] ? (h[j][i] - t0) / 10 : 0ull; };
                fprintf(stderr, "cta %3d done %6llu fin [%llu %llu %llu %llu]:", i, h[3][i] - t0, rel(4), rel(5), rel(6), rel(7));
                for (int q = 0; q < nu && q < 32; ++q)
                    fprintf(stderr, " [%llu %llu %llu %llu]", (u[i][q][0] - t0) / 10, (u[i][q][3] - t0) / 10,
                            (u[i][q][1] - t0) / 10, (u[i][q][2] - t0) / 10);
                fprintf(stderr, "\n");
            }
        }
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

template <int VSET>
int launch_v(int32_t T, vnm_dtype y_dtype, const StPlan& p, const StArgs& a, const StMaps& maps, cudaStream_t st) {
    const int nt8 = (T + 7) / 8;
    if (nt8 <= 1) return launch_nt<1, VSET>(y_dtype, p, a, maps, st);
    if (nt8 == 2) return launch_nt<2, VSET>(y_dtype, p, a, maps, st);
    if (nt8 == 3) return launch_nt<3, VSET>(y_dtype, p, a, maps, st);
    return launch_nt<4, VSET>(y_dtype, p, a, maps, st);
}

StPlan plan_of(const SpmmLaunch* Ls, int n, bool use_ldx) {
    const vnm_geom* gs[kMaxProb] = {};
    int64_t lx[kMaxProb] = {};
    if (n < 1 || n > kMaxProb) return StPlan{};
    for (int i = 0; i < n; ++i) {
        gs[i] = &Ls[i].P->g;
        lx[i] = use_ldx ? Ls[i].ldx : 0;
        if (Ls[i].T != Ls[0].T || Ls[i].y_dtype != Ls[0].y_dtype) return StPlan{};
    }
    return make_plan(gs, lx, n, Ls[0].T);
}

}  // namespace

bool spmm_smallt_applies(const vnm_geom& g, int32_t T) {
    if (T < 1 || T > 32 || g.V < 16 || g.nb_pad == 0) return false;
    const vnm_geom* gs[1] = {&g};
    return make_plan(gs, nullptr, 1, T).ok;
}

size_t spmm_smallt_workspace_bytes(const vnm_geom& g, int32_t T) {
    const vnm_geom* gs[1] = {&g};
    return spmm_smallt_applies(g, T) ? make_plan(gs, nullptr, 1, T).ws_bytes : 0;
}

bool spmm_smallt_batch_applies(const vnm_geom* const* gs, int n, int32_t T) {
    if (n < 1 || n > kMaxProb) return false;
    for (int i = 0; i < n; ++i)
        if (!spmm_smallt_applies(*gs[i], T)) return false;
    return make_plan(gs, nullptr, n, T).ok;
}

size_t spmm_smallt_batch_workspace_bytes(const vnm_geom* const* gs, int n, int32_t T) {
    return spmm_smallt_batch_applies(gs, n, T) ? make_plan(gs, nullptr, n, T).ws_bytes : 0;
}

int launch_spmm_smallt_batch(const SpmmLaunch* Ls, int n, uint32_t flags, cudaStream_t stream) {
    const StPlan p = plan_of(Ls, n, true);
    if (!p.ok) return kLaunchUnsupported;
    for (int i = 0; i < n; ++i)
        if (!spmm_smallt_applies(Ls[i].P->g, Ls[i].T)) return kLaunchUnsupported;
    const SpmmLaunch& L0 = Ls[0];
    StArgs a{};
    // without a workspace (or a too small one) every CTA takes whole row groups: nothing is cut, no tickets
    a.rg_mode = (!L0.workspace || L0.workspace_bytes < p.ws_bytes) ? 1 : 0;
    a.grid = a.rg_mode ? (p.n_rg < num_sms() ? p.n_rg : num_sms()) : p.grid;
    a.tickets = a.rg_mode ? nullptr : static_cast<uint32_t*>(L0.workspace);
    a.ws = a.rg_mode ? nullptr : reinterpret_cast<float*>(static_cast<uint8_t*>(L0.workspace) + kTicketWords * 4);
    a.T = L0.T;
    a.units = p.units;
    a.n_rg = p.n_rg;
    a.maxseg = p.maxseg;
    a.n_prob = n;
    for (int i = 0; i <= n; ++i) {
        a.ub[i] = p.ub[i];
        a.gb[i] = p.gb[i];
    }
    a.S = p.S;
    a.wready = (flags & 1u) ? 1 : 0;
    a.nph = p.nph;
    a.x_bytes = p.x_bytes;
    a.slot_bytes = p.slot_bytes;
    a.trace = VNM_ENV_INT("VNM_SPMM_TRACE", 0);
    a.abl = VNM_ABLATION_FLAGS();
    StMaps maps;
    for (int i = 0; i < n; ++i) {
        const SpmmLaunch& L = Ls[i];
        const vnm_geom& g = L.P->g;
        const StProbPlan& q = p.pr[i];
        StProb& pr = a.pr[i];
        pr.YT = L.YT;
        pr.ldy = L.ldy;
        pr.rows = g.rows;
        pr.rows_p = g.rows_p;
        pr.V = g.V;
        pr.M = g.M;
        pr.n_st = q.n_st;
        pr.n_rp = q.n_rp;
        pr.c_rows = q.c_rows;
        pr.x_pack = q.x_pack;
        pr.x_l8 = static_cast<int32_t>(L.ldx / 8);
        pr.x_pack_log2 = q.x_pack == 8 ? 3 : q.x_pack == 4 ? 2 : q.x_pack == 2 ? 1 : 0;
        pr.x_box = q.x_box;
        pr.x_nbox = q.x_nbox;
        pr.x_box_bytes = q.x_box_bytes;
        pr.c_bytes = q.c_rows * kCRow;
        pr.tx_bytes = kABytes + static_cast<uint32_t>(q.x_nbox) * q.x_box_bytes + pr.c_bytes;
        // A_n [rows_p][ld_val] bf16, boxes [128 rows][64 values]; X^T as lines of x_pack channels [cols / x_pack][64]
        // (SW128) or [cols][T] (boxes TP wide, 32B / 64B swizzle).  Past an edge boxes are zero-filled (rows past
        // rows_p, pad k-steps, channels past cols, tokens past T).
        CUtensorMap* tm = maps.m[i];
        const CUtensorMapSwizzle xsw = q.x_pack > 1 ? CU_TENSOR_MAP_SWIZZLE_128B
                                      : (p.tp == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                                   : (p.tp == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B));
        const bool okx = q.x_pack > 1
            ? encode_2d(&tm[1], L.XT, 64, static_cast<uint64_t>(g.cols / q.x_pack), 128, 64, static_cast<uint32_t>(q.x_box),
                        CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xsw)
            : encode_2d(&tm[1], L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), static_cast<uint64_t>(L.ldx) * 2,
                        static_cast<uint32_t>(p.tp), static_cast<uint32_t>(q.x_box), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xsw);
        // A_i2 [rows_p][ld_meta] u32, boxes [128 rows][32 words] (SW128; past n_ks: zero, never read); A_i1 as u32
        // [rows_p / V][nb_pad], boxes [c_rows][32 words]
        if (!okx || !encode_2d(&tm[0], L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                               static_cast<uint64_t>(g.ld_val) * 2, 64, kRowsU) ||
            !encode_2d(&tm[2], L.P->meta, static_cast<uint64_t>(g.ld_meta), static_cast<uint64_t>(g.rows_p),
                       static_cast<uint64_t>(g.ld_meta) * 4, 32, kRowsU, CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !encode_2d(&tm[3], L.P->col_idx, static_cast<uint64_t>(g.nb_pad), static_cast<uint64_t>(g.rows_p / g.V),
                       static_cast<uint64_t>(g.nb_pad) * 4, kBlkU, static_cast<uint32_t>(q.c_rows), CU_TENSOR_MAP_DATA_TYPE_UINT32,
                       CU_TENSOR_MAP_SWIZZLE_NONE))
            return kLaunchCudaError;
    }
    const int vset = L0.P->g.V >= 64 ? 1 : 64 / L0.P->g.V;
    if (vset == 1) return launch_v<1>(L0.T, L0.y_dtype, p, a, maps, stream);
    if (vset == 2) return launch_v<2>(L0.T, L0.y_dtype, p, a, maps, stream);
    return launch_v<4>(L0.T, L0.y_dtype, p, a, maps, stream);
}

int launch_spmm_smallt(const SpmmLaunch& L, cudaStream_t stream) { return launch_spmm_smallt_batch(&L, 1, 0u, stream); }

}  // namespace vnm
