// spmm_tc3.cu — the window-form V:N:M SpMM (include/vnm.h values_tc / meta_tc) on CTA
// pairs (tcgen05.mma.sp.cta_group::2, M = 256), built from the round-1c measurements (profiles/r01c_*):
//
//  * A (values_tc) and the metadata either stay RESIDENT for the pair's lifetime (short K: the DeiT layers;
//    A in shared memory, metadata copied once into TMEM) or STREAM through the ring with X^T (long K: Llama);
//  * X^T is staged in a K-RING: per 64-token chunk one contiguous run of rows, stage s at rows
//    [slot * rows_stage, +rows_stage) — each X^T row is loaded once per tile (the per-stage window overhang of
//    the 1-CTA / tc2 kernels is gone).  For 5 <= M <= 7 the windows of a stage's last blocks reach <= 7 rows
//    into the next slot, so stage q is issued only after stage q + 1 has landed; slot S-1 reaches into an
//    8-row shadow loaded together with slot 0.  Window positions outside a block carry zero values, so stale
//    rows there multiply zeros (the ring is zero-filled at start, X^T is finite by precondition);
//  * each CTA loads exactly its NT/2 tokens: a 64-token box plus a second box of NT/2 - 64 tokens (TMA keeps
//    the 128-byte row pitch and swizzle for boxes narrower than the span: tests/probes/probe_box.cu), issued
//    by two producer threads;
//  * NT = 224 with two accumulators (2 x 224 + metadata <= 512 TMEM columns: the epilogue of tile i overlaps
//    the MMAs of tile i + 1) or NT = 256 with one (token counts that are multiples of 256: no padded tile;
//    the epilogue drains the accumulator into registers first and releases it before storing);
//  * the MMA warp stays converged and issues each stage from one asm block (ptx.cuh mma_sp_stage);
//  * 8 epilogue warps (2 per TMEM lane quadrant, alternate 64-token chunks) store Y^T with coalesced
//    st.global.v4 (4 rows x 128 B per instruction) after a warp-private SW128 transpose in shared memory —
//    no TMA stores (they queued behind the X^T loads in the same TMA unit), no proxy fences;
//  * the accumulator release from the peer CTA is a CTA-scope remote mbarrier arrive (the cluster-scope
//    release compiled to MEMBAR.ALL.GPU + ERRBAR and was 18 % of the stall samples).
//
// Roles: warps 0 and 2 TMA producers (both CTAs), warp 1 MMA (leader CTA), warps 4-11 epilogue (both CTAs:
// TMEM lanes 32q.. = rows 32q.. of the CTA's 128-row tile).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <type_traits>

#include "ptx.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr uint32_t kABytes = 128 * 128;  // one 4-MMA chunk of A: 128 rows x 64 bf16 (SW128)
constexpr uint32_t kEBytes = 128 * 16;   // one 4-MMA chunk of metadata: 128 lanes x 4 words
constexpr uint32_t kYSlot = 32 * 64;     // epilogue transpose slot: 32 rows x 64 B (half a 128-byte row chunk)
#ifndef VNM_TC3_EPI
#define VNM_TC3_EPI 8
#endif
constexpr int kEpi = VNM_TC3_EPI;        // epilogue warps (a multiple of 4: kEpi / 4 per TMEM lane quadrant)
constexpr int kEq = kEpi / 4;
constexpr int kThreads = 128 + 32 * kEpi;  // warps 0 + 2 TMA, 1 MMA, 3 idle, 4.. epilogue
#ifndef VNM_TC3_EARLY
#define VNM_TC3_EARLY 0
#endif
constexpr bool kEarlyRelease = VNM_TC3_EARLY != 0;  // two accumulators too: release before the stores (experiment)

struct Tc3Args {
    int32_t T, M;
    int32_t n_mma;       // MMAs per tile (K direction)
    int32_t n_chunk;     // 4-MMA chunks of A / metadata = ceil(n_mma / 4)
    int32_t ms;          // MMAs per ring stage (2 or 4; 4 when A streams)
    int32_t n_st;        // ring stages per tile = ceil(n_mma / ms)
    int32_t rows_stage;  // X^T rows per stage
    int32_t n_rt, n_rp, n_tt;
    int32_t S;           // ring slots
    int32_t a_res;       // 1: A + metadata resident; 0: streamed per stage
    int32_t rp_per;      // resident: pairs per row pair;  streaming: total pairs
    int32_t peek;        // windows cross stage boundaries (5 <= M <= 7: an 8-channel window is wider than a block)
    int32_t ts_direct;   // with ts: A goes global -> registers -> TMEM (tcgen05.st by the epilogue warps at the start),
                         // never through shared memory, whose A space becomes more X^T ring slots
    const uint16_t* values_tc;
    int32_t ld_tc;
    int32_t ts;          // 1: resident A copied once into TMEM (tcgen05.cp) and the MMAs read it from there (TS form);
                         // NT = 256 (one accumulator) only: TMEM = accumulator | A (32 columns per chunk) | metadata
    int32_t ovh;         // 1: every slot also holds the next stage's first 8 rows (loaded twice; no cross-stage
                         // wait, no shadow); 0: K-ring with the MMA waiting for the next stage too
    int32_t slot_rows;   // rows per slot: rows_stage (+ 8 with ovh and peek)
    uint32_t ring_rows;  // S * slot_rows (+ 8 shadow rows without ovh): rows per token-chunk region
    uint32_t stage_tx, shadow_tx;  // expect_tx bytes for both CTAs (X^T; + A / metadata when streaming)
    void* Y;
    int64_t ldy;
    int32_t rows;
    int32_t trace;
    int32_t abl;  // VNM_ABL timing ablations (results invalid): 1 no epilogue, 2 no Y stores, 4 no
                  // loads at all, 16 no A / metadata loads (streaming), 32 no X^T loads
};

__device__ unsigned long long g_tc3_t[9][160];
// timing-ablation flags (VNM_ABL): a compile-time 0 in production builds, so no ablation test is left in the loops;
// the general MMA loop runs for the MMA-issue ablations
#ifdef VNM_ABLATIONS
#define ABL(args) ((args).abl)
#else
#define ABL(args) 0
#endif
#define VNM_ABLATION_FLAGS_DEVICE(args) (ABL(args) & (64 | 128))

// tile i of this pair; false past the end.  Resident A: every pair owns one row pair and the row pair's token
// tiles are dealt round-robin over its pairs.  Streaming: tiles row-pair-major over all pairs (consecutive
// pairs share a row pair's A in L2).
__device__ __forceinline__ bool tile3(const Tc3Args& a, int cid, int i, int& rp, int& tt) {
    if (a.a_res) {
        rp = cid % a.n_rp;
        tt = cid / a.n_rp + i * a.rp_per;
        return tt < a.n_tt;
    }
    const int w = cid + i * a.rp_per;
    rp = w / a.n_tt;
    tt = w % a.n_tt;
    return rp < a.n_rp;
}

template <int NT, bool kBf16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    vnm_spmm_tc3_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_e,
                        const __grid_constant__ CUtensorMap tmap_b0, const __grid_constant__ CUtensorMap tmap_b1,
                        const __grid_constant__ CUtensorMap tmap_s0, const __grid_constant__ CUtensorMap tmap_s1,
                        const Tc3Args a) {
    constexpr int kNH = NT / 2;                    // tokens per CTA of B
    constexpr int kW1 = kNH - 64;                  // width of the second token box
    constexpr int kNacc = NT == 256 ? 1 : 2;       // accumulators in TMEM
    constexpr uint32_t kMetaCol = kNacc * NT;      // metadata columns after the accumulators
    constexpr int kCw = kBf16 ? 64 : 32;           // tokens per 128-byte row of a transpose slot
    constexpr int kNch = (NT + kCw - 1) / kCw;     // epilogue chunks per tile
    constexpr int kCpw = (kNch + kEq - 1) / kEq;   // chunks per epilogue warp (kEq warps per lane quadrant)
    static_assert(kW1 > 0 && kW1 <= 64 && kW1 % 16 == 0, "token split");
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = a.S;
    const int na = a.a_res ? (a.ts_direct ? 0 : a.n_chunk) : S;  // A chunks held in shared memory (resident: all;
                                                                 // streaming: one per slot; A straight to TMEM: none)
    // [A: na x 16 KB][E: na x 2 KB, padded to 1 KB (unless aliased)][X^T ring: 2 token chunks x ring_rows x 128 B]
    // [transpose slots: kEpi x 2 KB][barriers]
    // (resident mode: the metadata staging aliases the epilogue slots — it is read once by tcgen05.cp before the
    // first MMA, and the epilogue first touches the slots after that tile's MMAs, i.e. after the copies, completed)
    const bool e_alias = a.a_res && a.n_chunk * kEBytes <= kEpi * kYSlot;
    uint8_t* sA = smem;
    uint8_t* ring = smem + na * kABytes + (e_alias ? 0u : (na * kEBytes + 1023) / 1024 * 1024);
    const uint32_t region = a.ring_rows * 128u;  // bytes per token-chunk region
    uint8_t* sY = ring + 2 * region;
    uint8_t* sE = e_alias ? sY : smem + na * kABytes;  // (ts_direct requires e_alias: checked on the host)
    uint64_t* full = reinterpret_cast<uint64_t*>(sY + kEpi * kYSlot);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;       // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint64_t* res_full = tmem_empty + 2;
    uint64_t* a_ready = res_full + 1;  // ts_direct: every epilogue warp of both CTAs has stored its A rows in TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_ready + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = static_cast<int>(cluster_id_x());

    // zero the ring once: window positions outside their block read it (times zero values); must be finite
    {
        uint4* r = reinterpret_cast<uint4*>(ring);
        const uint32_t n16 = 2 * region / 16;
        for (uint32_t i = threadIdx.x; i < n16; i += kThreads) r[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 2 * kEpi);  // epilogue warps x 2 CTAs
        }
        mbar_init(res_full, 1);
        mbar_init(a_ready, 2 * kEpi);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_e);
        tma_prefetch_desc(&tmap_b0);
        tma_prefetch_desc(&tmap_b1);
        tma_prefetch_desc(&tmap_s0);
        tma_prefetch_desc(&tmap_s1);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_wait();    // the previous kernel's outputs (e.g. this layer's inputs) are visible
    grid_dep_launch();  // the next kernel may take SMs as this grid's CTAs exit

    if (warp == 0 || warp == 2) {
        // ------------------------------------------------------------ TMA producers (both CTAs): warp 0 the
        // A / metadata, the expect_tx and the 64-token box, warp 2 the second box
        const int pb = warp / 2;
        if (lane == 0) {
            int q = 0, rp, tt;
            unsigned long long c_emp = 0, c0;
            for (int i = 0; tile3(a, cid, i, rp, tt); ++i) {
                const int rt = 2 * rp + static_cast<int>(rank);  // row tiles past n_rt read as zeros (TMA OOB)
                const int rte = rt < a.n_rt ? rt : 0;             // ... with valid metadata
                if (a.a_res && i == 0 && pb == 0) {  // the pair's A and metadata, once
                    if (leader) mbar_arrive_expect_tx(res_full, 2 * a.n_chunk * ((a.ts_direct ? 0u : kABytes) + kEBytes));
                    for (int c = 0; c < a.n_chunk; ++c) {
                        if (!a.ts_direct) tma_load_2d_pair(sA + c * kABytes, &tmap_a, c * 64, rt * 128, res_full);
                        tma_load_2d_pair(sE + c * kEBytes, &tmap_e, 0, (rte * a.n_chunk + c) * 128, res_full);
                    }
                }
                const int x0 = tt * NT + kNH * static_cast<int>(rank);
                for (int st = 0; st < a.n_st; ++st, ++q) {
                    const int s = q % S;
                    if (a.trace) c0 = clock64();
                    mbar_wait(&empty[s], ((q / S) & 1) ^ 1);
                    if (a.trace) c_emp += clock64() - c0;
                    if (ABL(a) & 4) {
                        if (leader && pb == 0) mbar_arrive(&full[s]);
                        continue;
                    }
                    // (box 1's bytes may land before box 0's thread registers the stage's expect_tx: the
                    // phase still needs that arrival, and the transaction count is signed)
                    if (pb == 0) {
                        uint32_t tx = a.stage_tx + (s == 0 && !a.ovh ? a.shadow_tx : 0u);
                        if (ABL(a) & 16) tx -= 2u * (kABytes + kEBytes);                  // ablation: no A / E loads
                        if (ABL(a) & 32) tx = a.a_res ? 0u : 2u * (kABytes + kEBytes);    // ablation: no X^T loads
                        if (leader) {
                            if (tx) mbar_arrive_expect_tx(&full[s], tx);
                            else mbar_arrive(&full[s]);
                        }
                        if (!a.a_res && !(ABL(a) & 16)) {  // this stage's A / metadata chunk (ms = 4: stage == chunk)
                            tma_load_2d_pair(sA + s * kABytes, &tmap_a, st * 64, rt * 128, &full[s]);
                            tma_load_2d_pair(sE + s * kEBytes, &tmap_e, 0, (rte * a.n_chunk + st) * 128, &full[s]);
                        }
                    }
                    if (ABL(a) & 32) continue;
                    const int y = st * a.rows_stage;
                    uint8_t* dst = ring + static_cast<uint32_t>(s * a.slot_rows) * 128u + pb * region;
                    tma_load_2d_pair(dst, pb ? &tmap_b1 : &tmap_b0, x0 + 64 * pb, y, &full[s]);
                    if (s == 0 && a.peek && !a.ovh) {  // the shadow after the last slot: a copy of slot 0's first 8 rows
                        uint8_t* sh = ring + static_cast<uint32_t>(S * a.rows_stage) * 128u + pb * region;
                        tma_load_2d_pair(sh, pb ? &tmap_s1 : &tmap_s0, x0 + 64 * pb, y, &full[s]);
                    }
                }
            }
            if (a.trace && pb == 0) g_tc3_t[3][blockIdx.x] = c_emp;
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader; converged warp)
        if (leader) {
            int q = 0, tl = 0, rp, tt;
            const uint32_t idesc0 = idesc_bf16(256, NT, true, 0, true);
            const uint32_t idesc1 = idesc_bf16(256, NT, true, 1, true);
            const uint64_t b_step = (a.M == 4 ? 32u : 4u * a.M) * 128u >> 4;  // B descriptor advance per MMA
            const uint32_t sbo = a.M == 4 ? 1024u : a.M * 128u;                 // K-group (window) stride
            const uint32_t meta_col = a.ts ? NT + 32u * a.n_chunk : kMetaCol;   // metadata after A in the TS form
            unsigned long long c_full = 0, c_emp = 0, c_all = clock64(), c0, c_full0 = 0;
            // The production loop, specialised per mode (RES: A + metadata resident; TS: A read from TMEM) with
            // nothing else in it.  The general loop below (kept for VNM_SPMM_TRACE, the opt-out K-ring peek and the
            // MMA ablations) ran the MMA-only skeleton of DeiT-S qkv 1.6x slower per MMA for the same MMAs; no
            // single feature of it accounts for that (bisected: profiles/r02_experiments.md, round-2 re-entry).
            auto mma_loop = [&](auto res_c, auto ts_c) {
                constexpr bool RES = decltype(res_c)::value, TS = decltype(ts_c)::value;
                if constexpr (RES) {
                    mbar_wait(res_full, 0);  // resident metadata (and A for TS) -> TMEM, both CTAs
                    tc_fence_after();
                    for (int c = 0; c < a.n_chunk; ++c)
                        tmem_cp_elect<2>(tmem + meta_col + 4 * c, sdesc(smem_u32(sE + c * kEBytes), 16, 128, 0));
                    if constexpr (TS) {
                        if (a.ts_direct) {  // the epilogue warps store A into TMEM themselves
                            mbar_wait(a_ready, 0);
                            tc_fence_after();
                        } else {
                            for (int c = 0; c < a.n_chunk; ++c)
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    tmem_cp256_elect<2>(tmem + NT + 32 * c + 8 * i,
                                                        sdesc(smem_u32(sA + c * kABytes), 16, 1024, kLayoutSW128) + 2 * i);
                        }
                    }
                }
                const uint64_t a_base = sdesc(smem_u32(sA), 16, 1024, kLayoutSW128);
                for (; tile3(a, cid, tl, rp, tt); ++tl) {
                    const int acc = kNacc == 2 ? (tl & 1) : 0;
                    const int use = kNacc == 2 ? (tl >> 1) : tl;
                    mbar_wait(&tmem_empty[acc], (use & 1) ^ 1);
                    tc_fence_after();
                    for (int st = 0; st < a.n_st; ++st, ++q) {
                        const int s = q % S;
                        mbar_wait(&full[s], (q / S) & 1);
                        tc_fence_after();
                        const int mi0 = st * a.ms;
                        const int left = a.n_mma - mi0;
                        const uint32_t n = static_cast<uint32_t>(left < a.ms ? left : a.ms);
                        const uint64_t bd =
                            sdesc(smem_u32(ring + static_cast<uint32_t>(s * a.slot_rows) * 128u), region, sbo, kLayoutSW128);
                        if constexpr (RES) {
                            const uint32_t e = tmem + meta_col + 4 * (mi0 >> 2) + (mi0 & 2);
                            if constexpr (TS)
                                mma_sp_stage_ts_pair(tmem + acc * NT, tmem + NT + 8 * mi0, bd, b_step, e, idesc0, idesc1,
                                                     st > 0 ? 1u : 0u, n);
                            else
                                mma_sp_stage<2>(tmem + acc * NT, a_base + (((mi0 >> 2) * kABytes) >> 4) + 2 * (mi0 & 3), bd,
                                                b_step, e, idesc0, idesc1, st > 0 ? 1u : 0u, n);
                        } else {  // this slot's chunk: metadata into the slot's TMEM columns first (tensor-pipe order)
                            const uint32_t e = tmem + meta_col + 4 * s;
                            tmem_cp_elect<2>(e, sdesc(smem_u32(sE + s * kEBytes), 16, 128, 0));
                            mma_sp_stage<2>(tmem + acc * NT, a_base + ((s * kABytes) >> 4), bd, b_step, e, idesc0, idesc1,
                                            st > 0 ? 1u : 0u, n);
                        }
                        mma_commit_pair_elect(&empty[s], 0x3);
                    }
                    mma_commit_pair_elect(&tmem_full[acc], 0x3);
                }
            };
#ifdef VNM_TC3_TRACE_FAST  // (experiment builds: the specialised loop under VNM_SPMM_TRACE too; its own counters stay 0)
            if (!(a.peek && !a.ovh) && !VNM_ABLATION_FLAGS_DEVICE(a)) {
#else
            if (!a.trace && !(a.peek && !a.ovh) && !VNM_ABLATION_FLAGS_DEVICE(a)) {
#endif
                if (a.a_res) {
                    if (a.ts) mma_loop(std::true_type{}, std::true_type{});
                    else mma_loop(std::true_type{}, std::false_type{});
                } else {
                    mma_loop(std::false_type{}, std::false_type{});
                }
                tl = 1 << 30;
            }
            for (; tl < (1 << 30) && tile3(a, cid, tl, rp, tt); ++tl) {
                if (a.a_res && tl == 0) {  // resident metadata -> TMEM columns meta_col + 4c (both CTAs)
                    mbar_wait(res_full, 0);
                    tc_fence_after();
                    for (int c = 0; c < a.n_chunk; ++c)
                        tmem_cp_elect<2>(tmem + meta_col + 4 * c, sdesc(smem_u32(sE + c * kEBytes), 16, 128, 0));
                    if (a.ts && a.ts_direct) {
                        mbar_wait(a_ready, 0);
                        tc_fence_after();
                    } else if (a.ts)  // resident A -> TMEM columns NT + 8 mi (MMA mi's 128 rows x 16 compressed values)
                        for (int c = 0; c < a.n_chunk; ++c)
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                tmem_cp256_elect<2>(tmem + NT + 32 * c + 8 * i,
                                                    sdesc(smem_u32(sA + c * kABytes), 16, 1024, kLayoutSW128) + 2 * i);
                }
                const int acc = kNacc == 2 ? (tl & 1) : 0;
                const int use = kNacc == 2 ? (tl >> 1) : tl;  // uses of this accumulator so far
                // (the wait counters read the clock only when tracing)
                if (a.trace) c0 = clock64();
                mbar_wait(&tmem_empty[acc], (use & 1) ^ 1);
                if (a.trace) c_emp += clock64() - c0;
                tc_fence_after();
                for (int st = 0; st < a.n_st; ++st, ++q) {
                    const int s = q % S;
                    if (a.trace) c0 = clock64();
                    mbar_wait(&full[s], (q / S) & 1);
                    if (a.peek && !a.ovh && st + 1 < a.n_st) mbar_wait(&full[(q + 1) % S], ((q + 1) / S) & 1);  // overhang
                    if (a.trace) {
                        c_full += clock64() - c0;
                        if (st == 0) c_full0 += clock64() - c0;
                    }
                    tc_fence_after();
                    const int mi0 = st * a.ms;
                    const int left = a.n_mma - mi0;
                    const uint32_t n = static_cast<uint32_t>(left < a.ms ? left : a.ms);
                    const uint64_t bd =
                        sdesc(smem_u32(ring + static_cast<uint32_t>(s * a.slot_rows) * 128u), region, sbo, kLayoutSW128);
                    uint64_t ad;
                    uint32_t e;
                    if (a.a_res) {
                        ad = sdesc(smem_u32(sA + (mi0 >> 2) * kABytes), 16, 1024, kLayoutSW128) + 2 * (mi0 & 3);
                        e = tmem + meta_col + 4 * (mi0 >> 2) + (mi0 & 2);
                    } else {  // this slot's chunk: metadata into the slot's TMEM columns first (tensor-pipe order)
                        e = tmem + meta_col + 4 * s;
                        tmem_cp_elect<2>(e, sdesc(smem_u32(sE + s * kEBytes), 16, 128, 0));
                        ad = sdesc(smem_u32(sA + s * kABytes), 16, 1024, kLayoutSW128);
                    }
                    if (a.ts)
                        mma_sp_stage_ts_pair(tmem + acc * NT, tmem + NT + 8 * mi0, bd, b_step, e, idesc0, idesc1,
                                             st > 0 ? 1u : 0u, n);
#ifdef VNM_ABLATIONS
                    else if (a.abl & 64)  // every MMA of the stage reads the stage's first A slice (timing only)
                        mma_sp_stage_astep_pair(tmem + acc * NT, ad, 0, bd, b_step, e, idesc0, idesc1, st > 0 ? 1u : 0u, n);
                    else if (a.abl & 128)  // the same issue code with the normal A offsets (control)
                        mma_sp_stage_astep_pair(tmem + acc * NT, ad, 2, bd, b_step, e, idesc0, idesc1, st > 0 ? 1u : 0u, n);
#endif
                    else
                        mma_sp_stage<2>(tmem + acc * NT, ad, bd, b_step, e, idesc0, idesc1, st > 0 ? 1u : 0u, n);
                    mma_commit_pair_elect(&empty[s], 0x3);
                }
                mma_commit_pair_elect(&tmem_full[acc], 0x3);
            }
            if (a.trace && lane == 0 && tl < (1 << 30)) {
                g_tc3_t[0][blockIdx.x] = c_full;
                g_tc3_t[1][blockIdx.x] = c_emp;
                g_tc3_t[2][blockIdx.x] = clock64() - c_all;
                g_tc3_t[7][blockIdx.x] = tl;
                g_tc3_t[8][blockIdx.x] = c_full0;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue (both CTAs)
        // warp 4 + qd + 4h: TMEM lanes 32qd.. (rows 32qd.. of the CTA's row tile), token chunks c = h, h + 2, ..
        // of kCw tokens: TMEM -> registers (-> bf16) -> the warp's transpose slot (SW128: chunk k of row r at
        // k ^ (r % 8), conflict-free) -> read back 4 rows x 8 chunks per instruction -> st.global.v4 of whole
        // 128-byte lines (no TMA, no proxy fence); rows >= rows / tokens >= T are not stored.
        const int qd = (warp - 4) % 4, half = (warp - 4) / 4;
        uint8_t* slot = sY + (warp - 4) * kYSlot;
        const uint32_t srow = smem_u32(slot);
        int tl = 0, rp, tt;
        unsigned long long c_wait = 0, c_epi = 0, c0, c1;
        // TMEM -> 32 packed words (one 128-byte row chunk per lane)
        auto drain = [&](uint32_t taddr, int c, uint32_t (&w)[32]) {
            if constexpr (kBf16) {
                uint32_t v[64];
                tmem_ld_32x32b_x32(taddr + c * 64, v);
                tmem_ld_32x32b_x32(taddr + c * 64 + 32, v + 32);  // past NT: other columns, never stored
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                    w[k] = *reinterpret_cast<uint32_t*>(&b2);
                }
            } else {
                tmem_ld_32x32b_x32(taddr + c * 32, w);
                tmem_wait_ld();
            }
        };
        // the same in two halves: TMEM loads issued (no wait), then wait + pack — so the loads of chunk c + kEq run
        // under the stores of chunk c
        auto ld_issue = [&](uint32_t taddr, int c, uint32_t (&v)[64]) {
            if constexpr (kBf16) {
                tmem_ld_32x32b_x32(taddr + c * 64, v);
                tmem_ld_32x32b_x32(taddr + c * 64 + 32, v + 32);  // past NT: other columns, never stored
            } else {
                tmem_ld_32x32b_x32(taddr + c * 32, v);
            }
        };
        auto ld_finish = [&](const uint32_t (&v)[64], uint32_t (&w)[32]) {
            tmem_wait_ld();
            if constexpr (kBf16) {
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                    w[k] = *reinterpret_cast<uint32_t*>(&b2);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) w[k] = v[k];
            }
        };
        auto release = [&](int acc) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(&tmem_empty[acc]);
                else mbar_arrive_remote(&tmem_empty[acc], 0);
            }
        };
        auto store = [&](int rt, int c, const uint32_t (&w)[32]) {
            const int t0 = tt * NT + c * kCw;
            if (rt >= a.n_rt || t0 >= a.T || (ABL(a) & 2)) return;
            constexpr int kEl = kBf16 ? 8 : 4;  // elements per 16 bytes
            const int t_end = min(a.T, tt * NT + NT);
            const int grow0 = rt * 128 + 32 * qd;
            // two halves of 64 B per row (the slot holds 32 rows x 64 B: chunk k of row r at k ^ ((r / 2) % 4),
            // conflict-free both ways); read back 8 rows x 4 chunks per instruction
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int th = t0 + h2 * (kCw / 2);
                if (th >= t_end) break;
                __syncwarp();  // the previous reads of the slot are done
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(srow + lane * 64 + (((k ^ (lane >> 1)) & 3) << 4)),
                                 "r"(w[16 * h2 + 4 * k]), "r"(w[16 * h2 + 4 * k + 1]), "r"(w[16 * h2 + 4 * k + 2]),
                                 "r"(w[16 * h2 + 4 * k + 3])
                                 : "memory");
                __syncwarp();
                const int cc = lane & 3, tok = th + cc * kEl;
                // the four shared-memory reads first (volatile asm keeps its order: interleaved with the stores, each
                // read's latency was exposed once per row group), then the four global stores
                uint32_t xr[4][4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = 8 * j + (lane >> 2);
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(xr[j][0]), "=r"(xr[j][1]), "=r"(xr[j][2]), "=r"(xr[j][3])
                                 : "r"(srow + r * 64 + (((cc ^ (r >> 1)) & 3) << 4)));
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = 8 * j + (lane >> 2);
                    const uint32_t x0 = xr[j][0], x1 = xr[j][1], x2 = xr[j][2], x3 = xr[j][3];
                    const int grow = grow0 + r;
                    if (grow >= a.rows || tok >= t_end) continue;
                    uint8_t* dst = static_cast<uint8_t*>(a.Y) + (static_cast<int64_t>(grow) * a.ldy + tok) * (kBf16 ? 2 : 4);
                    if (tok + kEl <= t_end) {
                        asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(x0), "r"(x1), "r"(x2), "r"(x3)
                                     : "memory");
                    } else {  // ragged token tail: element by element
                        const uint32_t xs[4] = {x0, x1, x2, x3};
                        for (int e = 0; e < t_end - tok; ++e) {
                            if constexpr (kBf16)
                                reinterpret_cast<uint16_t*>(dst)[e] = static_cast<uint16_t>(xs[e >> 1] >> (16 * (e & 1)));
                            else
                                reinterpret_cast<uint32_t*>(dst)[e] = xs[e];
                        }
                    }
                }
            }
        };
        if (a.ts_direct) {
            // A straight into TMEM (TS form): this warp's 32 rows (its lane quadrant), chunks half, half + kEq, ..:
            // MMA mi's 16 values of a row (32 bytes of values_tc) -> TMEM columns NT + 8 mi .. + 7 of its lane, in
            // order (the layout tcgen05.cp 128x256b produces from the SW128 tile); row tiles past n_rt get zeros
            int rp0 = 0, tt0 = 0;
            const bool any = tile3(a, cid, 0, rp0, tt0);
            const int rt0 = 2 * rp0 + static_cast<int>(rank);
            const bool real = any && rt0 < a.n_rt;
            const uint4* vrow = reinterpret_cast<const uint4*>(a.values_tc + static_cast<int64_t>(rt0 * 128 + 32 * qd + lane) * a.ld_tc);
            const uint32_t tbase = tmem + ((32 * qd) << 16) + NT;
            for (int c = half; c < a.n_chunk; c += kEq) {
                uint4 x[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)  // (a row holds 2 x n_mma of these 16-byte groups)
                    x[i] = real && 8 * c + i < 2 * a.n_mma ? __ldg(vrow + 8 * c + i) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int i = 0; i < 8; ++i) tmem_st_32x32b_x4(tbase + 32 * c + 4 * i, x[i].x, x[i].y, x[i].z, x[i].w);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(a_ready);
                else mbar_arrive_remote(a_ready, 0);
            }
        }
        for (; tile3(a, cid, tl, rp, tt); ++tl) {
            const int rt = 2 * rp + static_cast<int>(rank);
            const int acc = kNacc == 2 ? (tl & 1) : 0;
            const int use = kNacc == 2 ? (tl >> 1) : tl;
            if (a.trace) c0 = clock64();
            mbar_wait(&tmem_full[acc], use & 1);
            if (a.trace) {
                c1 = clock64();
                c_wait += c1 - c0;
            }
            tc_fence_after();
            const uint32_t taddr = tmem + ((32 * qd) << 16) + acc * NT;
            if (ABL(a) & 1) {
                release(acc);
                continue;
            }
            if constexpr (kNacc == 1 || kEarlyRelease) {
                // drain this warp's chunks into registers, release, then store (one accumulator; with two only when
                // kEarlyRelease: measured, the stores then never hold an accumulator)
                uint32_t w[kCpw][32];
#pragma unroll
                for (int j = 0; j < kCpw; ++j)
                    if (half + kEq * j < kNch) drain(taddr, half + kEq * j, w[j]);
                release(acc);
#pragma unroll
                for (int j = 0; j < kCpw; ++j)
                    if (half + kEq * j < kNch) store(rt, half + kEq * j, w[j]);
            } else {
                const int last = half < kNch ? ((kNch - 1 - half) / kEq) * kEq + half : -1;  // this warp's last chunk
                if (last < 0) release(acc);  // no chunk for this warp in this tile
                uint32_t v[64], w[32];
                if (half < kNch) ld_issue(taddr, half, v);
#pragma unroll 1
                for (int c = half; c < kNch; c += kEq) {
                    ld_finish(v, w);
                    if (c == last) release(acc);
                    else ld_issue(taddr, c + kEq, v);  // the next chunk's TMEM loads under this chunk's stores
                    store(rt, c, w);
                }
            }
            if (a.trace) c_epi += clock64() - c1;
        }
        if (a.trace && warp == 4 && lane == 0) {
            g_tc3_t[4][blockIdx.x] = c_wait;
            g_tc3_t[5][blockIdx.x] = c_epi;
        }
    }
    tc_fence_before();
    cluster_sync_all();  // the peer's remote arrivals / the leader's reads of peer shared memory are done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

template <int NT>
int launch_nt3(const SpmmLaunch& L, Tc3Args a, int want_res, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    constexpr int kNH = NT / 2, kW1 = kNH - 64, kNacc = NT == 256 ? 1 : 2;
    a.n_tt = (L.T + NT - 1) / NT;
    const uint32_t fixed = kEpi * kYSlot + 1024;
    auto ebytes = [](int n) { return static_cast<uint32_t>(n * kEBytes + 1023) / 1024 * 1024; };
    const int pairs_all = num_sms() / 2;
    // resident A when the row pair's A + metadata fit next to >= 4 ring slots and every row pair gets a pair
    const bool alias = a.n_chunk * kEBytes <= kEpi * kYSlot;  // resident metadata staged in the epilogue slots
    const uint32_t res = static_cast<uint32_t>(a.n_chunk) * kABytes + (alias ? 0u : ebytes(a.n_chunk));
    a.a_res = want_res != 0 && pairs_all >= a.n_rp && kNacc * NT + 4 * a.n_chunk <= 512 &&
              res + 2u * (4 * a.slot_rows + 8) * 128u + fixed <= kMaxSmem;
    if (want_res == 1 && !a.a_res) return kLaunchUnsupported;
    if (!a.a_res && a.ms != 4) return kLaunchUnsupported;  // streamed A arrives in 4-MMA chunks
    // TS form: resident A and one accumulator, TMEM = NT + 32 columns per A chunk + 4 per metadata chunk
    if (!a.a_res || kNacc != 1 || NT + 36 * a.n_chunk > 512) a.ts = 0;
    // TS form with A stored into TMEM by the epilogue warps (no shared-memory copy of A: its space becomes ring
    // slots); VNM_TC3_TS_STAGED=1 keeps the shared-memory staging + tcgen05.cp
    a.ts_direct = a.ts && alias && VNM_ENV_INT("VNM_TC3_TS_STAGED", 0) == 0 ? 1 : 0;
    const uint32_t res_smem = a.ts_direct ? 0u : res;
    // ring slots: as many as fit (bytes in flight hide the load latency), at least 3
    int S = 0;
    for (int s = 10; s >= 3 && !S; --s) {
        const uint32_t ab = a.a_res ? res_smem : static_cast<uint32_t>(s) * kABytes + ebytes(s);
        const bool tmem_ok = kNacc * NT + 4 * (a.a_res ? a.n_chunk : s) <= 512;
        if (tmem_ok && ab + 2u * (s * a.slot_rows + 8) * 128u + fixed <= kMaxSmem) S = s;
    }
    if (!S) return kLaunchUnsupported;
    if (const int v = VNM_ENV_INT("VNM_TC3_S", 0); v >= 3 && v < S) S = v;
    a.S = S;
    a.ring_rows = static_cast<uint32_t>(S * a.slot_rows + (a.ovh ? 0 : 8));
    a.stage_tx = 2u * a.slot_rows * (64 + kW1) * 2u + (a.a_res ? 0u : 2u * (kABytes + kEBytes));
    a.shadow_tx = a.peek ? 2u * 8u * (64 + kW1) * 2u : 0u;
    int pairs;
    if (a.a_res) {  // every pair owns one row pair; the token tiles of a row pair are dealt round-robin
        a.rp_per = pairs_all / a.n_rp;
        if (a.rp_per > a.n_tt) a.rp_per = a.n_tt;
        pairs = a.rp_per * a.n_rp;
    } else {
        pairs = pairs_all < a.n_rp * a.n_tt ? pairs_all : a.n_rp * a.n_tt;
        a.rp_per = pairs;
    }

    CUtensorMap ta, te, tb0, tb1, ts0, ts1;
    const int ld_tc = 16 * a.n_mma;
    if (!encode_2d(&ta, L.P->values_tc, static_cast<uint64_t>(ld_tc), static_cast<uint64_t>(a.n_rt) * 128,
                   static_cast<uint64_t>(ld_tc) * 2, 64, 128))
        return kLaunchCudaError;
    if (!encode_2d(&te, L.P->meta_tc, 4, static_cast<uint64_t>(a.n_rt) * a.n_chunk * 128, 16, 4, 128,
                   CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    const uint64_t xr = static_cast<uint64_t>(L.ldx) * 2;
    if (!encode_2d(&tb0, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, 64,
                   static_cast<uint32_t>(a.slot_rows)) ||
        !encode_2d(&tb1, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, kW1,
                   static_cast<uint32_t>(a.slot_rows)) ||
        !encode_2d(&ts0, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, 64, 8) ||
        !encode_2d(&ts1, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, kW1, 8))
        return kLaunchCudaError;
    const bool bf = L.y_dtype == VNM_BF16;
    const int na = a.a_res ? (a.ts_direct ? 0 : a.n_chunk) : S;  // (as the kernel's layout)
    const size_t smem = static_cast<size_t>(na) * kABytes + (a.a_res && alias ? 0u : ebytes(na)) +
                        2u * a.ring_rows * 128u + fixed;
    auto k = bf ? vnm_spmm_tc3_kernel<NT, true> : vnm_spmm_tc3_kernel<NT, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return kLaunchCudaError;
    a.trace = VNM_ENV_INT("VNM_SPMM_TRACE", 0) ? 1 : 0;
    a.abl = VNM_ABLATION_FLAGS();
    a.Y = L.YT;
    a.ldy = L.ldy;
    a.rows = g.rows;
    a.values_tc = L.P->values_tc;
    a.ld_tc = ld_tc;
    cudaError_t e = launch_pdl(false, k, dim3(2 * pairs), dim3(kThreads), smem, stream, ta, te, tb0, tb1, ts0, ts1, a);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess && a.trace) {
        static unsigned long long h[9][160];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(h, g_tc3_t, sizeof(h));
        fprintf(stderr, "tc3 NT=%d: grid %d a_res %d S %d ms %d n_st %d n_mma %d smem %zu\n", NT, 2 * pairs, a.a_res,
                a.S, a.ms, a.n_st, a.n_mma, smem);
        for (int i = 0; i < 2 * pairs; i += 10)
            fprintf(stderr, "  cta %3d tiles %llu | mma: wait_full %7llu (stage 0: %7llu) wait_empty %7llu total %8llu | "
                            "prod wait %8llu | epi wait %8llu busy %8llu\n", i, h[7][i], h[0][i], h[8][i], h[1][i], h[2][i],
                    h[3][i], h[4][i], h[5][i]);
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

// Window form, 4 <= M <= 8, T > 64.  mode: 1 resident A only, 0 streamed A only, -1 resident when it fits.
// kLaunchUnsupported when the configuration does not fit (the caller then uses the tc / tc2 kernels).
int launch_spmm_tc3(const SpmmLaunch& L, int mode, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (g.M > 8 || g.M < 4) return kLaunchUnsupported;
    Tc3Args a;
    a.T = L.T;
    a.M = g.M;
    a.n_mma = g.nb_pad / (g.M == 4 ? 8 : 4);
    a.n_chunk = (a.n_mma + 3) / 4;
    a.n_rt = (g.rows_p + 127) / 128;
    a.n_rp = (a.n_rt + 1) / 2;
    a.peek = g.M >= 5 && g.M <= 7;
    a.ovh = VNM_ENV_INT("VNM_TC3_OVH", 1) ? 1 : 0;
    a.ts = 0;
    a.ts_direct = 0;
    a.values_tc = nullptr;
    a.ld_tc = 0;
    const int res = mode < 0 ? 1 : mode;
    // resident A: 4 MMAs per stage (16 blocks), 2 when a 4-MMA stage would be large (M >= 7: >= 112 rows)
    a.ms = g.M >= 7 && res ? 2 : 4;
    if (const int v = VNM_ENV_INT("VNM_TC3_MS", 0)) a.ms = v == 2 ? 2 : 4;
    a.n_st = (a.n_mma + a.ms - 1) / a.ms;
    a.rows_stage = a.ms * (g.M == 4 ? 32 : 4 * g.M);
    a.slot_rows = a.rows_stage + (a.ovh && a.peek ? 8 : 0);
    // NT = 256 (one accumulator) when T is a multiple of 256 and A streams (long K: the per-tile hand-off is
    // amortised), else NT = 224 (two accumulators)
    int nt = (mode == 0 && L.T % 256 == 0) ? 256 : 224;
    // opt-in (VNM_TC3_TS=1): resident A in TMEM (TS form, one accumulator, NT = 256) — the MMAs stop reading A
    // from shared memory; parity-tested, but measured no faster in the bench's cold steps (warm: ~3 %), so off by
    // default (profiles/r02_experiments.md)
    if (mode != 0 && L.T % 256 == 0 && VNM_ENV_INT("VNM_TC3_TS", 0) && 256 + 36 * a.n_chunk <= 512) {
        nt = 256;
        a.ts = 1;
    }
    if (const int v = VNM_ENV_INT("VNM_TC3_NT", 0)) nt = v;
    const int want = mode < 0 ? -1 : res;
    auto launch = [&](int w) {
        return nt == 256 ? launch_nt3<256>(L, a, w, stream) : nt == 192 ? launch_nt3<192>(L, a, w, stream)
                                                                    : launch_nt3<224>(L, a, w, stream);
    };
    int rc = launch(want);
    if (rc == kLaunchUnsupported && mode < 0 && a.ms != 4) {  // resident did not fit: stream, 4-MMA stages
        a.ms = 4;
        a.n_st = (a.n_mma + 3) / 4;
        a.rows_stage = 4 * (g.M == 4 ? 32 : 4 * g.M);
        a.slot_rows = a.rows_stage + (a.ovh && a.peek ? 8 : 0);
        rc = launch(0);
    }
    return rc;
}

}  // namespace vnm
