// spmm_tc2.cu — the window-form V:N:M SpMM (include/vnm.h values_tc / meta_tc) on CTA
// PAIRS: tcgen05.mma.sp.cta_group::2 with M = 256, N = 256.
//
// Why pairs.  A 1-CTA M = 128, N = 256 sparse MMA reads A (4 KB) and the whole B tile (16 KB) from one SM's
// shared memory per 128 x 256 x 16 effectual MACs; the measured back-to-back cost (~165 cycles,
// profiles/r01_probes.md MB2) is the shared-memory read rate (~124 B/clk), so any TMA or epilogue traffic
// in the same shared memory slows the MMAs down.  In a pair each CTA holds its own 128 rows of A and only
// HALF of the B tile (128 tokens), and the two SMs' tensor cores execute the M = 256 product together:
// 12 KB of shared memory per CTA per MMA instead of 20 KB, and every X^T tile is fetched from L2 once per
// 256 output rows.  Rows are independent in the window form (each row carries its own 2:4 metadata over
// the block's 8-channel window), so any V works as long as the window form was built for it.
//
// Tile = 256 output rows (row tiles 2p, 2p+1; CTA rank r owns 2p+r) x NT tokens (rank r holds B for tokens
// r*NT/2 .. (r+1)*NT/2 - 1, loaded as two 64-token boxes).  Stage = 4 MMAs (16 blocks; 32 for M = 4).
// NT = 256: one accumulator (256 TMEM columns) — long K, the per-tile hand-off is amortised; NT = 192: two
// accumulators (2 x 192 columns) so the epilogue of tile i overlaps the MMAs of tile i + 1 — short K.
//   warp 0       TMA (both CTAs): own A (values_tc 128 x 64), own metadata chunk, own half of the X^T
//                window rows; completion counted on the leader's full barrier (cta_group::2 TMA);
//   warp 1       TMEM allocation (both CTAs) and, in the leader only, the MMA thread: tcgen05.cp of both
//                CTAs' metadata -> their TMEM, 4 x tcgen05.mma.sp.cta_group::2, commits multicast to both;
//   warps 4..    epilogue (both CTAs): warp 4 + q + 4c drains TMEM lanes 32q.. x the 64 columns of token
//                chunk c into registers, releases the accumulator (leader's tmem_empty), then converts and
//                writes Y^T through swizzled shared staging with TMA tensor stores, overlapping the next
//                tile's main loop.
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

// timing-ablation flags (VNM_ABL): a compile-time 0 in production builds, so no ablation test is left in the loops
#ifdef VNM_ABLATIONS
#define ABL(args) ((args).abl)
#else
#define ABL(args) 0
#endif

constexpr uint32_t kABytes = 128 * 128;     // 128 rows x 64 bf16 (SW128)
constexpr uint32_t kEBytes = 128 * 16;      // 128 lanes x 4 words
constexpr uint32_t kYSlot = 32 * 128;       // one 32 row x 128 B staging slot (SW128)
constexpr uint32_t kBChunk = 64;            // tokens per B box / per epilogue chunk

struct Tc2Args {
    int32_t T, rows, M;
    int32_t n_mma, n_stage, n_rt, n_rp, n_tt, work;
    int32_t row_major;   // tile order: pair-row-major (A reused across token tiles) or token-tile-major
    int32_t rows_stage;  // X^T rows advanced per stage
    int32_t rb;          // X^T rows loaded per stage (windows of the stage's blocks), multiple of 8
    int32_t stages;
    int32_t a_res;       // 1: A (values_tc) and metadata of the pair's rows stay resident in shared memory
                         //    (short K): the ring carries X^T only; each pair keeps one row pair
    int32_t y_slots;     // epilogue staging slots per warp (1 or 2)
    uint32_t b_bytes, stage_bytes, res_bytes;
    int32_t trace;       // VNM_SPMM_TRACE: per-CTA wait / busy cycle counters into g_tc2_t
    int32_t pf;          // L2 prefetch distance in stages (0: none): X^T streamed from HBM (long K, large T)
    int32_t abl;         // VNM_ABL (timing ablations only, results invalid): 1 no epilogue, 2 no Y stores,
                         // 4 no X^T loads, 8 no metadata copies after the first stage, 16 no A loads (streaming)
};

// VNM_SPMM_TRACE counters per CTA: MMA wait full, MMA wait tmem_empty, MMA loop total, producer wait empty,
// epilogue (warp 4) wait tmem_full, drain, store, tiles
__device__ unsigned long long g_tc2_t[8][160];

template <int NT>
struct Cfg {
    static constexpr int kNACC = NT == 256 ? 1 : 2;             // accumulators in TMEM
    static constexpr uint32_t kMetaCol = kNACC * NT;             // metadata ring after the accumulators
    static constexpr int kChunks = NT / kBChunk;                 // 64-token chunks per tile
    static constexpr int kEpiWarps = 4 * kChunks;                // one warp per (lane quadrant, chunk)
    static constexpr int kThreads = 128 + 32 * kEpiWarps;
};

// i-th tile (row pair rp, token tile tt) of cluster cid; false past the end
__device__ __forceinline__ bool tile_of(const Tc2Args& a, int cid, int ncl, int i, int& rp, int& tt) {
    if (a.a_res) {  // pairs in groups of n_rp (one per row pair); group g walks token tiles g, g + ng, ...
        const int ng = ncl / a.n_rp, g = cid / a.n_rp;
        rp = cid % a.n_rp;
        tt = g + i * ng;
        return g < ng && tt < a.n_tt;
    }
    const int w = cid + i * ncl;
    if (w >= a.work) return false;
    rp = a.row_major ? w / a.n_tt : w % a.n_rp;
    tt = a.row_major ? w % a.n_tt : w / a.n_rp;
    return true;
}

// the warp's TMEM reads are complete: one arrival per warp on the leader's tmem_empty
__device__ __forceinline__ void release(uint64_t* tmem_empty, int lane, bool leader) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (leader) mbar_arrive(tmem_empty);
        else mbar_arrive_remote(tmem_empty, 0);
    }
}

// 32 rows x 128 B (32 words per lane = one row) -> staging slot (c % nslot) of the warp, SW128 (16-byte chunk k
// of row r at k ^ (r % 8): conflict-free), then one TMA tensor store; the store clips rows / tokens
__device__ __forceinline__ void stage_store(uint8_t* buf, int nslot, int c, int lane, const uint32_t* w,
                                            const CUtensorMap* tm, int x, int y) {
    uint8_t* slot = buf + (nslot == 2 ? (c & 1) * kYSlot : 0);
    if (lane == 0) {  // the store that last used this slot has read it
        if (nslot == 2) bulk_wait_read<1>();
        else bulk_wait_read<0>();
    }
    __syncwarp();
    const uint32_t row = smem_u32(slot) + lane * 128;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((k ^ lane) & 7) << 4)), "r"(w[4 * k]),
                     "r"(w[4 * k + 1]), "r"(w[4 * k + 2]), "r"(w[4 * k + 3])
                     : "memory");
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(tm, x, y, slot);
        bulk_commit();
    }
}

template <int NT, bool kBf16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg<NT>::kThreads, 1)
    vnm_spmm_tc2_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_y,
                        const Tc2Args a) {
    using C = Cfg<NT>;
    constexpr int kNH = NT / 2;  // tokens per CTA of B
    constexpr uint32_t kMetaCol = C::kMetaCol;
    extern __shared__ __align__(1024) uint8_t smem[];  // (not re-aligned through an integer: keeps LDS/STS)
    const int S = a.stages;
    // [resident A (n_stage x 16 KB) | resident E (n_stage x 2 KB)] (a_res only), ring, Y staging, barriers
    uint8_t* ring = smem + a.res_bytes;
    uint8_t* sY = ring + S * a.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sY + C::kEpiWarps * a.y_slots * kYSlot);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;        // [kNACC]
    uint64_t* tmem_empty = tmem_full + 2;   // [kNACC]
    uint64_t* res_full = tmem_empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 1);
    const uint32_t b_off = a.a_res ? 0u : kABytes, e_off = kABytes + a.b_bytes;
    uint8_t* resE = smem + a.n_stage * kABytes;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = static_cast<int>(cluster_id_x()), ncl = static_cast<int>(nclusters_x());
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < C::kNACC; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 2 * C::kEpiWarps);
        }
        mbar_init(res_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        tma_prefetch_desc(&tmap_e);
        tma_prefetch_desc(&tmap_y);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_wait();    // the previous kernel's outputs (e.g. this layer's inputs) are visible
    grid_dep_launch();  // the next kernel may take SMs as this grid's CTAs exit

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            int q = 0, rp, tt;
            unsigned long long c_emp = 0, c0;
            for (int i = 0; tile_of(a, cid, ncl, i, rp, tt); ++i) {
                const int rt = 2 * rp + static_cast<int>(rank);  // row tiles past n_rt read as zeros (TMA OOB)
                const int rte = rt < a.n_rt ? rt : 0;             // ... with valid metadata
                const int n0 = tt * NT + kNH * static_cast<int>(rank);
                if (a.a_res && i == 0) {  // the pair's A and metadata, once
                    if (leader) mbar_arrive_expect_tx(res_full, 2 * a.n_stage * (kABytes + kEBytes));
                    for (int st = 0; st < a.n_stage; ++st) {
                        tma_load_2d_pair(smem + st * kABytes, &tmap_a, st * 64, rt * 128, res_full);
                        tma_load_2d_pair(resE + st * kEBytes, &tmap_e, 0, (rte * a.n_stage + st) * 128, res_full);
                    }
                }
                for (int st = 0; st < a.n_stage; ++st, ++q) {
                    const int s = q % S;
                    if (a.trace) c0 = clock64();
                    mbar_wait(&empty[s], ((q / S) & 1) ^ 1);
                    if (a.trace) c_emp += clock64() - c0;
                    uint8_t* base = ring + s * a.stage_bytes;
                    if (ABL(a) & 4) {
                        if (leader) mbar_arrive(&full[s]);
                        continue;
                    }
                    if (a.a_res) {
                        if (leader) mbar_arrive_expect_tx(&full[s], 2 * a.b_bytes);
                    } else {
                        if (leader) mbar_arrive_expect_tx(&full[s], 2 * ((ABL(a) & 16 ? 0u : kABytes) + kEBytes + a.b_bytes));
                        if (!(ABL(a) & 16)) tma_load_2d_pair(base, &tmap_a, st * 64, rt * 128, &full[s]);
                        tma_load_2d_pair(base + e_off, &tmap_e, 0, (rte * a.n_stage + st) * 128, &full[s]);
                    }
                    tma_load_2d_pair(base + b_off, &tmap_b, n0, st * a.rows_stage, &full[s]);
                    tma_load_2d_pair(base + b_off + a.rb * 128, &tmap_b, n0 + 64, st * a.rows_stage, &full[s]);
                    if (a.pf && st + a.pf < a.n_stage) {  // warm L2 for a later stage of this tile (beyond the ring)
                        tma_prefetch_l2(&tmap_b, n0, (st + a.pf) * a.rows_stage);
                        tma_prefetch_l2(&tmap_b, n0 + 64, (st + a.pf) * a.rows_stage);
                    }
                }
            }
            if (a.trace) g_tc2_t[3][blockIdx.x] = c_emp;
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader CTA; converged warp,
        // elected lane: see mma_sp_stage)
        if (leader) {
            int q = 0, tl = 0, rp, tt;
            const uint32_t idesc0 = idesc_bf16(256, NT, true, 0, true);
            const uint32_t idesc1 = idesc_bf16(256, NT, true, 1, true);
            // B descriptor advance per MMA (window-16 form, M > 8: +8 rows to the second half-windows, then the next
            // block group 4M rows on: ptx.cuh mma_sp_stage)
            const uint64_t b_step = (a.M == 4 ? 32u : a.M > 8 ? 8u : 4u * a.M) * 128u >> 4;
            const uint64_t b_step2 = a.M > 8 ? (4u * a.M * 128u) >> 4 : 2 * b_step;
            const uint32_t sbo = a.M == 4 ? 1024u : a.M * 128u;                 // K-group (window) stride
            const uint32_t b_lbo = a.rb * 128;
            unsigned long long c_full = 0, c_emp = 0, c_all = clock64(), c0;
            // The production loop, specialised per mode (RES: A + metadata resident) with nothing else in it — as in
            // spmm_tc3.cu, whose general loop ran the MMA-only skeleton 1.6x slower; the general loop below runs for
            // VNM_SPMM_TRACE and the timing ablations.
            auto mma_loop = [&](auto res_c) {
                constexpr bool RES = decltype(res_c)::value;
                if constexpr (RES) mbar_wait(res_full, 0);
                for (; tile_of(a, cid, ncl, tl, rp, tt); ++tl) {
                    const int acc = C::kNACC == 2 ? (tl & 1) : 0;
                    const uint32_t d_tmem = tmem + acc * NT;
                    mbar_wait(&tmem_empty[acc], ((C::kNACC == 2 ? tl >> 1 : tl) & 1) ^ 1);
                    tc_fence_after();
                    for (int st = 0; st < a.n_stage; ++st, ++q) {
                        const int s = q % S;
                        mbar_wait(&full[s], (q / S) & 1);
                        tc_fence_after();
                        uint8_t* base = ring + s * a.stage_bytes;
                        const uint32_t meta_s = tmem + kMetaCol + 4 * s;
                        const uint32_t e_s = RES ? smem_u32(resE + st * kEBytes) : smem_u32(base + e_off);
                        tmem_cp_elect<2>(meta_s, sdesc(e_s, 16, 128, 0));
                        const uint32_t a0 = RES ? smem_u32(smem + st * kABytes) : smem_u32(base);
                        const int left = a.n_mma - st * 4;
                        mma_sp_stage<2>(d_tmem, sdesc(a0, 16, 1024, kLayoutSW128),
                                        sdesc(smem_u32(base + b_off), b_lbo, sbo, kLayoutSW128), b_step, b_step2, meta_s,
                                        idesc0, idesc1, st > 0 ? 1u : 0u, left < 4 ? static_cast<uint32_t>(left) : 4u);
                        mma_commit_pair_elect(&empty[s], 0x3);
                    }
                    mma_commit_pair_elect(&tmem_full[acc], 0x3);
                }
            };
            if (!a.trace && !(ABL(a) & 8)) {
                if (a.a_res) mma_loop(std::true_type{});
                else mma_loop(std::false_type{});
            }
            for (; tile_of(a, cid, ncl, tl, rp, tt); ++tl) {
                if (a.a_res && tl == 0) mbar_wait(res_full, 0);
                const int acc = C::kNACC == 2 ? (tl & 1) : 0;
                const uint32_t d_tmem = tmem + acc * NT;
                c0 = clock64();
                mbar_wait(&tmem_empty[acc], ((C::kNACC == 2 ? tl >> 1 : tl) & 1) ^ 1);
                c_emp += clock64() - c0;
                tc_fence_after();
                for (int st = 0; st < a.n_stage; ++st, ++q) {
                    const int s = q % S;
                    c0 = clock64();
                    mbar_wait(&full[s], (q / S) & 1);
                    c_full += clock64() - c0;
                    tc_fence_after();
                    uint8_t* base = ring + s * a.stage_bytes;
                    const uint32_t meta_s = tmem + kMetaCol + 4 * s;
                    const uint32_t e_s = a.a_res ? smem_u32(resE + st * kEBytes) : smem_u32(base + e_off);
                    if (!(ABL(a) & 8) || q < S) tmem_cp_elect<2>(meta_s, sdesc(e_s, 16, 128, 0));
                    const uint32_t a0 = a.a_res ? smem_u32(smem + st * kABytes) : smem_u32(base);
                    const int left = a.n_mma - st * 4;
                    mma_sp_stage<2>(d_tmem, sdesc(a0, 16, 1024, kLayoutSW128),
                                    sdesc(smem_u32(base + b_off), b_lbo, sbo, kLayoutSW128), b_step, b_step2, meta_s, idesc0,
                                    idesc1, st > 0 ? 1u : 0u, left < 4 ? static_cast<uint32_t>(left) : 4u);
                    mma_commit_pair_elect(&empty[s], 0x3);
                }
                mma_commit_pair_elect(&tmem_full[acc], 0x3);
            }
            if (a.trace && lane == 0) {
                g_tc2_t[0][blockIdx.x] = c_full;
                g_tc2_t[1][blockIdx.x] = c_emp;
                g_tc2_t[2][blockIdx.x] = clock64() - c_all;
                g_tc2_t[7][blockIdx.x] = tl;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue (both CTAs)
        // warp 4 + q + 4c: TMEM lanes 32q.. (rows 32q.. of the CTA's row tile) x token chunk c (64 columns)
        const int ew = warp - 4, qd = ew % 4, ch = ew / 4;
        uint8_t* buf = sY + ew * a.y_slots * kYSlot;
        int tl = 0, rp, tt;
        unsigned long long c_wait = 0, c_drain = 0, c_store = 0, c0, c1;
        for (; tile_of(a, cid, ncl, tl, rp, tt); ++tl) {
            const int rt = 2 * rp + static_cast<int>(rank);
            const int t0 = tt * NT + kBChunk * ch;  // first token of this warp's chunk
            const int acc = C::kNACC == 2 ? (tl & 1) : 0;
            if (a.trace) c0 = clock64();
            mbar_wait(&tmem_full[acc], (C::kNACC == 2 ? tl >> 1 : tl) & 1);
            if (a.trace) {
                c1 = clock64();
                c_wait += c1 - c0;
            }
            tc_fence_after();
            const uint32_t taddr = tmem + ((32 * qd) << 16) + acc * NT + kBChunk * ch;
            const bool store = rt < a.n_rt && t0 < a.T && !(ABL(a) & 2);
            if (ABL(a) & 1) {
                release(&tmem_empty[acc], lane, leader);
                continue;
            }
            if constexpr (kBf16) {
                // drain the warp's 32 x 64 accumulator block (two loads, one wait) into 32 packed registers,
                // release the accumulator, then stage + store one 128-byte-per-row chunk
                uint32_t v[64], pk[32];
                tmem_ld_32x32b_x32(taddr, v);
                tmem_ld_32x32b_x32(taddr + 32, v + 32);
                tmem_wait_ld();
                release(&tmem_empty[acc], lane, leader);
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                    pk[k] = *reinterpret_cast<uint32_t*>(&b2);
                }
                if (a.trace) {
                    c0 = clock64();
                    c_drain += c0 - c1;
                }
                if (store) stage_store(buf, 1, 0, lane, pk, &tmap_y, t0, rt * 128 + 32 * qd);
                if (a.trace) c_store += clock64() - c0;
            } else {
                // fp32 (parity path): two 32-token chunks straight from TMEM; release at the end
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(taddr + 32 * c, v);
                    tmem_wait_ld();
                    if (store && t0 + 32 * c < a.T) stage_store(buf, 1, c, lane, v, &tmap_y, t0 + 32 * c, rt * 128 + 32 * qd);
                }
                release(&tmem_empty[acc], lane, leader);
            }
        }
        if (lane == 0) bulk_wait0();
        if (a.trace && warp == 4 && lane == 0) {
            g_tc2_t[4][blockIdx.x] = c_wait;
            g_tc2_t[5][blockIdx.x] = c_drain;
            g_tc2_t[6][blockIdx.x] = c_store;
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
int launch_nt(const SpmmLaunch& L, Tc2Args a, cudaStream_t stream) {
    using C = Cfg<NT>;
    const vnm_geom& g = L.P->g;
    a.n_tt = (L.T + NT - 1) / NT;
    a.work = a.n_rp * a.n_tt;
    // resident A when the pair's whole A + metadata fit next to >= 3 X^T stages (short K: DeiT layers)
    a.y_slots = 1;
    const uint32_t y_bytes = C::kEpiWarps * kYSlot;
    a.res_bytes = static_cast<uint32_t>(a.n_stage) * (kABytes + kEBytes);
    const uint32_t b_stage = (a.b_bytes + 1023) / 1024 * 1024;
    const uint32_t fixed = 1024 + 256;
    a.a_res = a.res_bytes + 3 * b_stage + y_bytes + fixed <= kMaxSmem ? 1 : 0;
    if (VNM_ENV_INT("VNM_TC2_ARES", 1) == 0) a.a_res = 0;
    if (a.a_res && num_sms() / 2 < a.n_rp) a.a_res = 0;  // every row pair needs a CTA pair of its own
    if (a.a_res) {
        a.stage_bytes = b_stage;
    } else {
        a.res_bytes = 0;
        a.stage_bytes = (kABytes + kEBytes + a.b_bytes + 1023) / 1024 * 1024;
    }
    const uint32_t avail = static_cast<uint32_t>(kMaxSmem) - a.res_bytes - y_bytes - fixed;
    a.stages = static_cast<int>(avail / a.stage_bytes);
    if (a.stages > 8) a.stages = 8;
    if (a.stages < 2) return kLaunchUnsupported;
    if (C::kMetaCol + 4 * a.stages > 512) a.stages = (512 - C::kMetaCol) / 4;
    // the larger operand stays hot in L2 across the tiles resident at a time (see spmm_tc.cu)
    const int64_t w_bytes = static_cast<int64_t>(a.n_rt) * 128 * 16 * a.n_mma;
    a.row_major = w_bytes > static_cast<int64_t>(g.cols) * L.T ? 1 : 0;
    if (const int v = VNM_ENV_INT("VNM_TC2_ORDER", -1); v >= 0) a.row_major = v;

    CUtensorMap ta, tb, te, ty;
    const int ld_tc = 16 * a.n_mma;
    if (!encode_2d(&ta, L.P->values_tc, static_cast<uint64_t>(ld_tc), static_cast<uint64_t>(a.n_rt) * 128,
                   static_cast<uint64_t>(ld_tc) * 2, 64, 128))
        return kLaunchCudaError;
    if (!encode_2d(&tb, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols),
                   static_cast<uint64_t>(L.ldx) * 2, 64, static_cast<uint32_t>(a.rb)))
        return kLaunchCudaError;
    if (!encode_2d(&te, L.P->meta_tc, 4, static_cast<uint64_t>(a.n_rt) * a.n_stage * 128, 16, 4, 128,
                   CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    const bool bf = L.y_dtype == VNM_BF16;
    if (!encode_2d(&ty, L.YT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.rows),
                   static_cast<uint64_t>(L.ldy) * (bf ? 2 : 4), bf ? 64 : 32, 32,
                   bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32))
        return kLaunchCudaError;
    const size_t smem = a.res_bytes + static_cast<size_t>(a.stages) * a.stage_bytes + y_bytes + fixed;
    auto k = bf ? vnm_spmm_tc2_kernel<NT, true> : vnm_spmm_tc2_kernel<NT, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return kLaunchCudaError;
    int pairs = num_sms() / 2;
    if (a.a_res) {
        const int ng = pairs / a.n_rp;  // groups of n_rp pairs, at most one group per token tile
        pairs = (ng < a.n_tt ? ng : a.n_tt) * a.n_rp;
    } else if (a.work < pairs) {
        pairs = a.work;
    }
    a.trace = VNM_ENV_INT("VNM_SPMM_TRACE", 0) ? 1 : 0;
    a.abl = VNM_ABLATION_FLAGS();
    // off by default: measured in whole steps it slowed DeiT-B 0.519 -> 0.554 ms (profiles/r01f_experiments.md)
    a.pf = VNM_ENV_INT("VNM_TC_PF", 0);
    cudaError_t e = launch_pdl(false, k, dim3(2 * pairs), dim3(C::kThreads), smem, stream, ta, tb, te, ty, a);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess && a.trace) {
        static unsigned long long h[8][160];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(h, g_tc2_t, sizeof(h));
        fprintf(stderr, "tc2 NT=%d: grid %d stages %d a_res %d n_stage %d work %d row_major %d\n", NT, 2 * pairs,
                a.stages, a.a_res, a.n_stage, a.work, a.row_major);
        for (int i = 0; i < 2 * pairs; i += 9)
            fprintf(stderr, "  cta %3d tiles %llu | mma: wait_full %7llu wait_empty %7llu total %8llu | prod wait %8llu | "
                            "epi wait %8llu drain %6llu store %7llu\n", i, h[7][i], h[0][i], h[1][i], h[2][i], h[3][i],
                    h[4][i], h[5][i], h[6][i]);
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

// T > 64, 4 <= M <= 8 (window form).  Returns kLaunchUnsupported when the configuration does not fit.
int launch_spmm_tc2(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (g.M > 15) return kLaunchUnsupported;  // M > 8: the window-16 form (include/vnm.h)
    Tc2Args a;
    a.T = L.T;
    a.rows = g.rows;
    a.M = g.M;
    a.n_mma = g.M > 8 ? g.nb_pad / 2 : g.nb_pad / (g.M == 4 ? 8 : 4);
    a.n_stage = (a.n_mma + 3) / 4;
    a.n_rt = (g.rows_p + 127) / 128;
    a.n_rp = (a.n_rt + 1) / 2;
    // X^T rows per stage and rows one stage's windows touch: window form 16 blocks (block 15: 15M .. 15M+7);
    // window-16 form 8 blocks (block 7: 7M .. 7M+15)
    a.rows_stage = g.M == 4 ? 128 : g.M > 8 ? 8 * g.M : 16 * g.M;
    const int need = g.M == 4 ? 128 : g.M > 8 ? 7 * g.M + 16 : 15 * g.M + 8;
    a.rb = (need + 7) / 8 * 8;
    a.b_bytes = static_cast<uint32_t>(2 * a.rb * 128);
    // long K: 256-token tiles, one accumulator (the per-tile hand-off is amortised over many stages);
    // short K: 192-token tiles with two accumulators so the epilogue overlaps the next tile
    int nt = a.n_stage >= 12 ? 256 : 192;
    if (const int v = VNM_ENV_INT("VNM_TC2_NT", 0)) nt = v;
    return nt == 256 ? launch_nt<256>(L, a, stream) : launch_nt<192>(L, a, stream);
}

}  // namespace vnm
