// spmm_tc3.cu — the window-form V:N:M SpMM (include/vnm.h values_tc / meta_tc) on CTA
// pairs for SHORT K and many tokens (DeiT layers: K = 384 / 768, T = 50,432): the HBM-bound shapes whose
// limits on B200 were measured to be shared-memory bandwidth (1-CTA kernel) and bytes in flight (pair
// kernel), profiles/r01c_*.
//
// What differs from spmm_tc2.cu:
//  * the pair's A (values_tc) and metadata stay resident for the CTA pair's lifetime: A in shared memory,
//    the metadata in TMEM (copied once), so the ring carries X^T only;
//  * X^T is staged in a K-RING: per 64-token chunk one contiguous run of rows, stage s at rows
//    [slot * rows_stage, +rows_stage) — each X^T row is loaded once per tile (the per-stage window overhang of
//    the 1-CTA / tc2 kernels is gone).  The windows of a stage's last blocks reach <= 7 rows into the next
//    slot, so stage q is issued only after stage q + 1 has landed; slot S-1 reaches into an 8-row shadow that
//    is loaded together with slot 0.  Window positions outside a block carry zero values, so stale rows
//    there multiply zeros (the ring is zero-filled at start, X^T is finite by precondition);
//  * each CTA loads exactly its NT/2 tokens: a 64-token box plus a narrower one (TMA keeps the 128-byte row
//    pitch and swizzle for boxes narrower than the span: tests/probes/probe_box.cu);
//  * NT = 192 or 224 tokens per pair tile with TWO accumulators (2 x NT + metadata <= 512 TMEM columns), so
//    the epilogue of tile i overlaps the MMAs of tile i + 1; 8 epilogue warps (2 per TMEM lane quadrant, taking
//    alternate 64-token chunks: a 4-warp epilogue could not keep up with the pair's store rate), one
//    staging slot each.
//
// Roles: warps 0 and 2 TMA producers (both CTAs), warp 1 MMA (leader CTA, converged warp, elected lane), warps 4-11
// epilogue (both CTAs: TMEM lanes 32q.. = rows 32q.. of the CTA's 128-row tile).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tmap.h"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr uint32_t kABytes = 128 * 128;  // one 4-MMA chunk of A: 128 rows x 64 bf16 (SW128)
constexpr uint32_t kEBytes = 128 * 16;   // one 4-MMA chunk of metadata: 128 lanes x 4 words
constexpr uint32_t kYSlot = 32 * 128;    // epilogue staging slot: 32 rows x 128 B (SW128)
constexpr int kEpi = 8;                  // epilogue warps: 2 per TMEM lane quadrant, alternating token chunks
constexpr int kThreads = 128 + 32 * kEpi;  // warps 0 + 2 TMA, 1 MMA, 3 idle, 4.. epilogue

struct Tc3Args {
    int32_t T, M;
    int32_t n_mma;       // MMAs per tile (K direction)
    int32_t n_chunk;     // 4-MMA chunks of A / metadata = ceil(n_mma / 4)
    int32_t ms;          // MMAs per ring stage (2 or 4)
    int32_t n_st;        // ring stages per tile = ceil(n_mma / ms)
    int32_t rows_stage;  // X^T rows per stage
    int32_t n_rt, n_rp, n_tt;
    int32_t S;           // ring slots
    int32_t rp_per;      // pairs per row pair group (pairs sharing one row pair)
    uint32_t ring_rows;  // S * rows_stage + 8 (shadow): rows per token-chunk region
    uint32_t stage_tx, shadow_tx;  // expect_tx bytes for both CTAs
    int32_t trace;
    int32_t peek; // windows cross stage boundaries (5 <= M <= 7: an 8-channel window is wider than a block)
    int32_t epi;  // 1: Y^T written with coalesced st.global from a warp-private shared transpose; 0: TMA stores
    void* Y;
    int64_t ldy;
    int32_t rows;
    int32_t abl;  // VNM_ABL timing ablations (results invalid): 1 no epilogue, 2 no Y stores, 4 no X^T loads
};

__device__ unsigned long long g_tc3_t[12][160];

// token tile i of this pair (pairs of one row pair share the token tiles round-robin); false past the end
__device__ __forceinline__ bool tile3(const Tc3Args& a, int cid, int i, int& rp, int& tt) {
    rp = cid % a.n_rp;
    const int g = cid / a.n_rp;
    tt = g + i * a.rp_per;
    return tt < a.n_tt;
}

template <int NT, bool kBf16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    vnm_spmm_tc3_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_e,
                        const __grid_constant__ CUtensorMap tmap_b0, const __grid_constant__ CUtensorMap tmap_b1,
                        const __grid_constant__ CUtensorMap tmap_s0, const __grid_constant__ CUtensorMap tmap_s1,
                        const __grid_constant__ CUtensorMap tmap_y, const __grid_constant__ CUtensorMap tmap_yt,
                        const Tc3Args a) {
    constexpr int kNH = NT / 2;          // tokens per CTA of B
    constexpr int kW1 = kNH - 64;        // width of the second token box
    constexpr uint32_t kMetaCol = 2 * NT;
    constexpr int kCw = kBf16 ? 64 : 32;           // tokens per 128-byte staging row
    constexpr int kNch = (NT + kCw - 1) / kCw;     // epilogue chunks per tile
    static_assert(kW1 > 0 && kW1 <= 64 && kW1 % 16 == 0, "token split");
    extern __shared__ __align__(1024) uint8_t smem[];
    const int S = a.S;
    // [A resident: n_chunk x 16 KB][E resident: n_chunk x 2 KB, padded to 1 KB][ring: 2 token chunks x ring_rows
    //  x 128 B][Y staging: kEpi warps x 1 slot][barriers]
    uint8_t* sA = smem;
    uint8_t* sE = smem + a.n_chunk * kABytes;
    uint8_t* ring = sE + (a.n_chunk * kEBytes + 1023) / 1024 * 1024;
    const uint32_t region = a.ring_rows * 128u;  // bytes per token-chunk region
    uint8_t* sY = ring + 2 * region;
    uint64_t* full = reinterpret_cast<uint64_t*>(sY + kEpi * kYSlot);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;   // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint64_t* res_full = tmem_empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 1);

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
        tma_prefetch_desc(&tmap_y);
        tma_prefetch_desc(&tmap_yt);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 2) {
        // ------------------------------------------------------------ TMA producers (both CTAs): warp 0 the
        // resident A / metadata, the expect_tx and the 64-token box, warp 2 the narrower box — two issuing
        // threads (one TMA-issuing thread capped the X^T stream, profiles/r01c_probes.md)
        const int pb = warp / 2;
        if (lane == 0) {
            int q = 0, rp, tt;
            unsigned long long c_emp = 0, c0;
            for (int i = 0; tile3(a, cid, i, rp, tt); ++i) {
                const int rt = 2 * rp + static_cast<int>(rank);  // row tiles past n_rt read as zeros (TMA OOB)
                if (i == 0 && pb == 0) {  // the pair's A and metadata, once
                    const int rte = rt < a.n_rt ? rt : 0;
                    if (leader) mbar_arrive_expect_tx(res_full, 2 * a.n_chunk * (kABytes + kEBytes));
                    for (int c = 0; c < a.n_chunk; ++c) {
                        tma_load_2d_pair(sA + c * kABytes, &tmap_a, c * 64, rt * 128, res_full);
                        tma_load_2d_pair(sE + c * kEBytes, &tmap_e, 0, (rte * a.n_chunk + c) * 128, res_full);
                    }
                }
                const int x0 = tt * NT + kNH * static_cast<int>(rank);
                for (int st = 0; st < a.n_st; ++st, ++q) {
                    const int s = q % S;
                    c0 = clock64();
                    mbar_wait(&empty[s], ((q / S) & 1) ^ 1);
                    c_emp += clock64() - c0;
                    if (a.abl & 4) {
                        if (leader && pb == 0) mbar_arrive(&full[s]);
                        continue;
                    }
                    // (box 1's bytes may land before box 0's thread registers the stage's expect_tx: the
                    // phase still needs that arrival, and the transaction count is signed)
                    if (leader && pb == 0) mbar_arrive_expect_tx(&full[s], a.stage_tx + (s == 0 ? a.shadow_tx : 0u));
                    const int y = st * a.rows_stage;
                    uint8_t* dst = ring + static_cast<uint32_t>(s * a.rows_stage) * 128u + pb * region;
                    tma_load_2d_pair(dst, pb ? &tmap_b1 : &tmap_b0, x0 + 64 * pb, y, &full[s]);
                    if (s == 0) {  // the shadow after the last slot: a copy of slot 0's first 8 rows
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
            unsigned long long c_full = 0, c_emp = 0, c_all = clock64(), c0;
            for (; tile3(a, cid, tl, rp, tt); ++tl) {
                if (tl == 0) {  // resident metadata -> TMEM columns kMetaCol + 4c (both CTAs)
                    mbar_wait(res_full, 0);
                    tc_fence_after();
                    for (int c = 0; c < a.n_chunk; ++c)
                        tmem_cp_elect<2>(tmem + kMetaCol + 4 * c, sdesc(smem_u32(sE + c * kEBytes), 16, 128, 0));
                }
                const int acc = tl & 1;
                c0 = clock64();
                mbar_wait(&tmem_empty[acc], ((tl >> 1) & 1) ^ 1);
                c_emp += clock64() - c0;
                tc_fence_after();
                for (int st = 0; st < a.n_st; ++st, ++q) {
                    const int s = q % S;
                    c0 = clock64();
                    mbar_wait(&full[s], (q / S) & 1);
                    if (a.peek && st + 1 < a.n_st) mbar_wait(&full[(q + 1) % S], ((q + 1) / S) & 1);  // window overhang
                    c_full += clock64() - c0;
                    tc_fence_after();
                    const int mi0 = st * a.ms;
                    const int left = a.n_mma - mi0;
                    const uint32_t n = static_cast<uint32_t>(left < a.ms ? left : a.ms);
                    const uint64_t ad = sdesc(smem_u32(sA + (mi0 >> 2) * kABytes), 16, 1024, kLayoutSW128) + 2 * (mi0 & 3);
                    const uint64_t bd =
                        sdesc(smem_u32(ring + static_cast<uint32_t>(s * a.rows_stage) * 128u), region, sbo, kLayoutSW128);
                    const uint32_t e = tmem + kMetaCol + 4 * (mi0 >> 2) + (mi0 & 2);
                    mma_sp_stage<2>(tmem + acc * NT, ad, bd, b_step, e, idesc0, idesc1, st > 0 ? 1u : 0u, n);
                    mma_commit_pair_elect(&empty[s], 0x3);
                }
                mma_commit_pair_elect(&tmem_full[acc], 0x3);
            }
            if (a.trace && lane == 0) {
                g_tc3_t[0][blockIdx.x] = c_full;
                g_tc3_t[1][blockIdx.x] = c_emp;
                g_tc3_t[2][blockIdx.x] = clock64() - c_all;
                g_tc3_t[7][blockIdx.x] = tl;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue (both CTAs)
        // warp 4 + qd: TMEM lanes 32qd.. (rows 32qd.. of the CTA's row tile), all NT columns in chunks of kCw
        // tokens (128 B per row): TMEM -> registers -> (bf16) -> staging slot (SW128, conflict-free) -> TMA
        // tensor store (a narrower box for a partial last chunk); the store clips rows >= rows, tokens >= T.
        const int qd = (warp - 4) % 4, half = (warp - 4) / 4;
        uint8_t* slot = sY + (warp - 4) * kYSlot;
        int tl = 0, rp, tt;
        unsigned long long c_wait = 0, c_epi = 0, c0, c1, c_ld = 0, c_slot = 0, c_st = 0, c_cvt = 0, c_iss = 0, d0;
        for (; tile3(a, cid, tl, rp, tt); ++tl) {
            const int rt = 2 * rp + static_cast<int>(rank);
            const int acc = tl & 1;
            c0 = clock64();
            mbar_wait(&tmem_full[acc], (tl >> 1) & 1);
            c1 = clock64();
            c_wait += c1 - c0;
            tc_fence_after();
            const uint32_t taddr = tmem + ((32 * qd) << 16) + acc * NT;
            const bool rows_ok = rt < a.n_rt && !(a.abl & 2);
            if (a.abl & 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&tmem_empty[acc]);
                    else mbar_arrive_remote(&tmem_empty[acc], 0);
                }
                continue;
            }
            const int last = ((kNch - 1 - half) / 2) * 2 + half;  // this warp's last chunk
#pragma unroll 1
            for (int c = half; c < kNch; c += 2) {
                const int t0 = tt * NT + c * kCw;
                uint32_t w[32];
                d0 = clock64();
                if constexpr (kBf16) {
                    uint32_t v[64];
                    tmem_ld_32x32b_x32(taddr + c * 64, v);
                    tmem_ld_32x32b_x32(taddr + c * 64 + 32, v + 32);  // past NT: other columns, not stored
                    tmem_wait_ld();
                    c_ld += clock64() - d0;
                    d0 = clock64();
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                        w[k] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                } else {
                    tmem_ld_32x32b_x32(taddr + c * 32, w);
                    tmem_wait_ld();
                }
                c_cvt += clock64() - d0;
                if (c == last) {  // this warp's part of the accumulator is drained: release it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tmem_empty[acc]);
                        else mbar_arrive_remote(&tmem_empty[acc], 0);
                    }
                }
                if (!rows_ok || t0 >= a.T) continue;
                d0 = clock64();
                const uint32_t row = smem_u32(slot) + lane * 128;
                if (a.epi) {
                    // rows -> the warp's slot (SW128: chunk k of row r at k ^ (r % 8), conflict-free), then read
                    // back 4 rows x 8 chunks per instruction (8 lanes per 128-byte row, conflict-free) and store
                    // full 128-byte lines with st.global.v4: no TMA, no proxy fence, no bulk-group waits
                    __syncwarp();  // the previous chunk's reads of the slot are done
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((k ^ lane) & 7) << 4)),
                                     "r"(w[4 * k]), "r"(w[4 * k + 1]), "r"(w[4 * k + 2]), "r"(w[4 * k + 3])
                                     : "memory");
                    __syncwarp();
                    c_st += clock64() - d0;
                    d0 = clock64();
                    constexpr int kEl = kBf16 ? 8 : 4;  // elements per 16 bytes
                    const int cc = lane & 7, tok = t0 + cc * kEl;
                    const int t_end = min(a.T, tt * NT + NT);
                    const int grow0 = rt * 128 + 32 * qd;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int r = 4 * j + (lane >> 3);
                        uint32_t x0, x1, x2, x3;
                        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                                     : "r"(smem_u32(slot) + r * 128 + (((cc ^ r) & 7) << 4)));
                        const int grow = grow0 + r;
                        if (grow >= a.rows || tok >= t_end) continue;
                        uint8_t* dst = static_cast<uint8_t*>(a.Y) + (static_cast<int64_t>(grow) * a.ldy + tok) * (kBf16 ? 2 : 4);
                        if (tok + kEl <= t_end) {
                            asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(x0), "r"(x1), "r"(x2),
                                         "r"(x3)
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
                    c_iss += clock64() - d0;
                    continue;
                }
                if (lane == 0) bulk_wait_read<0>();  // the previous store has read the slot
                __syncwarp();
                c_slot += clock64() - d0;
                d0 = clock64();
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((k ^ lane) & 7) << 4)),
                                 "r"(w[4 * k]), "r"(w[4 * k + 1]), "r"(w[4 * k + 2]), "r"(w[4 * k + 3])
                                 : "memory");
                fence_proxy_async_smem();
                __syncwarp();
                c_st += clock64() - d0;
                d0 = clock64();
                if (lane == 0) {
                    const bool tail = kBf16 && (NT % 64) != 0 && c == kNch - 1;
                    tma_store_2d(tail ? &tmap_yt : &tmap_y, t0, rt * 128 + 32 * qd, slot);
                    bulk_commit();
                }
                __syncwarp();
                c_iss += clock64() - d0;
            }
            c_epi += clock64() - c1;
        }
        if (lane == 0) bulk_wait0();
        if (a.trace && warp == 4 && lane == 0) {
            g_tc3_t[4][blockIdx.x] = c_wait;
            g_tc3_t[5][blockIdx.x] = c_epi;
            g_tc3_t[8][blockIdx.x] = c_ld;
            g_tc3_t[9][blockIdx.x] = c_slot;
            g_tc3_t[10][blockIdx.x] = c_st;
            g_tc3_t[6][blockIdx.x] = c_cvt;
            g_tc3_t[11][blockIdx.x] = c_iss;
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
int launch_nt3(const SpmmLaunch& L, Tc3Args a, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    constexpr int kNH = NT / 2, kW1 = kNH - 64;
    a.n_tt = (L.T + NT - 1) / NT;
    if (2 * NT + 4 * a.n_chunk > 512) return kLaunchUnsupported;  // accumulators + resident metadata
    const uint32_t res = static_cast<uint32_t>(a.n_chunk) * kABytes + (a.n_chunk * kEBytes + 1023) / 1024 * 1024;
    const uint32_t fixed = kEpi * kYSlot + 1024;
    // ring slots: as many as fit (bytes in flight hide the HBM latency), at least 3
    int S = 0;
    for (int s = 8; s >= 3 && !S; --s)
        if (res + 2u * (s * a.rows_stage + 8) * 128u + fixed <= kMaxSmem) S = s;
    if (!S) return kLaunchUnsupported;
    if (const char* e = getenv("VNM_TC3_S")) { const int v = atoi(e); if (v >= 3 && v < S) S = v; }
    a.S = S;
    a.ring_rows = static_cast<uint32_t>(S * a.rows_stage + 8);
    a.stage_tx = 2u * a.rows_stage * (64 + kW1) * 2u;
    a.shadow_tx = 2u * 8u * (64 + kW1) * 2u;
    const int pairs_all = num_sms() / 2;
    if (pairs_all < a.n_rp) return kLaunchUnsupported;
    // pairs per row pair: every pair owns one row pair; the token tiles of a row pair are dealt round-robin
    a.rp_per = pairs_all / a.n_rp;
    if (a.rp_per > a.n_tt) a.rp_per = a.n_tt;
    const int pairs = a.rp_per * a.n_rp;

    CUtensorMap ta, te, tb0, tb1, ts0, ts1, ty, tyt;
    const int ld_tc = 16 * a.n_mma;
    if (!encode_2d(&ta, L.P->values_tc, static_cast<uint64_t>(ld_tc), static_cast<uint64_t>(a.n_rt) * 128,
                   static_cast<uint64_t>(ld_tc) * 2, 64, 128))
        return kLaunchCudaError;
    if (!encode_2d(&te, L.P->meta_tc, 4, static_cast<uint64_t>(a.n_rt) * a.n_chunk * 128, 16, 4, 128,
                   CU_TENSOR_MAP_DATA_TYPE_UINT32, CU_TENSOR_MAP_SWIZZLE_NONE))
        return kLaunchCudaError;
    const uint64_t xr = static_cast<uint64_t>(L.ldx) * 2;
    if (!encode_2d(&tb0, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, 64,
                   static_cast<uint32_t>(a.rows_stage)) ||
        !encode_2d(&tb1, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, kW1,
                   static_cast<uint32_t>(a.rows_stage)) ||
        !encode_2d(&ts0, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, 64, 8) ||
        !encode_2d(&ts1, L.XT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.cols), xr, kW1, 8))
        return kLaunchCudaError;
    const bool bf = L.y_dtype == VNM_BF16;
    const CUtensorMapDataType ydt = bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const uint64_t yr = static_cast<uint64_t>(L.ldy) * (bf ? 2 : 4);
    if (!encode_2d(&ty, L.YT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.rows), yr, bf ? 64 : 32, 32, ydt) ||
        !encode_2d(&tyt, L.YT, static_cast<uint64_t>(L.T), static_cast<uint64_t>(g.rows), yr,
                   bf ? (NT % 64 ? NT % 64 : 64) : 32, 32, ydt))
        return kLaunchCudaError;
    const size_t smem = res + 2u * a.ring_rows * 128u + fixed;
    auto k = bf ? vnm_spmm_tc3_kernel<NT, true> : vnm_spmm_tc3_kernel<NT, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return kLaunchCudaError;
    a.trace = getenv("VNM_SPMM_TRACE") ? 1 : 0;
    a.abl = getenv("VNM_ABL") ? atoi(getenv("VNM_ABL")) : 0;
    a.epi = getenv("VNM_TC3_EPI") ? atoi(getenv("VNM_TC3_EPI")) : 1;
    a.Y = L.YT;
    a.ldy = L.ldy;
    a.rows = g.rows;
    k<<<2 * pairs, kThreads, smem, stream>>>(ta, te, tb0, tb1, ts0, ts1, ty, tyt, a);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && a.trace) {
        static unsigned long long h[12][160];
        cudaStreamSynchronize(stream);
        cudaMemcpyFromSymbol(h, g_tc3_t, sizeof(h));
        fprintf(stderr, "tc3 NT=%d: grid %d S %d ms %d n_st %d n_mma %d rp_per %d smem %zu\n", NT, 2 * pairs, a.S, a.ms,
                a.n_st, a.n_mma, a.rp_per, smem);
        for (int i = 0; i < 2 * pairs; i += 10)
            fprintf(stderr, "  cta %3d tiles %llu | mma: wait_full %7llu wait_empty %7llu total %8llu | prod wait %8llu | "
                            "epi wait %8llu busy %8llu (ld %llu cvt %llu slot %llu st %llu iss %llu)\n", i, h[7][i], h[0][i],
                    h[1][i], h[2][i], h[3][i], h[4][i], h[5][i], h[8][i], h[6][i], h[9][i], h[10][i], h[11][i]);
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

// Window form, 4 <= M <= 8, A + metadata of a row pair resident (short K).  kLaunchUnsupported when the
// configuration does not fit (the caller then uses the tc / tc2 kernels).
int launch_spmm_tc3(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (g.M > 8 || g.M < 4) return kLaunchUnsupported;
    Tc3Args a;
    a.T = L.T;
    a.M = g.M;
    a.n_mma = g.nb_pad / (g.M == 4 ? 8 : 4);
    a.n_chunk = (a.n_mma + 3) / 4;
    a.n_rt = (g.rows_p + 127) / 128;
    a.n_rp = (a.n_rt + 1) / 2;
    // 4 MMAs per stage (16 blocks); 2 when a 4-MMA stage would be large (M = 8: 128 rows)
    a.ms = g.M >= 7 ? 2 : 4;
    if (const char* e = getenv("VNM_TC3_MS")) a.ms = atoi(e) == 2 ? 2 : 4;
    a.n_st = (a.n_mma + a.ms - 1) / a.ms;
    a.peek = g.M >= 5 && g.M <= 7;
    a.rows_stage = a.ms * (g.M == 4 ? 32 : 4 * g.M);
    int nt = 224;
    if (const char* e = getenv("VNM_TC3_NT")) nt = atoi(e);
    return nt == 192 ? launch_nt3<192>(L, a, stream) : launch_nt3<224>(L, a, stream);
}

}  // namespace vnm
