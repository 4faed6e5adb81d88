// prune.cu — the V:N:M mask + compression pass for sm_100a.
//
// S_{V:N:M} (§3 "Pruning of V:N:M sparsity"):
//   1) importance e = |score| (ABS: e = |W|)
//   2) per V x M block, column L1 of e over the V rows; keep the 4 largest
//   3) per row, keep the 2 largest e among the 4 kept columns
// followed by the compressed-format conversion A_n / A_i1 / A_i2 (App. A).
//
// Design (B200): one CTA = a tile of RT rows (RT = max(V, 32)) x CB column blocks (CB*M columns).
//   load   : the W (and score) tile is staged into shared memory with 16-byte cp.async
//            (coalesced, zero-fill past the logical extent = implicit padding);
//   compute: Lb = min(8, V) lanes own one block; each lane holds rows j, j+Lb, ... of the block, sums
//            them with an in-lane halving tree, then Lb-lane xor butterflies finish the canonical
//            stride-halving tree (Q3) — bit-identical in every lane to the oracle's order;
//            top-4 by a running insertion list (ties -> smaller column), per-row top-2 (ties -> smaller
//            position), all integer / compare work in registers;
//   store  : outputs are staged in shared memory and written row-wise with 16-byte stores.
// The pass is HBM-bound: algorithmic bytes per weight element = 2 (W) [+4 score] + (4 + 0.5)/M
// (values + meta) + 4/(V M) (col_idx) + 1/8 (mask).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "tc_form.cuh"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct PruneArgs {
    const uint16_t* W;
    int64_t ldw;
    const float* score;
    int64_t lds;
    const uint32_t* mask_in;  // FROM_MASK
    uint32_t* mask_out;       // may be null
    uint16_t* values;         // may be null (mask-only prune)
    uint8_t* col_idx;
    uint32_t* meta;
    int32_t* status;  // FROM_MASK, may be null
    uint16_t* values_tc;  // optional window form (V = 64, M <= 8, CB = 32), see tc_form.cuh
    uint32_t* meta_tc;
    int32_t ld_tc, n_stage_tc;
    int32_t rows, cols, M, rows_p, cols_p, nb, nb_pad, ld_val, ld_meta, ld_mask;
    int32_t CB;  // column blocks per CTA (32, 16 or 8)
};

__device__ __forceinline__ float bf16_abs_to_f32(uint16_t h) {
    return __uint_as_float(static_cast<uint32_t>(h & 0x7FFFu) << 16);
}

template <int V>
struct Shape {
    static constexpr int Lb = V < 8 ? V : 8;  // lanes per block
    static constexpr int RPL = V / Lb;        // rows per lane
    static constexpr int RT = V < 32 ? 32 : V;
    static constexpr int IPW = 32 / Lb;  // items per warp pass
};

template <int LB>
__device__ __forceinline__ float butterfly_sum(float v) {
#pragma unroll
    for (int s = LB / 2; s >= 1; s >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, s);
    return v;
}
template <int LB>
__device__ __forceinline__ uint32_t butterfly_or(uint32_t v) {
#pragma unroll
    for (int s = LB / 2; s >= 1; s >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, s);
    return v;
}

// MT: compile-time M (0 = runtime a.M).  With M known the tile pitch and every block offset fold into
// immediate shared-memory offsets (address arithmetic was a third of the instructions with runtime M).
template <int V, int MT, bool FROM_MASK, bool HAS_SCORE>
__global__ void __launch_bounds__(kThreads) prune_pack_kernel(const PruneArgs a) {
    using S = Shape<V>;
    constexpr int RT = S::RT, Lb = S::Lb, RPL = S::RPL, IPW = S::IPW;
    extern __shared__ __align__(16) uint8_t smem[];
    const int CB = MT ? 32 : a.CB, M = MT ? MT : a.M;
    const int tile_cols = CB * M;
    const int pitch_w = tile_cols + 8;  // bf16 elements; +16 B breaks row-to-row bank aliasing
    const int pitch_s = tile_cols + 4;  // fp32
    const int mwords = tile_cols / 32;  // mask words per row in this tile
    const int b0 = blockIdx.x * CB;
    const int r0 = blockIdx.y * RT;
    const int c0 = b0 * M;

    // ---- shared memory carve-up
    uint8_t* p = smem;
    uint16_t* sW = reinterpret_cast<uint16_t*>(p);
    p += static_cast<size_t>(RT) * pitch_w * 2;
    float* sS = reinterpret_cast<float*>(p);
    if (HAS_SCORE) p += static_cast<size_t>(RT) * pitch_s * 4;
    uint32_t* sM = reinterpret_cast<uint32_t*>(p);
    if (FROM_MASK) p += static_cast<size_t>(RT) * mwords * 4;
    uint16_t* sVal = reinterpret_cast<uint16_t*>(p);
    p += static_cast<size_t>(RT) * 2 * CB * 2;
    uint32_t* sBits = reinterpret_cast<uint32_t*>(p);
    p += static_cast<size_t>(RT) * CB * 4;
    uint32_t* sCi = reinterpret_cast<uint32_t*>(p);
    p += static_cast<size_t>(RT / V) * CB * 4;
    uint8_t* sNib = p;
    p += static_cast<size_t>(RT) * CB;
    // window form staging (only when a.values_tc): 4 values and a nibble pair per row-block
    p = smem + ((p - smem + 15) & ~static_cast<ptrdiff_t>(15));  // 16-B aligned, still a shared pointer
    uint16_t* sTcv = reinterpret_cast<uint16_t*>(p);
    p += static_cast<size_t>(RT) * 4 * CB * 2;
    uint8_t* sTcn = p;

    // ---- load the tile (zero-filled outside rows x cols)
    {
        const int chunks = tile_cols / 8;  // 16-byte chunks of bf16 per row
        for (int i = threadIdx.x; i < RT * chunks; i += kThreads) {
            const int r = i / chunks, ch = i % chunks;
            const int gr = r0 + r, gc = c0 + ch * 8;
            int bytes = (gr < a.rows) ? (a.cols - gc) * 2 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            const uint16_t* src = bytes ? a.W + static_cast<int64_t>(gr) * a.ldw + gc : a.W;
            cp_async_16(sW + r * pitch_w + ch * 8, src, static_cast<uint32_t>(bytes));
        }
        if (HAS_SCORE) {
            const int schunks = tile_cols / 4;
            for (int i = threadIdx.x; i < RT * schunks; i += kThreads) {
                const int r = i / schunks, ch = i % schunks;
                const int gr = r0 + r, gc = c0 + ch * 4;
                int bytes = (gr < a.rows) ? (a.cols - gc) * 4 : 0;
                bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
                const float* src = bytes ? a.score + static_cast<int64_t>(gr) * a.lds + gc : a.score;
                cp_async_16(sS + r * pitch_s + ch * 4, src, static_cast<uint32_t>(bytes));
            }
        }
        cp_async_commit();
        if (FROM_MASK) {
            const int w0 = c0 / 32;
            for (int i = threadIdx.x; i < RT * mwords; i += kThreads) {
                const int r = i / mwords, w = i % mwords;
                const int gr = r0 + r, gw = w0 + w;
                sM[i] = (gr < a.rows_p && gw < a.ld_mask) ? a.mask_in[static_cast<int64_t>(gr) * a.ld_mask + gw] : 0u;
            }
            // bits at columns >= cols_p (only the last word of a row can hold them)
            if (a.status && (a.cols_p % 32) != 0) {
                const int lw = a.ld_mask - 1;
                if (lw >= w0 && lw < w0 + mwords) {
                    const uint32_t over = ~((1u << (a.cols_p % 32)) - 1u);
                    for (int r = threadIdx.x; r < RT; r += kThreads) {
                        const int gr = r0 + r;
                        if (gr < a.rows_p && (a.mask_in[static_cast<int64_t>(gr) * a.ld_mask + lw] & over))
                            atomicMin(a.status, 1 + (a.rows_p / V) * a.nb);
                    }
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();
    }

    // ---- compute: items (vb_local, b_local), IPW per warp pass
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int g = lane / Lb, j = lane % Lb;
    const int items = (RT / V) * CB;
    const uint32_t colmask = (M >= 32) ? 0xffffffffu : ((1u << M) - 1u);
    for (int base = warp * IPW; base < items; base += kWarps * IPW) {
        const int it = base + g;
        const bool live = it < items;  // whole-warp control flow stays uniform (shuffles below)
        const int vbl = live ? it / CB : 0, bl = live ? it % CB : 0;
        const int b = b0 + bl;
        const bool real = live && b < a.nb && (r0 + vbl * V) < a.rows_p;
        const int rbase = vbl * V;  // tile-local first row of the block
        uint32_t rowbits[RPL];      // per owned row: block-local columns kept (2 bits)
        uint32_t uni = 0;
        bool bad = false;
        if (!FROM_MASK) {
            // step 2: column L1 (canonical tree) + running top-4 (ties -> smaller column)
            float tv[4] = {-1.f, -1.f, -1.f, -1.f};
            int ti[4] = {0, 1, 2, 3};
            for (int c = 0; c < M; ++c) {
                float s[RPL];
#pragma unroll
                for (int i = 0; i < RPL; ++i) {
                    const int r = rbase + j + Lb * i;
                    s[i] = HAS_SCORE ? fabsf(sS[r * pitch_s + bl * M + c]) : bf16_abs_to_f32(sW[r * pitch_w + bl * M + c]);
                }
#pragma unroll
                for (int st = RPL / 2; st >= 1; st >>= 1)
#pragma unroll
                    for (int i = 0; i < st; ++i) s[i] = s[i] + s[i + st];
                const float L = butterfly_sum<Lb>(s[0]);
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
            uint32_t kp = 0;  // kept columns ascending, 8 bits each
#pragma unroll
            for (int q = 0; q < 4; ++q) { kp |= static_cast<uint32_t>(__ffs(km) - 1) << (8 * q); km &= km - 1; }
            // step 3: per row top-2 of the kept 4 (ties -> smaller position), branch-free: key = (e, 3 - pos)
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
                const int r = rbase + j + Lb * i;
                const uint16_t* wr = sW + r * pitch_w + bl * M;
                uint16_t w4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) w4[q] = wr[(kp >> (8 * q)) & 0xFFu];
                int f, sc;
                if (HAS_SCORE) {
                    const float* sr = sS + r * pitch_s + bl * M;
                    unsigned long long k[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        k[q] = (static_cast<unsigned long long>(__float_as_uint(fabsf(sr[(kp >> (8 * q)) & 0xFFu]))) << 2) |
                               static_cast<unsigned long long>(3 - q);
                    const unsigned long long m01 = k[0] > k[1] ? k[0] : k[1], n01 = k[0] > k[1] ? k[1] : k[0];
                    const unsigned long long m23 = k[2] > k[3] ? k[2] : k[3], n23 = k[2] > k[3] ? k[3] : k[2];
                    const unsigned long long k1 = m01 > m23 ? m01 : m23;
                    const unsigned long long lo2 = m01 > m23 ? m23 : m01, hi2 = n01 > n23 ? n01 : n23;
                    const unsigned long long k2 = lo2 > hi2 ? lo2 : hi2;
                    f = 3 - static_cast<int>(k1 & 3u);
                    sc = 3 - static_cast<int>(k2 & 3u);
                } else {
                    uint32_t k[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) k[q] = (static_cast<uint32_t>(w4[q] & 0x7FFFu) << 2) | (3u - q);
                    const uint32_t m01 = max(k[0], k[1]), n01 = min(k[0], k[1]);
                    const uint32_t m23 = max(k[2], k[3]), n23 = min(k[2], k[3]);
                    const uint32_t k1 = max(m01, m23), k2 = max(min(m01, m23), max(n01, n23));
                    f = 3 - static_cast<int>(k1 & 3u);
                    sc = 3 - static_cast<int>(k2 & 3u);
                }
                rowbits[i] = (1u << ((kp >> (8 * f)) & 0xFFu)) | (1u << ((kp >> (8 * sc)) & 0xFFu));
                uni |= rowbits[i];
            }
        } else {
            // the mask decides: each row must hold exactly 2 bits in the block
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
                const int r = rbase + j + Lb * i;
                const int cb = bl * M;  // tile-local first column
                const uint32_t* mrow = sM + r * mwords;
                const int w = cb / 32, sh = cb % 32;
                uint64_t two = static_cast<uint64_t>(mrow[w]);
                if (w + 1 < mwords) two |= static_cast<uint64_t>(mrow[w + 1]) << 32;
                const uint32_t rb = static_cast<uint32_t>(two >> sh) & colmask;
                rowbits[i] = rb;
                bad |= __popc(rb) != 2;
                uni |= rb;
            }
        }
        uni = butterfly_or<Lb>(uni);
        if (FROM_MASK) {
            bad |= __popc(uni) > 4;
            const bool any_bad = butterfly_or<Lb>(bad ? 1u : 0u) != 0u;
            if (real && any_bad && j == 0 && a.status)
                atomicMin(a.status, 1 + (blockIdx.y * (RT / V) + vbl) * a.nb + b);
        }
        // A_i1: columns carrying bits, completed with the lowest free columns (Q19)
        uint32_t ci = real ? uni : 0u;
        for (int need = 4 - __popc(ci); need > 0; --need) ci |= 1u << (__ffs(~ci & colmask) - 1);
        if (__popc(ci) > 4) ci = 0xFu;  // invalid mask: any well-formed value
        // outputs of the owned rows
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
            const int r = rbase + j + Lb * i;
            uint32_t rb = real ? rowbits[i] : 0u;
            if (__popc(rb) != 2) rb = 0u;  // pad block / invalid row
            uint32_t nib = 0x4u;
            uint16_t v0 = 0, v1 = 0;
            if (rb) {
                const int clo = __ffs(rb) - 1, chi = 31 - __clz(rb);
                const uint32_t plo = __popc(ci & ((1u << clo) - 1u)), phi = __popc(ci & ((1u << chi) - 1u));
                nib = plo | (phi << 2);
                v0 = sW[r * pitch_w + bl * M + clo];
                v1 = sW[r * pitch_w + bl * M + chi];
            }
            if (live) {
                sVal[r * 2 * CB + 2 * bl + 0] = v0;
                sVal[r * 2 * CB + 2 * bl + 1] = v1;
                sNib[r * CB + bl] = static_cast<uint8_t>(nib);
                if (a.values_tc) {
                    const int cl = rb ? __ffs(rb) - 1 : 0, ch = rb ? 31 - __clz(rb) : 1;
                    const TcBlock t = tc_encode_block(cl, ch, v0, v1);
                    if (M == 4) {
                        sTcv[r * 4 * CB + 2 * bl] = v0;
                        sTcv[r * 4 * CB + 2 * bl + 1] = v1;
                    } else {
                        uint2 pk;
                        pk.x = static_cast<uint32_t>(t.val[0]) | (static_cast<uint32_t>(t.val[1]) << 16);
                        pk.y = static_cast<uint32_t>(t.val[2]) | (static_cast<uint32_t>(t.val[3]) << 16);
                        *reinterpret_cast<uint2*>(sTcv + r * 4 * CB + 4 * bl) = pk;
                    }
                    sTcn[r * CB + bl] = static_cast<uint8_t>(t.nibs);
                }
                sBits[r * CB + bl] = rb;
            }
        }
        if (live && j == 0) {
            uint32_t word = 0, m = ci;
#pragma unroll
            for (int q = 0; q < 4; ++q) { word |= static_cast<uint32_t>(__ffs(m) - 1) << (8 * q); m &= m - 1; }
            sCi[vbl * CB + bl] = word;
        }
    }
    __syncthreads();

    // ---- store (row-wise, vectorised)
    const int cbv = min(CB, a.nb_pad - b0);  // blocks of this tile inside nb_pad
    const int rows_here = min(RT, a.rows_p - r0);
    if (a.values && cbv > 0) {
        // values: 2*cbv bf16 per row = cbv/2 chunks of 16 B (cbv is a multiple of 8)
        const int vch = cbv / 4;
        for (int i = threadIdx.x; i < rows_here * vch; i += kThreads) {
            const int r = i / vch, ch = i % vch;
            const uint4 v = *reinterpret_cast<const uint4*>(sVal + r * 2 * CB + ch * 8);
            *reinterpret_cast<uint4*>(a.values + static_cast<int64_t>(r0 + r) * a.ld_val + 2 * b0 + ch * 8) = v;
        }
        // meta: cbv/8 words per row
        const int mw = cbv / 8;
        for (int i = threadIdx.x; i < rows_here * mw; i += kThreads) {
            const int r = i / mw, w = i % mw;
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) word |= static_cast<uint32_t>(sNib[r * CB + 8 * w + q]) << (4 * q);
            a.meta[static_cast<int64_t>(r0 + r) * a.ld_meta + b0 / 8 + w] = word;
        }
        if (b0 + cbv == a.nb_pad) {  // last column tile: the row's pad words past nb_pad / 8 (8 pad blocks each)
            const int pw0 = a.nb_pad / 8, npw = a.ld_meta - pw0;
            for (int i = threadIdx.x; i < rows_here * npw; i += kThreads)
                a.meta[static_cast<int64_t>(r0 + i / npw) * a.ld_meta + pw0 + i % npw] = 0x44444444u;
        }
        // col_idx: [vb][b][4]
        const int nvb_here = rows_here / V;
        for (int i = threadIdx.x; i < nvb_here * cbv; i += kThreads) {
            const int v = i / cbv, bl = i % cbv;
            const int vbg = (r0 / V) + v;
            reinterpret_cast<uint32_t*>(a.col_idx)[static_cast<int64_t>(vbg) * a.nb_pad + b0 + bl] = sCi[v * CB + bl];
        }
    }
    if (a.values_tc && cbv > 0) {
        // window form (include/vnm.h values_tc / meta_tc): this CTA = one V-block (64 rows) x 32 blocks
        const int bpm = M == 4 ? 8 : 4;
        const int vpb = M == 4 ? 2 : 4;  // window-form values per block
        const int tch = cbv * vpb / 8;   // 16-byte chunks per row
        for (int i = threadIdx.x; i < rows_here * tch; i += kThreads) {
            const int r = i / tch, c = i % tch;
            const uint4 v = *reinterpret_cast<const uint4*>(sTcv + r * 4 * CB + 8 * c);
            *reinterpret_cast<uint4*>(a.values_tc + static_cast<int64_t>(r0 + r) * a.ld_tc + vpb * b0 + 8 * c) = v;
        }
        // meta_tc words of this V-block's 64 lanes (lanes 64h..64h+63 of the 128-row tile)
        const int tile = r0 / 128, half = (r0 / 64) & 1;
        const int mi0 = b0 / bpm, n_mi = cbv / bpm;
        for (int i = threadIdx.x; i < n_mi * 64; i += kThreads) {
            const int L = 64 * half + (i % 64), mi = mi0 + i / 64;
            const int h = (L / 8) & 1;
            const int ra = (L % 8) + 16 * (L / 16) - 64 * half, rb_ = ra + 8;
            uint32_t wa = 0, wb = 0;
            if (M == 4) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int bl = 8 * (mi - mi0) + 4 * h + q;
                    wa |= static_cast<uint32_t>(sNib[ra * CB + bl]) << (4 * q);
                    wb |= static_cast<uint32_t>(sNib[rb_ * CB + bl]) << (4 * q);
                }
            } else {
                const int bl = 4 * (mi - mi0) + 2 * h;
                wa = static_cast<uint32_t>(sTcn[ra * CB + bl]) | (static_cast<uint32_t>(sTcn[ra * CB + bl + 1]) << 8);
                wb = static_cast<uint32_t>(sTcn[rb_ * CB + bl]) | (static_cast<uint32_t>(sTcn[rb_ * CB + bl + 1]) << 8);
            }
            a.meta_tc[((static_cast<int64_t>(tile) * a.n_stage_tc + mi / 4) * 128 + L) * 4 + (mi % 4)] = wa | (wb << 16);
        }
        // MMA slots past the last real MMA of the last stage: filler metadata (as vnm_pack_tc writes)
        const int n_mma = a.ld_tc / 16;
        if (b0 + CB >= a.nb_pad) {
            for (int i = threadIdx.x; i < (4 * a.n_stage_tc - n_mma) * 64; i += kThreads) {
                const int L = 64 * half + (i % 64), mi = n_mma + i / 64;
                a.meta_tc[((static_cast<int64_t>(tile) * a.n_stage_tc + mi / 4) * 128 + L) * 4 + (mi % 4)] = 0x44444444u;
            }
        }
    }
    if (a.mask_out) {
        const int w0 = c0 / 32;
        const int nw = min(mwords, a.ld_mask - w0);
        for (int i = threadIdx.x; i < rows_here * nw; i += kThreads) {
            const int r = i / nw, w = i % nw;
            const int lo_col = 32 * w, hi_col = lo_col + 31;  // tile-local columns of this word
            uint32_t word = 0;
            for (int bl = lo_col / M; bl <= hi_col / M && bl < CB; ++bl) {
                const uint32_t bits = sBits[r * CB + bl];
                const int sh = bl * M - lo_col;
                word |= sh >= 0 ? (sh < 32 ? bits << sh : 0u) : bits >> (-sh);
            }
            a.mask_out[static_cast<int64_t>(r0 + r) * a.ld_mask + w0 + w] = word;
        }
    }
}

__global__ void status_init_kernel(int32_t* s) { *s = 0x7fffffff; }
__global__ void status_fini_kernel(int32_t* s) {
    if (*s == 0x7fffffff) *s = 0;
}

size_t smem_bytes(int V, int M, int CB, bool from_mask, bool has_score, bool tc) {
    const int RT = V < 32 ? 32 : V;
    const int tile_cols = CB * M;
    size_t b = static_cast<size_t>(RT) * (tile_cols + 8) * 2;
    if (has_score) b += static_cast<size_t>(RT) * (tile_cols + 4) * 4;
    if (from_mask) b += static_cast<size_t>(RT) * (tile_cols / 32) * 4;
    b += static_cast<size_t>(RT) * 2 * CB * 2 + static_cast<size_t>(RT) * CB * 4 +
         static_cast<size_t>(RT / V) * CB * 4 + static_cast<size_t>(RT) * CB;
    if (tc) b += 16 + static_cast<size_t>(RT) * 4 * CB * 2 + static_cast<size_t>(RT) * CB;
    return b;
}

template <int V, int MT, bool FROM_MASK, bool HAS_SCORE>
cudaError_t launch_t(const PruneArgs& a, size_t smem, cudaStream_t st) {
    auto k = prune_pack_kernel<V, MT, FROM_MASK, HAS_SCORE>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    constexpr int RT = Shape<V>::RT;
    dim3 grid((a.nb_pad + a.CB - 1) / a.CB, (a.rows_p + RT - 1) / RT);
    k<<<grid, kThreads, smem, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

// V = 64 with M in 4..8 and CB = 32 (the paper's configurations) get compile-time M
template <bool FROM_MASK, bool HAS_SCORE>
cudaError_t launch_m64(const PruneArgs& a, size_t smem, cudaStream_t st) {
    if (a.CB == 32) {
        switch (a.M) {
            case 4: return launch_t<64, 4, FROM_MASK, HAS_SCORE>(a, smem, st);
            case 5: return launch_t<64, 5, FROM_MASK, HAS_SCORE>(a, smem, st);
            case 6: return launch_t<64, 6, FROM_MASK, HAS_SCORE>(a, smem, st);
            case 7: return launch_t<64, 7, FROM_MASK, HAS_SCORE>(a, smem, st);
            case 8: return launch_t<64, 8, FROM_MASK, HAS_SCORE>(a, smem, st);
            default: break;
        }
    }
    return launch_t<64, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
}

template <bool FROM_MASK, bool HAS_SCORE>
cudaError_t launch_v(int V, const PruneArgs& a, size_t smem, cudaStream_t st) {
    switch (V) {
        case 1: return launch_t<1, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 2: return launch_t<2, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 4: return launch_t<4, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 8: return launch_t<8, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 16: return launch_t<16, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 32: return launch_t<32, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 64: return launch_m64<FROM_MASK, HAS_SCORE>(a, smem, st);
        case 128: return launch_t<128, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        case 256: return launch_t<256, 0, FROM_MASK, HAS_SCORE>(a, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

// Host entry used by api.cpp.  Picks CB so that the tile fits in shared memory.
int launch_prune_pack(const PruneLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = *L.g;
    // V >= 32: the instruction-lean kernel (prune2.cu); VNM_PRUNE_V1=1 keeps this one (comparisons)
    static const bool v1 = [] { const char* e = getenv("VNM_PRUNE_V1"); return e && e[0] == '1'; }();
    if (!v1 && !L.mask_in) {
        const int rc = launch_prune2(L, stream);
        if (rc != kLaunchUnsupported) return rc;
    }
    if (L.values_tc && g.M > 8) {
        // the window-16 / M = 16 natural 2:4 forms are written fused by prune2 only: here the canonical arrays
        // first, then the form packed from them (pack_tc.cu; identical bytes)
        PruneLaunch Lc = L;
        Lc.values_tc = nullptr;
        Lc.meta_tc = nullptr;
        const int rc = launch_prune_pack(Lc, stream);
        if (rc) return rc;
        vnm_packed P;
        P.g = g;
        P.values = L.values;
        P.col_idx = L.col_idx;
        P.meta = L.meta;
        P.values_tc = L.values_tc;
        P.meta_tc = L.meta_tc;
        return g.M % 4 == 0 ? launch_pack_nat24(P, stream) : launch_pack_tc(P, stream);
    }
    const bool from_mask = L.mask_in != nullptr;
    const bool has_score = L.score != nullptr;
    int CB = 0;
    for (int cb : {32, 16, 8}) {
        if ((cb * g.M) % 32 != 0) continue;  // whole mask words per tile
        if (smem_bytes(g.V, g.M, cb, from_mask, has_score, L.values_tc != nullptr) > kMaxSmem) continue;
        CB = cb;
        break;
    }
    if (CB == 0) return kLaunchUnsupported;
    PruneArgs a;
    a.W = L.W; a.ldw = L.ldw; a.score = L.score; a.lds = L.lds;
    a.mask_in = L.mask_in; a.mask_out = L.mask_out;
    a.values = L.values; a.col_idx = L.col_idx; a.meta = L.meta; a.status = L.status;
    a.rows = g.rows; a.cols = g.cols; a.M = g.M; a.rows_p = g.rows_p; a.cols_p = g.cols_p;
    a.nb = g.nb; a.nb_pad = g.nb_pad; a.ld_val = g.ld_val; a.ld_meta = g.ld_meta; a.ld_mask = g.ld_mask;
    a.CB = CB;
    a.values_tc = L.values_tc;
    a.meta_tc = L.meta_tc;
    a.ld_tc = 0;
    a.n_stage_tc = 0;
    if (a.values_tc) {
        if (g.V != 64 || g.M > 8 || CB != 32 || !a.meta_tc) return kLaunchUnsupported;
        const int n_mma = g.nb_pad / (g.M == 4 ? 8 : 4);
        a.ld_tc = 16 * n_mma;
        a.n_stage_tc = (n_mma + 3) / 4;
        // rows of the last 128-row tile beyond rows_p: zero values, nibble 0x4 metadata
        const int rows_w = (g.rows_p + 127) / 128 * 128;
        if (rows_w > g.rows_p) {
            cudaMemsetAsync(a.values_tc + static_cast<int64_t>(g.rows_p) * a.ld_tc, 0,
                            static_cast<size_t>(rows_w - g.rows_p) * a.ld_tc * 2, stream);
            cudaMemset2DAsync(a.meta_tc + (static_cast<int64_t>(rows_w / 128 - 1) * a.n_stage_tc * 128 + 64) * 4, 2048,
                              0x44, 1024, a.n_stage_tc, stream);
        }
    }
    const size_t smem = smem_bytes(g.V, g.M, CB, from_mask, has_score, a.values_tc != nullptr);
    cudaError_t e;
    if (from_mask && a.status) {
        status_init_kernel<<<1, 1, 0, stream>>>(a.status);
        count_launch();
    }
    if (from_mask)
        e = launch_v<true, false>(g.V, a, smem, stream);
    else if (has_score)
        e = launch_v<false, true>(g.V, a, smem, stream);
    else
        e = launch_v<false, false>(g.V, a, smem, stream);
    if (e == cudaSuccess && from_mask && a.status) {
        status_fini_kernel<<<1, 1, 0, stream>>>(a.status);
        count_launch();
        e = cudaGetLastError();
    }
    return e == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace vnm
