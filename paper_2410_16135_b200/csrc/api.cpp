// api.cpp — the C ABI declared in include/vnm.h: host-side validation, geometry, dispatch.
// Every argument / shape / alignment error is returned before any launch; nothing here allocates
// device memory.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "vnm_internal.h"

namespace vnm {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace vnm

namespace {

// below this many tokens the weights dominate the traffic: the gather plan reads A_n (2 values / block),
// the window plan 4 values / block
constexpr int32_t kTcMinTokens = 64;

bool is_pow2(int32_t v) { return v > 0 && (v & (v - 1)) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
int32_t ceil_to(int32_t a, int32_t m) { return ((a + m - 1) / m) * m; }

bool same_geom(const vnm_geom& a, const vnm_geom& b) {
    return a.rows == b.rows && a.cols == b.cols && a.V == b.V && a.M == b.M && a.rows_p == b.rows_p &&
           a.cols_p == b.cols_p && a.nb == b.nb && a.nb_pad == b.nb_pad && a.ld_val == b.ld_val &&
           a.ld_meta == b.ld_meta && a.ld_mask == b.ld_mask;
}

vnm_status check_geom(const vnm_geom* g) {
    if (!g) return VNM_ERR_ARG;
    vnm_geom ref;
    if (vnm_geometry(g->rows, g->cols, g->V, g->M, &ref) != VNM_OK) return VNM_ERR_SHAPE;
    if (!same_geom(ref, *g)) return VNM_ERR_SHAPE;
    return VNM_OK;
}

vnm_status check_w(const uint16_t* W, int64_t ldw, const vnm_geom* g) {
    if (g->rows > 0 && g->cols > 0 && !W) return VNM_ERR_ARG;
    if (ldw < g->cols || ldw < 0) return VNM_ERR_SHAPE;
    if (W && (!aligned16(W) || (ldw % 8) != 0)) return VNM_ERR_ALIGN;
    return VNM_OK;
}

vnm_status check_score(const float* s, int64_t lds, const vnm_geom* g) {
    if (!s) return VNM_OK;
    if (lds < g->cols) return VNM_ERR_SHAPE;
    if (!aligned16(s) || (lds % 4) != 0) return VNM_ERR_ALIGN;
    return VNM_OK;
}

vnm_status check_packed(const vnm_packed* P, const vnm_geom* g) {
    if (!P) return VNM_ERR_ARG;
    if (!same_geom(P->g, *g)) return VNM_ERR_SHAPE;
    if (g->rows_p > 0 && g->nb_pad > 0 && (!P->values || !P->col_idx || !P->meta)) return VNM_ERR_ARG;
    if ((P->values && !aligned16(P->values)) || (P->col_idx && !aligned16(P->col_idx)) ||
        (P->meta && !aligned16(P->meta)))
        return VNM_ERR_ALIGN;
    return VNM_OK;
}

vnm_status from_launch(int rc) {
    if (rc == 0) return VNM_OK;
    if (rc == vnm::kLaunchUnsupported) return VNM_ERR_UNSUPPORTED;
    return VNM_ERR_CUDA;
}

}  // namespace

extern "C" {

vnm_status vnm_geometry(int32_t rows, int32_t cols, int32_t V, int32_t M, vnm_geom* out) {
    if (!out) return VNM_ERR_ARG;
    if (rows < 0 || cols < 0 || !is_pow2(V) || V > 256 || M < 4 || M > 32) return VNM_ERR_SHAPE;
    if (rows > (1 << 30) || cols > (1 << 30)) return VNM_ERR_SHAPE;
    vnm_geom g;
    g.rows = rows;
    g.cols = cols;
    g.V = V;
    g.M = M;
    g.rows_p = ceil_to(rows, V);
    g.cols_p = ceil_to(cols, M);
    g.nb = g.cols_p / M;
    g.nb_pad = ceil_to(g.nb, 8);
    g.ld_val = 2 * g.nb_pad;
    g.ld_meta = (g.nb_pad / 8 + 3) / 4 * 4;  // rows padded to 16 B (TMA-loadable), pad words 0x44444444
    g.ld_mask = (g.cols_p + 31) / 32;
    *out = g;
    return VNM_OK;
}

// Natural 2:4 tensor-core form (M % 4 == 0, M > 8; include/vnm.h): the masked W is 2:4-sparse in the natural
// channel order, so the window-form kernels run it as the M = 4 layout over 4-channel groups.
static bool nat24(const vnm_geom* g) { return g->M > 8 && g->M % 4 == 0 && g->V >= 32 && g->V <= 128; }
// the tensor-core form is written by the prune pass itself (window, window-16, and the natural 2:4 form at M = 16);
// the other natural 2:4 forms are packed by a second launch
static bool tc_fused(const vnm_geom* g) { return !nat24(g) || g->M == 16; }
// Window-16 form (8 < M < 16, M % 4 != 0; include/vnm.h): 16-channel windows, two MMAs per 4 blocks — e.g. the
// paper's 128:2:9 / 10 / 11 / 13 (tab:bs-sped) at prefill sizes
static bool w16(const vnm_geom* g) { return g->M > 8 && g->M < 16 && g->M % 4 != 0 && g->V >= 32 && g->V <= 128; }
// the tensor-core form applies: window form (M <= 8), natural 2:4 form (M % 4 == 0) or window-16 form
static bool tc_geom(const vnm_geom* g) {
    return g->V >= 32 && g->V <= 128 && (g->M <= 8 || g->M % 4 == 0 || w16(g));
}
// the M = 4 view of a natural-2:4 geometry: blocks = 4-channel groups
static vnm_geom view4(const vnm_geom& g) {
    vnm_geom v = g;
    v.M = 4;
    v.nb = g.cols_p / 4;
    v.nb_pad = (v.nb + 7) / 8 * 8;
    v.ld_val = 2 * v.nb_pad;
    v.ld_meta = v.nb_pad / 8;
    return v;
}

size_t vnm_bytes(const vnm_geom* g, int which) {
    if (check_geom(g) != VNM_OK) return 0;
    const size_t rp = static_cast<size_t>(g->rows_p);
    switch (which) {
        case 0: return rp * static_cast<size_t>(g->ld_val) * 2;
        case 1: return rp / static_cast<size_t>(g->V) * static_cast<size_t>(g->nb_pad) * 4;
        case 2: return rp * static_cast<size_t>(g->ld_meta) * 4;
        case 3: return rp * static_cast<size_t>(g->ld_mask) * 4;
        case 4:
        case 5: {
            if (!tc_geom(g)) return 0;
            const size_t rows_w = (rp + 127) / 128 * 128;
            const vnm_geom gv = nat24(g) ? view4(*g) : *g;
            const size_t bpm = gv.M == 4 ? 8 : 4;
            // window-16 form: two MMAs (half-windows) per 4 blocks
            const size_t n_mma = w16(g) ? static_cast<size_t>(gv.nb_pad) / 2 : static_cast<size_t>(gv.nb_pad) / bpm;
            const size_t n_stage = (n_mma + 3) / 4;
            return which == 4 ? rows_w * 16 * n_mma * 2 : rows_w / 128 * n_stage * 128 * 4 * 4;
        }
        default: return 0;
    }
}

vnm_status vnm_prune(const uint16_t* W, int64_t ldw, const float* score, int64_t lds, const vnm_geom* g,
                     uint32_t* mask, vnm_stream_t stream) {
    vnm_status s = check_geom(g);
    if (s) return s;
    if ((s = check_w(W, ldw, g))) return s;
    if ((s = check_score(score, lds, g))) return s;
    if (g->rows_p == 0 || g->ld_mask == 0) return VNM_OK;
    if (!mask) return VNM_ERR_ARG;
    if (!aligned16(mask)) return VNM_ERR_ALIGN;
    if (!W && !score) return VNM_ERR_ARG;
    vnm::PruneLaunch L{g, W, ldw, score, lds, nullptr, mask, nullptr, nullptr, nullptr, nullptr};
    if (!W) return VNM_ERR_ARG;
    return from_launch(vnm::launch_prune_pack(L, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_compress(const uint16_t* W, int64_t ldw, const uint32_t* mask, const vnm_geom* g, vnm_packed* out,
                        int32_t* d_status, vnm_stream_t stream) {
    vnm_status s = check_geom(g);
    if (s) return s;
    if ((s = check_w(W, ldw, g))) return s;
    if ((s = check_packed(out, g))) return s;
    if (g->rows_p == 0 || g->nb_pad == 0) {
        if (d_status) cudaMemsetAsync(d_status, 0, sizeof(int32_t), reinterpret_cast<cudaStream_t>(stream));
        return VNM_OK;
    }
    if (!mask || !W) return VNM_ERR_ARG;
    if (!aligned16(mask)) return VNM_ERR_ALIGN;
    if (d_status && (reinterpret_cast<uintptr_t>(d_status) & 3u)) return VNM_ERR_ALIGN;
    vnm::PruneLaunch L{g, W, ldw, nullptr, 0, mask, nullptr, out->values, out->col_idx, out->meta, d_status};
    return from_launch(vnm::launch_prune_pack(L, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_prune_compress(const uint16_t* W, int64_t ldw, const float* score, int64_t lds, const vnm_geom* g,
                              vnm_packed* out, uint32_t* mask, vnm_stream_t stream) {
    vnm_status s = check_geom(g);
    if (s) return s;
    if ((s = check_w(W, ldw, g))) return s;
    if ((s = check_score(score, lds, g))) return s;
    if ((s = check_packed(out, g))) return s;
    if (mask && !aligned16(mask)) return VNM_ERR_ALIGN;
    if (g->rows_p == 0 || g->nb_pad == 0) return VNM_OK;
    if (!W) return VNM_ERR_ARG;
    vnm::PruneLaunch L{g, W, ldw, score, lds, nullptr, mask, out->values, out->col_idx, out->meta, nullptr};
    if (out->values_tc || out->meta_tc) {  // tensor-core form (include/vnm.h): fused window form (M <= 8) or
        if (!tc_geom(g)) return VNM_ERR_UNSUPPORTED;  // the natural 2:4 form packed after the pass (M % 4 == 0)
        if (!out->values_tc || !out->meta_tc) return VNM_ERR_ARG;
        if (!aligned16(out->values_tc) || !aligned16(out->meta_tc)) return VNM_ERR_ALIGN;
        if (tc_fused(g)) {
            L.values_tc = out->values_tc;
            L.meta_tc = out->meta_tc;
        }
    }
    const vnm_status st = from_launch(vnm::launch_prune_pack(L, reinterpret_cast<cudaStream_t>(stream)));
    if (st || !out->values_tc || tc_fused(g)) return st;
    return from_launch(vnm::launch_pack_nat24(*out, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_prune_compress_batched(int32_t n, const uint16_t* const* W, const int64_t* ldw,
                                      const float* const* score, const int64_t* lds, vnm_packed* const* out,
                                      uint32_t* const* mask, vnm_stream_t stream) {
    if (n < 1 || n > 64 || !W || !ldw || !out) return VNM_ERR_ARG;
    vnm::PruneLaunch Ls[64];
    int live = 0;
    bool same = true;
    for (int i = 0; i < n; ++i) {
        if (!out[i]) return VNM_ERR_ARG;
        const vnm_geom* g = &out[i]->g;
        const float* sc = score ? score[i] : nullptr;
        const int64_t ls = lds ? lds[i] : 0;
        uint32_t* mk = mask ? mask[i] : nullptr;
        vnm_status s = check_geom(g);
        if (s) return s;
        if ((s = check_w(W[i], ldw[i], g))) return s;
        if ((s = check_score(sc, ls, g))) return s;
        if ((s = check_packed(out[i], g))) return s;
        if (mk && !aligned16(mk)) return VNM_ERR_ALIGN;
        if (g->rows_p == 0 || g->nb_pad == 0) continue;
        if (!W[i]) return VNM_ERR_ARG;
        vnm::PruneLaunch L{g, W[i], ldw[i], sc, ls, nullptr, mk, out[i]->values, out[i]->col_idx, out[i]->meta, nullptr};
        if (out[i]->values_tc || out[i]->meta_tc) {
            if (!tc_geom(g)) return VNM_ERR_UNSUPPORTED;
            if (!out[i]->values_tc || !out[i]->meta_tc) return VNM_ERR_ARG;
            if (!aligned16(out[i]->values_tc) || !aligned16(out[i]->meta_tc)) return VNM_ERR_ALIGN;
            if (tc_fused(g)) {
                L.values_tc = out[i]->values_tc;
                L.meta_tc = out[i]->meta_tc;
            }
        }
        if (live > 0 && (g->V != Ls[0].g->V || g->M != Ls[0].g->M)) same = false;
        Ls[live++] = L;
    }
    if (live == 0) return VNM_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    bool done = false;
    if (same && live <= 8) {
        const int rc = vnm::launch_prune2_batch(Ls, live, st);
        if (rc != vnm::kLaunchUnsupported) {
            if (rc) return from_launch(rc);
            done = true;
        }
    }
    for (int i = 0; i < live && !done; ++i) {
        const vnm_status s = from_launch(vnm::launch_prune_pack(Ls[i], st));
        if (s) return s;
    }
    for (int i = 0; i < n; ++i)  // natural 2:4 tensor-core forms, packed after the pass
        if (out[i]->values_tc && !tc_fused(&out[i]->g) && out[i]->g.rows_p > 0 && out[i]->g.nb_pad > 0) {
            const vnm_status s = from_launch(vnm::launch_pack_nat24(*out[i], st));
            if (s) return s;
        }
    return VNM_OK;
}

vnm_status vnm_pack_tc(const vnm_packed* P, vnm_stream_t stream) {
    if (!P) return VNM_ERR_ARG;
    const vnm_geom* g = &P->g;
    vnm_status s = check_geom(g);
    if (s) return s;
    if ((s = check_packed(P, g))) return s;
    if (!tc_geom(g)) return VNM_ERR_UNSUPPORTED;
    if (g->rows_p == 0 || g->nb_pad == 0) return VNM_OK;
    if (!P->values_tc || !P->meta_tc) return VNM_ERR_ARG;
    if (!aligned16(P->values_tc) || !aligned16(P->meta_tc)) return VNM_ERR_ALIGN;
    if (nat24(g)) return from_launch(vnm::launch_pack_nat24(*P, reinterpret_cast<cudaStream_t>(stream)));
    return from_launch(vnm::launch_pack_tc(*P, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_spmm(const uint16_t* XT, int64_t ldx, int32_t T, const vnm_packed* P, void* YT, int64_t ldy,
                    vnm_dtype y_dtype, void* workspace, size_t workspace_bytes, vnm_stream_t stream) {
    if (!P) return VNM_ERR_ARG;
    const vnm_geom* g = &P->g;
    vnm_status s = check_geom(g);
    if (s) return s;
    if ((s = check_packed(P, g))) return s;
    if (y_dtype != VNM_F32 && y_dtype != VNM_BF16) return VNM_ERR_ARG;
    if (T < 0 || ldx < T || ldy < T) return VNM_ERR_SHAPE;
    // tensor-core form: 32 <= V <= 128 with M <= 8 (window form) or M % 4 == 0 (natural 2:4 form; the kernels
    // see its M = 4 view); small-T plan (T <= 32): any V >= 16, any M, canonical arrays; gather plan: V = 64
    const bool tc_form = P->values_tc && P->meta_tc && tc_geom(g);
    const bool small = vnm::spmm_smallt_applies(*g, T);
    if (g->V < 64 && !tc_form && !small) return VNM_ERR_UNSUPPORTED;  // gather plan: V = 64, 128, 256
    if (T == 0 || g->rows == 0) return VNM_OK;
    if (!YT) return VNM_ERR_ARG;
    if (g->cols > 0 && !XT) return VNM_ERR_ARG;
    if ((XT && !aligned16(XT)) || !aligned16(YT) || (ldx % 8) != 0 || (ldy % 8) != 0) return VNM_ERR_ALIGN;
    if (workspace && !aligned16(workspace)) return VNM_ERR_ALIGN;
    vnm::SpmmLaunch L{P, XT, ldx, T, YT, ldy, y_dtype, workspace, workspace ? workspace_bytes : 0};
    const bool tc = tc_form && g->nb_pad > 0 && (T > kTcMinTokens || (!small && g->V < 64));
    if (tc && (!aligned16(P->values_tc) || !aligned16(P->meta_tc))) return VNM_ERR_ALIGN;
    vnm_packed Pv;
    if (tc && nat24(g)) {  // the natural 2:4 form runs as the M = 4 layout over 4-channel groups
        Pv = *P;
        Pv.g = view4(*g);
        L.P = &Pv;
        g = &Pv.g;
    }
    if (tc) {
        // Measured (profiles/r01b_*): the CTA-pair kernel wins for long K with an even number of 128-row tiles
        // (Llama layers, DeiT-B fc2) — tensor-bound; the single-CTA kernel wins for short K / HBM-bound shapes
        // (DeiT qkv / proj / fc1), where its deeper X^T prefetch and finer tiles matter more.
        // VNM_TC_PLAN=1 / 2 forces the single-CTA / pair kernel (comparisons).
        static const int force = [] { const char* e = getenv("VNM_TC_PLAN"); return e ? atoi(e) : 0; }();
        const int n_stage = (g->nb_pad / (g->M == 4 ? 8 : 4) + 3) / 4, n_rt = (g->rows_p + 127) / 128;
        // CTA pairs with the row pair's A resident (spmm_tc3.cu): measured faster for short K, M <= 6 and >= 6
        // row tiles at large T (DeiT-S qkv / fc1: profiles/r01c_probes.md); slower for M = 8 and 3-row-tile
        // layers, where the single-CTA kernel stays.
        const int n_mma = g->nb_pad / (g->M == 4 ? 8 : 4);
        // The single-CTA / pair kernels store Y^T with TMA, whose stores are whole 16-byte chunks: a row of Y^T that
        // is not a multiple of 16 bytes (T % 8 bf16 / T % 4 fp32) would get up to 7 tokens past T written.  Those
        // shapes take the resident / streamed pair kernel (st.global with element-wise tails; tests/test_gpu_bounds.py).
        const bool ragged = (static_cast<int64_t>(T) * (y_dtype == VNM_BF16 ? 2 : 4)) % 16 != 0;
        // the window-16 form runs in the single-CTA / pair kernels only (the resident pair kernel has no
        // half-window stepping): a ragged Y^T row then takes the small-T or gather plan below
        const bool win16 = g->M > 8;
        const bool tc3 = !win16 && (ragged || (force ? force >= 3 : (g->M >= 5 && g->M <= 6 && n_rt >= 6 && n_mma <= 32 && T >= 8192)));
        if (ragged && !win16) {
            const int rc = vnm::launch_spmm_tc3(L, -1, reinterpret_cast<cudaStream_t>(stream));
            if (rc != vnm::kLaunchUnsupported) return from_launch(rc);
            return VNM_ERR_UNSUPPORTED;
        }
        if (tc3) {  // VNM_TC_PLAN=4: the same kernel with A streamed
            const int rc = vnm::launch_spmm_tc3(L, force == 4 ? 0 : (force == 3 ? -1 : 1), reinterpret_cast<cudaStream_t>(stream));
            if (rc != vnm::kLaunchUnsupported) return from_launch(rc);
        }
        if (!(win16 && ragged)) {
            const int n_stage16 = win16 ? (g->nb_pad / 2 + 3) / 4 : n_stage;
            const bool pair = force ? force == 2 : (n_stage16 >= 12 && n_rt % 2 == 0);
            if (pair) return from_launch(vnm::launch_spmm_tc2(L, reinterpret_cast<cudaStream_t>(stream)));
            return from_launch(vnm::launch_spmm_tc(L, reinterpret_cast<cudaStream_t>(stream)));
        }
        if (!small && g->V != 64 && g->V != 128 && g->V != 256) return VNM_ERR_UNSUPPORTED;
    }
    if (small) return from_launch(vnm::launch_spmm_smallt(L, reinterpret_cast<cudaStream_t>(stream)));
    return from_launch(vnm::launch_spmm(L, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_spmm_batched(int32_t n, const uint16_t* const* XT, const int64_t* ldx, int32_t T,
                            const vnm_packed* const* P, void* const* YT, const int64_t* ldy, vnm_dtype y_dtype,
                            uint32_t flags, void* workspace, size_t workspace_bytes, vnm_stream_t stream) {
    if (n < 1 || n > 64 || !XT || !ldx || !P || !YT || !ldy) return VNM_ERR_ARG;
    if (flags & ~static_cast<uint32_t>(VNM_SPMM_WEIGHTS_READY)) return VNM_ERR_ARG;
    if (y_dtype != VNM_F32 && y_dtype != VNM_BF16) return VNM_ERR_ARG;
    if (workspace && !aligned16(workspace)) return VNM_ERR_ALIGN;
    // validate every problem as vnm_spmm does before launching anything
    for (int i = 0; i < n; ++i) {
        if (!P[i]) return VNM_ERR_ARG;
        const vnm_geom* g = &P[i]->g;
        vnm_status s = check_geom(g);
        if (s) return s;
        if ((s = check_packed(P[i], g))) return s;
        if (T < 0 || ldx[i] < T || ldy[i] < T) return VNM_ERR_SHAPE;
        if (T == 0 || g->rows == 0) continue;
        if (!YT[i] || (g->cols > 0 && !XT[i])) return VNM_ERR_ARG;
        if ((XT[i] && !aligned16(XT[i])) || !aligned16(YT[i]) || (ldx[i] % 8) != 0 || (ldy[i] % 8) != 0) return VNM_ERR_ALIGN;
    }
    // groups of up to 4 consecutive problems in one small-T launch when they all take the small-T plan (T <= 32:
    // the window form is never used there); anything else is one vnm_spmm per problem (same stream order)
    for (int c = 0; c < n; c += 4) {
        const int m = n - c < 4 ? n - c : 4;
        const vnm_geom* gs[4];
        vnm::SpmmLaunch Ls[4];
        int live = 0;
        bool one = true;
        for (int i = c; i < c + m; ++i) {
            if (T == 0 || P[i]->g.rows == 0) continue;
            gs[live] = &P[i]->g;
            Ls[live] = vnm::SpmmLaunch{P[i], XT[i], ldx[i], T, YT[i], ldy[i], y_dtype, workspace, workspace ? workspace_bytes : 0};
            if (P[i]->g.nb_pad == 0) one = false;  // (K = 0: vnm_spmm writes zeros)
            ++live;
        }
        if (live == 0) continue;
        one = one && vnm::spmm_smallt_batch_applies(gs, live, T);
        if (one) {
            const vnm_status s =
                from_launch(vnm::launch_spmm_smallt_batch(Ls, live, flags, reinterpret_cast<cudaStream_t>(stream)));
            if (s) return s;
            continue;
        }
        for (int i = c; i < c + m; ++i) {
            const vnm_status s = vnm_spmm(XT[i], ldx[i], T, P[i], YT[i], ldy[i], y_dtype, workspace, workspace_bytes, stream);
            if (s) return s;
        }
    }
    return VNM_OK;
}

size_t vnm_spmm_batched_workspace_bytes(int32_t n, const vnm_geom* const* g, int32_t T) {
    if (n < 1 || n > 64 || !g || T < 0) return 0;
    size_t b = 0;
    for (int c = 0; c < n; c += 4) {
        const int m = n - c < 4 ? n - c : 4;
        for (int i = c; i < c + m; ++i) {
            if (!g[i] || check_geom(g[i]) != VNM_OK) return 0;
            const size_t o = vnm_spmm_workspace_bytes(g[i], T);
            b = o > b ? o : b;
        }
        const size_t o = vnm::spmm_smallt_batch_workspace_bytes(g + c, m, T);
        b = o > b ? o : b;
    }
    return b;
}

vnm_status vnm_spmm_workspace_init(void* ws, size_t bytes, vnm_stream_t stream) {
    if (bytes == 0) return VNM_OK;
    if (!ws) return VNM_ERR_ARG;
    return cudaMemsetAsync(ws, 0, bytes, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? VNM_OK : VNM_ERR_CUDA;
}

size_t vnm_spmm_workspace_bytes(const vnm_geom* g, int32_t T) {
    if (check_geom(g) != VNM_OK || T < 0) return 0;
    // the largest workspace any plan for (g, T) can use (the tickets / flags sit at offset 0 in every plan)
    const size_t b = vnm::spmm_smallt_workspace_bytes(*g, T), o = vnm::spmm_workspace_bytes(*g, T);
    return b > o ? b : o;
}

vnm_status vnm_act_norms(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, float* norms, vnm_stream_t stream) {
    if (cols < 0 || T < 0 || ldx < T) return VNM_ERR_SHAPE;
    if (cols == 0) return VNM_OK;
    if (!norms || (T > 0 && !XT)) return VNM_ERR_ARG;
    if ((XT && !aligned16(XT)) || (reinterpret_cast<uintptr_t>(norms) & 3u)) return VNM_ERR_ALIGN;
    return from_launch(vnm::launch_act_norms(XT, ldx, cols, T, norms, reinterpret_cast<cudaStream_t>(stream)));
}

size_t vnm_ria_workspace_bytes(int32_t rows, int32_t cols) {
    if (rows < 0 || cols < 0) return 0;
    return vnm::ria_workspace_bytes(rows, cols);
}

vnm_status vnm_ria_score(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, const float* act_norms, float a,
                         float* score, int64_t lds, void* workspace, size_t workspace_bytes, vnm_stream_t stream) {
    if (rows < 0 || cols < 0 || ldw < cols || lds < cols || !(a >= 0.f)) return VNM_ERR_SHAPE;
    if (rows == 0 || cols == 0) return VNM_OK;
    if (!W || !score || !workspace) return VNM_ERR_ARG;
    if (workspace_bytes < vnm::ria_workspace_bytes(rows, cols)) return VNM_ERR_SHAPE;
    if (!aligned16(W) || (ldw % 8) != 0 || !aligned16(score) || (lds % 4) != 0 || !aligned16(workspace) ||
        (act_norms && (reinterpret_cast<uintptr_t>(act_norms) & 3u)))
        return VNM_ERR_ALIGN;
    return from_launch(vnm::launch_ria(W, ldw, rows, cols, act_norms, a, score, lds, workspace,
                                       reinterpret_cast<cudaStream_t>(stream)));
}

size_t vnm_permute_gain_workspace_bytes(const vnm_geom* g) {
    if (check_geom(g) != VNM_OK) return 0;
    return vnm::permute_gain_workspace_bytes(*g);
}

vnm_status vnm_permute_gain(const float* score, int64_t lds, const vnm_geom* g, float* cost, int64_t ldc,
                            void* workspace, size_t workspace_bytes, vnm_stream_t stream) {
    vnm_status s = check_geom(g);
    if (s) return s;
    if (g->V > 128) return VNM_ERR_UNSUPPORTED;
    if (lds < g->cols || ldc < g->cols_p) return VNM_ERR_SHAPE;
    if (g->rows == 0 || g->cols == 0) return VNM_OK;
    if (!score || !cost || !workspace) return VNM_ERR_ARG;
    if (workspace_bytes < vnm::permute_gain_workspace_bytes(*g)) return VNM_ERR_SHAPE;
    if ((reinterpret_cast<uintptr_t>(score) & 3u) || (reinterpret_cast<uintptr_t>(cost) & 3u) || !aligned16(workspace))
        return VNM_ERR_ALIGN;
    return from_launch(vnm::launch_permute_gain(score, lds, *g, cost, ldc, workspace, reinterpret_cast<cudaStream_t>(stream)));
}

vnm_status vnm_permute_gain_out(const float* score, int64_t lds, const vnm_geom* g, float* cost, int64_t ldc,
                                vnm_stream_t stream) {
    vnm_status s = check_geom(g);
    if (s) return s;
    if (g->V > 128) return VNM_ERR_UNSUPPORTED;
    if (lds < g->cols || ldc < g->rows_p) return VNM_ERR_SHAPE;
    if (g->rows == 0 || g->cols == 0) return VNM_OK;
    if (!score || !cost) return VNM_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(score) & 3u) || (reinterpret_cast<uintptr_t>(cost) & 3u)) return VNM_ERR_ALIGN;
    return from_launch(vnm::launch_permute_gain_out(score, lds, *g, cost, ldc, reinterpret_cast<cudaStream_t>(stream)));
}

const char* vnm_status_string(vnm_status s) {
    switch (s) {
        case VNM_OK: return "ok";
        case VNM_ERR_ARG: return "invalid argument (null pointer or bad enum)";
        case VNM_ERR_SHAPE: return "shape out of range (V, M, rows, cols, T or leading dimension)";
        case VNM_ERR_ALIGN: return "misaligned pointer or leading dimension";
        case VNM_ERR_UNSUPPORTED: return "configuration not supported by this build";
        case VNM_ERR_CUDA: return "CUDA launch / driver error";
        default: return "unknown status";
    }
}

uint64_t vnm_launch_count(void) { return vnm::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
