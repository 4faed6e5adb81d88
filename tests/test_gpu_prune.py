"""GPU parity for the mask + compression pass (§8 rows a1-a5): bit-exact against the oracle.

Calls go through the C ABI (paper_2410_16135_b200.vnm -> libvnm.so)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import packed_np, to_dev_bf16, to_dev_f32, u32

pytestmark = pytest.mark.gpu

SMALL = [
    # rows, cols, V, M, kind
    (128, 64, 64, 8, "int"),       # BJ config 1 (tie-heavy variant)
    (128, 64, 64, 8, "normal"),    # BJ config 1
    (70, 23, 64, 5, "normal"),     # ragged rows and cols
    (200, 333, 16, 7, "wide"),
    (37, 50, 1, 4, "int"),
    (64, 96, 2, 6, "normal"),
    (300, 1000, 128, 16, "outlier"),
    (96, 200, 32, 13, "int"),
    (40, 120, 8, 9, "wide"),
    (260, 256, 256, 4, "normal"),
    (128, 4096, 4, 32, "normal"),
    (1152, 384, 64, 5, "normal"),  # DeiT-S qkv
]


def run_all(W, V, M, score=None):
    rows, cols = W.shape
    Wd = to_dev_bf16(W)
    Sd = to_dev_f32(score) if score is not None else None
    mask_d = vnm.prune(Wd, V, M, score=Sd)
    P, mask2_d = vnm.prune_compress(Wd, V, M, score=Sd, want_mask=True)
    torch.cuda.synchronize()
    return u32(mask_d), u32(mask2_d), packed_np(P), Wd


def check(W, V, M, score=None):
    mask_ref = oracle.prune(W, V, M, score=score)
    st, v_ref, c_ref, m_ref = oracle.pack(W, mask_ref, V, M)
    assert st == 0
    mask, mask2, (v, c, m), Wd = run_all(W, V, M, score)
    assert np.array_equal(mask, mask_ref), "vnm_prune mask"
    assert np.array_equal(mask2, mask_ref), "vnm_prune_compress mask"
    assert np.array_equal(v, v_ref), "A_n values"
    assert np.array_equal(c, c_ref), "A_i1 col_idx"
    assert np.array_equal(m, m_ref), "A_i2 meta"
    # vnm_compress from the oracle's mask gives the same bytes
    status = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    P3 = vnm.compress(Wd, torch.from_numpy(mask_ref.view(np.int32)).cuda(), V, M, status=status)
    v3, c3, m3 = packed_np(P3)
    assert int(status.item()) == 0
    assert np.array_equal(v3, v_ref) and np.array_equal(c3, c_ref) and np.array_equal(m3, m_ref)


@pytest.mark.parametrize("rows,cols,V,M,kind", SMALL)
def test_prune_compress_bitexact(rows, cols, V, M, kind):
    W = synth.weights(rows, cols, seed=rows * 7 + cols + V + M, kind=kind)
    check(W, V, M)


@pytest.mark.parametrize("rows,cols,V,M,kind", [(128, 64, 64, 8, "uniform"), (70, 23, 64, 5, "signed"),
                                                (300, 1000, 128, 16, "int"), (37, 50, 1, 4, "uniform")])
def test_score_path_bitexact(rows, cols, V, M, kind):
    W = synth.weights(rows, cols, seed=3)
    S = synth.scores(rows, cols, seed=4, kind=kind)
    check(W, V, M, score=S)


@pytest.mark.parametrize("rows,cols,M", [(11008, 4096, 5), (4096, 11008, 5), (4096, 4096, 5), (3072, 768, 8),
                                         (768, 3072, 8), (2304, 768, 8), (1536, 384, 5), (384, 1536, 5)])
def test_bj_weight_shapes_bitexact(rows, cols, M):
    """Every weight shape of BJ configs 2-5 at its (V, M), full outputs compared byte for byte."""
    W = synth.weights(rows, cols, seed=synth.seed(4, 0) + rows, kind="outlier")
    check(W, 64, M)


@pytest.mark.parametrize("M", [4, 6, 7, 16])
def test_llama_mlp_m_sweep(M):
    W = synth.weights(11008, 4096, seed=M, kind="normal")
    check(W, 64, M)


def test_invalid_mask_status():
    V, M = 64, 5
    W = synth.weights(128, 80, seed=5)
    mask = oracle.prune(W, V, M)
    g = oracle.geometry(128, 80, V, M)
    Wd = to_dev_bf16(W)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    # third bit in row 70 (V-block 1), block 9
    bad = mask.copy()
    dense = np.unpackbits(bad.view(np.uint8).reshape(128, -1), axis=1, bitorder="little")
    c = [c for c in range(45, 50) if not dense[70, c]][0]
    bad[70, c // 32] |= np.uint32(1 << (c % 32))
    vnm.compress(Wd, torch.from_numpy(bad.view(np.int32)).cuda(), V, M, status=status)
    exp, *_ = oracle.pack(W, bad, V, M)
    assert int(status.item()) == exp == 1 + 1 * g["nb"] + 9
    # a bit beyond cols_p (cols_p = 80 -> word 2 bit 16 = column 80)
    bad2 = mask.copy()
    bad2[3, 2] |= np.uint32(1 << 16)
    vnm.compress(Wd, torch.from_numpy(bad2.view(np.int32)).cuda(), V, M, status=status)
    exp2, *_ = oracle.pack(W, bad2, V, M)
    assert int(status.item()) == exp2 == 1 + 2 * g["nb"]


def test_determinism():
    W = synth.weights(4096, 4096, seed=1, kind="outlier")
    Wd = to_dev_bf16(W)
    a = packed_np(vnm.prune_compress(Wd, 64, 5))
    b = packed_np(vnm.prune_compress(Wd, 64, 5))
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_strided_input():
    """W with a leading dimension larger than cols (a view into a bigger buffer)."""
    W = synth.weights(192, 100, seed=9)
    Wd = to_dev_bf16(W, ld=136)
    assert Wd.stride(0) == 136
    mask = u32(vnm.prune(Wd, 64, 5))
    assert np.array_equal(mask, oracle.prune(W, 64, 5))


@pytest.mark.parametrize("rows,cols,M", [(128, 512, 5), (192, 333, 8), (70, 90, 4), (300, 1000, 6), (64, 257, 7),
                                         (4096, 4096, 5)])
def test_window_form_fused_equals_standalone(rows, cols, M):
    """vnm_prune_compress writing values_tc / meta_tc in the same pass == vnm_pack_tc of its canonical output."""
    W = synth.weights(rows, cols, seed=rows + cols + M)
    Wd = to_dev_bf16(W)
    P = vnm.prune_compress(Wd, 64, M, tc=True)
    Q = vnm.prune_compress(Wd, 64, M)
    vnm.pack_tc(Q)
    torch.cuda.synchronize()
    assert torch.equal(P.values.view(torch.int16), Q.values.view(torch.int16))
    assert torch.equal(P.values_tc.view(torch.int16), Q.values_tc.view(torch.int16))
    assert torch.equal(P.meta_tc, Q.meta_tc)


@pytest.mark.parametrize("V", [32, 128])
@pytest.mark.parametrize("rows,cols,M", [(256, 640, 5), (300, 333, 8), (128, 100, 4), (512, 1000, 7)])
def test_window_form_fused_any_v(V, rows, cols, M):
    """Window form written by the fused pass for V != 64 == vnm_pack_tc of the canonical output."""
    W = synth.weights(rows, cols, seed=rows + cols + M + V)
    Wd = to_dev_bf16(W)
    P = vnm.prune_compress(Wd, V, M, tc=True)
    Q = vnm.prune_compress(Wd, V, M)
    vnm.pack_tc(Q)
    torch.cuda.synchronize()
    assert torch.equal(P.values_tc.view(torch.int16), Q.values_tc.view(torch.int16))
    assert torch.equal(P.meta_tc, Q.meta_tc)
    mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, V, M)
    v, c, m = packed_np(P)
    assert np.array_equal(v, v_ref) and np.array_equal(c, c_ref) and np.array_equal(m, m_ref)


@pytest.mark.parametrize("V,M,kind", [(64, 5, "normal"), (128, 6, "int"), (32, 9, "wide"), (256, 4, "outlier"),
                                      (64, 16, "int"), (128, 32, "normal")])
def test_llama_scale_bitexact(V, M, kind):
    """Full-width weight (4096 x 4096-ish, ragged) through the V >= 32 kernel, every byte vs the oracle."""
    W = synth.weights(4160 if V <= 64 else 4096, 4100, seed=V * 31 + M, kind=kind)
    check(W, V, M)


@pytest.mark.parametrize("shapes,V,M,tc", [
    ([(1152, 384), (384, 384), (1536, 384), (384, 1536)], 64, 5, True),   # the DeiT-S layers (one launch)
    ([(2304, 768), (768, 768), (3072, 768), (768, 3072)], 64, 8, True),   # DeiT-B
    ([(70, 23), (128, 64), (200, 333)], 64, 7, False),                    # ragged
    ([(256, 640), (128, 100)], 32, 6, True),
    ([(96, 200), (40, 120)], 8, 9, False),                                # not the batched kernel: n launches
])
def test_batched_equals_single(shapes, V, M, tc):
    """vnm_prune_compress_batched == one vnm_prune_compress per weight, byte for byte (masks, A_n, A_i1, A_i2,
    window form), and the first weight == the oracle."""
    Ws = [synth.weights(r, c, seed=r + 3 * c + M) for r, c in shapes]
    Wd = [to_dev_bf16(W) for W in Ws]
    Ps, masks = vnm.prune_compress_batched(Wd, V, M, want_mask=True, tc=tc)
    for W, P, mk in zip(Wd, Ps, masks):
        Q, mq = vnm.prune_compress(W, V, M, want_mask=True, tc=tc)
        torch.cuda.synchronize()
        assert torch.equal(mk, mq)
        for a, b in zip(packed_np(P), packed_np(Q)):
            assert np.array_equal(a, b)
        if tc:
            assert torch.equal(P.values_tc.view(torch.int16), Q.values_tc.view(torch.int16))
            assert torch.equal(P.meta_tc, Q.meta_tc)
    mask_ref = oracle.prune(Ws[0], V, M)
    assert np.array_equal(u32(masks[0]), mask_ref)


def test_batched_with_scores():
    Ws = [synth.weights(r, c, seed=r + c) for r, c in [(256, 500), (192, 320)]]
    Ss = [np.abs(synth.weights(r, c, seed=r * c)).astype(np.float32) * 3 for r, c in [(256, 500), (192, 320)]]
    Ps = vnm.prune_compress_batched([to_dev_bf16(W) for W in Ws], 64, 6, scores=[to_dev_f32(S) for S in Ss])
    torch.cuda.synchronize()
    for W, S, P in zip(Ws, Ss, Ps):
        mask_ref = oracle.prune(W, 64, 6, score=S)
        st, v_ref, c_ref, m_ref = oracle.pack(W, mask_ref, 64, 6)
        v, c, m = packed_np(P)
        assert np.array_equal(v, v_ref) and np.array_equal(c, c_ref) and np.array_equal(m, m_ref)


@pytest.mark.parametrize("V", [64, 128])
@pytest.mark.parametrize("rows,cols,M", [(256, 640, 16), (200, 333, 12), (130, 4096, 16), (64, 96, 32)])
def test_natural_24_form_pack(V, rows, cols, M):
    """M % 4 == 0, M > 8: vnm_prune_compress(tc) == vnm_pack_tc of its canonical output, and the natural 2:4
    form holds exactly the masked weights: 2 values per 4-channel group, zero-completed (values_tc rows read
    back through the group nibbles == the oracle's masked W)."""
    W = synth.weights(rows, cols, seed=rows + cols + M + V)
    Wd = to_dev_bf16(W)
    P = vnm.prune_compress(Wd, V, M, tc=True)
    Q = vnm.prune_compress(Wd, V, M)
    vnm.pack_tc(Q)
    batched = vnm.prune_compress_batched([Wd, Wd], V, M, tc=True)
    torch.cuda.synchronize()
    for R in (Q, *batched):
        assert torch.equal(P.values_tc.view(torch.int16), R.values_tc.view(torch.int16))
        assert torch.equal(P.meta_tc, R.meta_tc)
    # decode the M = 4 view on the host: values_tc [rows_w][2*ng_pad] with the group nibbles in meta_tc's
    # lane order (lane L: rows (L%8)+16(L/16) and +8, half h = (L/8)%2 of the 8 group nibbles of MMA k)
    g = P.g
    ng_pad = (g.cols_p // 4 + 7) // 8 * 8
    n_mma = ng_pad // 8
    n_stage = (n_mma + 3) // 4
    rows_w = (g.rows_p + 127) // 128 * 128
    vals = P.values_tc.view(torch.int16).cpu().numpy().view(np.uint16).reshape(rows_w, 2 * ng_pad)
    mt = P.meta_tc.cpu().numpy().view(np.uint32).reshape(rows_w // 128, n_stage, 128, 4)
    dense = np.zeros((rows_w, 4 * ng_pad), np.uint16)
    for r in range(rows_w):
        t, rr = divmod(r, 128)
        j = 0 if (rr % 16) < 8 else 1  # bits 0-15 / 16-31 of the lane word
        for q in range(ng_pad):
            mi, gi = divmod(q, 8)
            st, k = divmod(mi, 4)
            h = gi // 4
            lane = (rr % 8) + 16 * (rr // 16) + 8 * h
            word = int(mt[t, st, lane, k])
            nib = (word >> (16 * j + 4 * (gi % 4))) & 0xF
            pa, pb = nib & 3, nib >> 2
            dense[r, 4 * q + pa] = vals[r, 2 * q]
            dense[r, 4 * q + pb] = vals[r, 2 * q + 1]
    mask = oracle.prune(W, V, M)
    Wm = oracle.apply_mask(W, mask, V, M)
    assert np.array_equal(dense[:rows, :cols], Wm)
    assert not dense[rows:].any() and not dense[:, cols:].any()


def test_batched_more_than_eight():
    """More than 8 weights (or mixed (V, M)) run as one launch per weight — same bytes as single calls."""
    shapes = [(64 + 8 * i, 40 + 16 * i) for i in range(10)]
    Ws = [to_dev_bf16(synth.weights(r, c, seed=r * c)) for r, c in shapes]
    Ps = vnm.prune_compress_batched(Ws, 64, 6, tc=True)
    for W, P in zip(Ws, Ps):
        Q = vnm.prune_compress(W, 64, 6, tc=True)
        torch.cuda.synchronize()
        for a, b in zip(packed_np(P), packed_np(Q)):
            assert np.array_equal(a, b)
        assert torch.equal(P.values_tc.view(torch.int16), Q.values_tc.view(torch.int16))
        assert torch.equal(P.meta_tc, Q.meta_tc)


def decode_window_form(P, rows, cols):
    """Host decode of the tensor-core window form (include/vnm.h; M <= 8) back to a dense [rows_w][cols_p + 8]
    weight: block b of a row is an 8-channel window starting at channel b*M holding two 2:4 groups (channels
    0-3, 4-7), 2 values per group (values_tc[4b + 2 sub + i]); its nibbles sit in meta_tc's M = 128 lane
    order (lane L: rows (L%8) + 16 (L/16) and + 8; K-group gi of MMA k -> bits 16 j + 4 (gi % 4) of lane
    (L with h = gi / 4)).  For M = 4 the form is the plain 2:4 layout (8 blocks of 4 channels per MMA).
    Window positions past the block (channel >= M) must hold zero values; every value lands exactly once."""
    g = P.g
    M = g.M
    bpm = 8 if M == 4 else 4          # blocks per MMA
    gpb = 1 if M == 4 else 2          # 2:4 groups per block
    n_mma = g.nb_pad // bpm
    n_stage = (n_mma + 3) // 4
    rows_w = (g.rows_p + 127) // 128 * 128
    vals = P.values_tc.view(torch.int16).cpu().numpy().view(np.uint16).reshape(rows_w, 16 * n_mma)
    mt = P.meta_tc.cpu().numpy().view(np.uint32).reshape(rows_w // 128, n_stage, 128, 4)
    dense = np.zeros((rows_w, g.cols_p + 8), np.uint16)
    for r in range(rows_w):
        t, rr = divmod(r, 128)
        j = 0 if (rr % 16) < 8 else 1
        for b in range(g.nb_pad):
            for sub in range(gpb):
                q = b * gpb + sub                 # 2:4 group index along the row (8 per MMA)
                mi, gi = divmod(q, 8)
                st, k = divmod(mi, 4)
                lane = (rr % 8) + 16 * (rr // 16) + 8 * (gi // 4)
                nib = (int(mt[t, st, lane, k]) >> (16 * j + 4 * (gi % 4))) & 0xF
                for i, pos in enumerate((nib & 3, nib >> 2)):
                    v = vals[r, 2 * q + i]
                    ch = 4 * sub + pos
                    if ch >= M or b >= g.nb:
                        assert v & 0x7FFF == 0, (r, b, sub, ch)  # window overhang / pad block: zero value
                        continue
                    c = b * M + ch
                    assert dense[r, c] == 0 or v & 0x7FFF == 0, (r, c)
                    if v & 0x7FFF:
                        dense[r, c] = v
    return dense[:rows, :cols]


@pytest.mark.parametrize("V", [32, 64, 128])
@pytest.mark.parametrize("M", [4, 5, 6, 7, 8])
@pytest.mark.parametrize("rows,cols,kind", [(200, 333, "outlier"), (128, 64, "int")])
def test_window_form_decodes_to_oracle(V, M, rows, cols, kind):
    """The window form written by the fused prune pass (single and batched) holds exactly the oracle's masked
    W: decoded on the host, value for value."""
    W = synth.weights(rows, cols, seed=rows + cols + M + V, kind=kind)
    Wd = to_dev_bf16(W)
    P = vnm.prune_compress(Wd, V, M, tc=True)
    B = vnm.prune_compress_batched([Wd, Wd], V, M, tc=True)[1]
    torch.cuda.synchronize()
    Wm = oracle.apply_mask(W, oracle.prune(W, V, M), V, M)
    zero = lambda a: np.where((a & 0x7FFF) == 0, 0, a)  # -0 and +0 both mean "no weight"
    for Q in (P, B):
        assert np.array_equal(zero(decode_window_form(Q, rows, cols)), zero(Wm))


@pytest.mark.parametrize("V", [32, 64, 128])
@pytest.mark.parametrize("M", [5, 6, 8])
def test_prune2_wide_exponent(V, M):
    """Wide-exponent weights (sign * 2^U(-24, 4) * U(1, 2); pin P13) through prune2.cu — the kernel the bench
    runs (32 <= V <= 128, M <= 8) — single and batched: every byte vs the oracle, whose fp32 column L1 follows
    the canonical stride-halving tree (Q3); a different summation order flips near-ties here."""
    W = synth.weights(520, 1000, seed=V * 7 + M, kind="wide")
    check(W, V, M)
    W2 = synth.weights(300, 333, seed=V + M, kind="wide")
    Ps, masks = vnm.prune_compress_batched([to_dev_bf16(W), to_dev_bf16(W2)], V, M, want_mask=True, tc=True)
    torch.cuda.synchronize()
    for Wx, P, mk in zip((W, W2), Ps, masks):
        mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(Wx, V, M)
        assert np.array_equal(u32(mk), mask_ref)
        v, c, m = packed_np(P)
        assert np.array_equal(v, v_ref) and np.array_equal(c, c_ref) and np.array_equal(m, m_ref)


def test_batched_eight_entries_vs_oracle():
    """The batched pass at its maximum of 8 weights in one launch (mixed shapes, one (V, M)): EVERY entry vs the
    oracle, byte for byte (not only against single GPU calls)."""
    shapes = [(1152, 384), (384, 384), (1536, 384), (384, 1536), (70, 23), (200, 333), (64, 4), (130, 1000)]
    Ws = [synth.weights(r, c, seed=5 * r + c, kind=k) for (r, c), k in
          zip(shapes, ["outlier", "normal", "wide", "int", "normal", "wide", "int", "outlier"])]
    Ps, masks = vnm.prune_compress_batched([to_dev_bf16(W) for W in Ws], 64, 5, want_mask=True, tc=True)
    torch.cuda.synchronize()
    for W, P, mk in zip(Ws, Ps, masks):
        mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, 64, 5)
        assert np.array_equal(u32(mk), mask_ref)
        v, c, m = packed_np(P)
        assert np.array_equal(v, v_ref) and np.array_equal(c, c_ref) and np.array_equal(m, m_ref)


def _packed_vs_oracle(P, W, V, M):
    mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, V, M)
    v, c, m = packed_np(P)
    assert np.array_equal(v, v_ref), "A_n values"
    assert np.array_equal(c, c_ref), "A_i1 col_idx"
    assert np.array_equal(m, m_ref), "A_i2 meta"


@pytest.mark.parametrize("V", [32, 64, 128])
@pytest.mark.parametrize("M", [9, 10, 11, 12, 13, 14, 15, 16])
@pytest.mark.parametrize("rows,cols,kind", [(200, 333, "outlier"), (128, 1000, "int"), (256, 517, "wide")])
def test_prune2_m9_to_16_bitexact(V, M, rows, cols, kind):
    """prune2 for 8 < M <= 16 (16-block tiles, two rows per warp step in the row pass; the paper's 128:2:9 .. 13
    points): canonical A_n / A_i1 / A_i2 byte for byte against the oracle, single and batched (no mask
    output: a mask routes to prune.cu), tie-heavy integers and wide exponents included."""
    W = synth.weights(rows, cols, seed=rows + cols + V + M, kind=kind)
    W2 = synth.weights(rows + 64, cols, seed=rows + cols + V + M + 1, kind=kind)
    Wd, W2d = to_dev_bf16(W), to_dev_bf16(W2)
    P = vnm.prune_compress(Wd, V, M)
    B = vnm.prune_compress_batched([Wd, W2d], V, M)
    torch.cuda.synchronize()
    _packed_vs_oracle(P, W, V, M)
    _packed_vs_oracle(B[0], W, V, M)
    _packed_vs_oracle(B[1], W2, V, M)


@pytest.mark.parametrize("V,M", [(128, 13), (128, 9), (64, 11)])
def test_prune2_m_gt_8_llama_shapes(V, M):
    """Llama2-7B up / down weights at the paper's V = 128 / M > 8 points through the batched pass (the bench's)."""
    Ws = [synth.weights(11008, 4096, seed=M, kind="outlier"), synth.weights(4096, 11008, seed=M + 1, kind="outlier")]
    Ps = vnm.prune_compress_batched([to_dev_bf16(W) for W in Ws], V, M, tc=True)
    torch.cuda.synchronize()
    for P, W in zip(Ps, Ws):
        _packed_vs_oracle(P, W, V, M)


def test_prune2_runs_for_m_gt_8():
    """The M > 8 batched pass really is prune2 (its trace line names it), not the prune.cu fallback."""
    import os
    import subprocess
    import sys
    code = ("import torch\nfrom paper_2410_16135_b200 import synth, vnm\nfrom tests.gpu_util import to_dev_bf16\n"
            "W = to_dev_bf16(synth.weights(1024, 4096, seed=1))\n"
            "vnm.prune_compress_batched([W, W], 128, 13, tc=True)\ntorch.cuda.synchronize()\nprint('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VNM_PRUNE_TRACE="1", PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    assert "prune2 V=128 M=13" in r.stderr, r.stderr[-2000:]
