"""Pins for the oracle's packing (App. A), unpacking, and the fp64 products (O8/O9)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2410_16135_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_pack_example():
    """a_n=[7,9], a_i2=[1,3] (nibble 1|3<<2 = 0xD).  A_i1 under reading Q19 is the columns
    carrying nonzeros {1,4} completed by the lowest free indices -> [0,1,2,4]; SPEC's [0,1,3,4] differs
    only in a column that carries no nonzero, so both unpack to the same matrix."""
    ex = GOLD["pack_single_block"]
    W = synth.f32_to_bf16_bits(np.array(ex["W"], np.float32))
    mask = np.zeros((1, 1), np.uint32)
    for c in ex["mask_cols"]:
        mask[0, 0] |= np.uint32(1 << c)
    st, values, col_idx, meta = oracle.pack(W, mask, ex["V"], ex["M"])
    assert st == 0
    assert list(synth.bf16_bits_to_f32(values[0, :2])) == ex["a_n"]
    nib = int(meta[0, 0]) & 0xF
    assert [nib & 3, nib >> 2] == ex["a_i2"] and nib == 0xD
    assert list(col_idx[0, 0]) == [0, 1, 2, 4]
    # SPEC's encoding and ours decode to the same dense row
    spec_dense = np.zeros(5)
    for v, p in zip(ex["a_n"], ex["a_i2"]):
        spec_dense[ex["a_i1_spec"][p]] = v
    ours = synth.bf16_bits_to_f32(oracle.unpack(values, col_idx, meta, 1, 5, 1, 5))[0]
    assert (ours == spec_dense).all()


def test_pad_contents():
    """Pad blocks (nb..nb_pad): values 0, col_idx {0,1,2,3}, nibble 0x4."""
    W = synth.weights(70, 23, seed=2)  # rows_p 128 (V=64), cols_p 25, nb 5, nb_pad 8
    mask, values, col_idx, meta = oracle.prune_pack(W, 64, 5)
    g = oracle.geometry(70, 23, 64, 5)
    assert (values[:, 2 * g["nb"]:] == 0).all()
    assert (col_idx[:, g["nb"]:] == np.arange(4)).all()
    nibs = (meta[:, :, None] >> (4 * np.arange(8, dtype=np.uint32))) & 0xF
    assert (nibs.reshape(g["rows_p"], -1)[:, g["nb"]:] == 0x4).all()
    # padded rows are all zero values
    assert (values[70:] == 0).all()


@pytest.mark.parametrize("V,M", [(1, 5), (2, 5), (16, 8), (64, 5), (64, 4), (64, 16), (128, 7)])
def test_roundtrip(V, M):
    """S:493, pin P8: unpack(pack(W (.) M)) == W (.) M bitwise, indices ascending."""
    rows, cols = 2 * V + 3, 9 * M + 2
    W = synth.weights(rows, cols, seed=V + M, kind="normal")
    mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
    g = oracle.geometry(rows, cols, V, M)
    dense = oracle.unpack(values, col_idx, meta, rows, cols, V, M)
    wm = oracle.apply_mask(W, mask, V, M)
    assert (dense[:rows, :cols] == wm).all()
    assert (dense[rows:] == 0).all() and (dense[:, cols:] == 0).all()
    ci = col_idx[:, :g["nb"]].astype(int)
    assert (np.diff(ci, axis=2) > 0).all() and (ci < M).all()


def test_invalid_mask_detected():
    W = synth.weights(64, 40, seed=4)
    mask = oracle.prune(W, 64, 5)
    bad = mask.copy()
    # row 10, block 3: add a third bit
    g = oracle.geometry(64, 40, 64, 5)
    m = np.unpackbits(bad.view(np.uint8).reshape(64, -1), axis=1, bitorder="little")
    free = [c for c in range(15, 20) if not m[10, c]]
    c = free[0]
    bad[10, c // 32] |= np.uint32(1 << (c % 32))
    st, *_ = oracle.pack(W, bad, 64, 5)
    assert st == 1 + 3
    # a bit beyond cols_p
    bad2 = mask.copy()
    bad2[0, 1] |= np.uint32(1 << 31)  # column 63 >= cols_p = 40
    st, *_ = oracle.pack(W, bad2, 64, 5)
    assert st == 1 + (64 // 64) * g["nb"]


def test_mult_count_and_ratio():
    """S:480 (96 multiplies) and S:478-479 (2/M): stored values per row = 2*nb, multiplies = rows_p*2*nb*T."""
    ex = GOLD["mult_count"]
    g = oracle.geometry(ex["rows"], ex["cols"], ex["V"], ex["M"])
    assert g["rows_p"] * 2 * g["nb"] * ex["T"] == ex["expected"]
    for Ms, r in ex["ratio"].items():
        M = int(Ms)
        g = oracle.geometry(64, 20 * M, 64, M)
        assert (2 * g["nb"]) / g["cols_p"] == r


def test_gemm_ref_exact_on_integers():
    """O8 pinned by exact rational arithmetic (integer x and w: every product and sum exact)."""
    rows, cols, T = 12, 20, 7
    W = synth.weights(rows, cols, seed=1, kind="int")
    XT = synth.activations_t(cols, T, seed=2, kind="int")
    Y, A = oracle.gemm_ref(XT, W)
    w = synth.bf16_bits_to_f32(W).astype(np.int64)
    x = synth.bf16_bits_to_f32(XT).astype(np.int64)
    assert (Y == (w @ x)).all()
    assert (A == (np.abs(w)[:, :, None] * np.abs(x)[None]).sum(1)).all()


def test_gemm_ref_vs_numpy():
    """O8 vs the library fp64 matmul on random bf16 data (relative 1e-12)."""
    rows, cols, T = 64, 200, 33
    W = synth.weights(rows, cols, seed=5)
    XT = synth.activations_t(cols, T, seed=6)
    Y, A = oracle.gemm_ref(XT, W)
    ref = synth.bf16_bits_to_f32(W).astype(np.float64) @ synth.bf16_bits_to_f32(XT).astype(np.float64)
    assert np.allclose(Y, ref, rtol=0, atol=1e-12 * (A.max() + 1))


def test_sampled_equals_full():
    W = synth.weights(40, 50, seed=9)
    XT = synth.activations_t(50, 20, seed=10)
    Y, A = oracle.gemm_ref(XT, W)
    o = np.array([0, 5, 39, 17]); t = np.array([0, 19, 3, 11])
    Ys, As = oracle.gemm_ref_sampled(XT, W, o, t)
    assert np.allclose(Ys, Y[o, t], rtol=1e-14, atol=1e-14) and np.allclose(As, A[o, t], rtol=1e-14)


@pytest.mark.parametrize("V,M", [(64, 8), (16, 5), (64, 5)])
def test_packed_spmm_equals_dense(V, M):
    """O9 (reads only values/col_idx/meta) == O8 on W (.) M within fp64 rounding."""
    rows, cols, T = 2 * V - 3, 11 * M - 1, 17
    W = synth.weights(rows, cols, seed=12)
    XT = synth.activations_t(cols, T, seed=13)
    mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
    Yp = oracle.spmm_packed(XT, values, col_idx, meta, rows, cols, V, M)
    Y, A = oracle.gemm_ref(XT, oracle.apply_mask(W, mask, V, M))
    assert np.allclose(Yp, Y, rtol=0, atol=1e-13 * (A.max() + 1))


def test_identity_x():
    """Pin P10: X = identity => Y^T == unpack(values) exactly."""
    V, M, rows, cols = 16, 5, 32, 40
    W = synth.weights(rows, cols, seed=14)
    mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
    XT = synth.f32_to_bf16_bits(np.eye(cols, dtype=np.float32))
    Yp = oracle.spmm_packed(XT, values, col_idx, meta, rows, cols, V, M)
    dense = synth.bf16_bits_to_f32(oracle.unpack(values, col_idx, meta, rows, cols, V, M))
    assert (Yp == dense[:rows, :cols]).all()


def test_linearity():
    """spmm(x1 + x2) == spmm(x1) + spmm(x2) (exact here: integer x, fp64)."""
    V, M, rows, cols, T = 16, 6, 32, 48, 9
    W = synth.weights(rows, cols, seed=15)
    _, values, col_idx, meta = oracle.prune_pack(W, V, M)
    x1 = synth.activations_t(cols, T, seed=16, kind="int")
    x2 = synth.activations_t(cols, T, seed=17, kind="int")
    s = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(x1) + synth.bf16_bits_to_f32(x2))
    f = lambda x: oracle.spmm_packed(x, values, col_idx, meta, rows, cols, V, M)
    assert np.allclose(f(s), f(x1) + f(x2), rtol=1e-14, atol=1e-14)


def test_deit_param_accounting():
    """Pin P17 (soft): Table tab:deit DeiT-B 86.6M -> 22.7M params at 64:2:8.  With density
    2/M (exact, checked above) on the 4 per-block linears (768x2304, 768x768, 768x3072, 3072x768; x12
    blocks) and the non-linear-layer params dense, the reduction is within 0.5 points of the table."""
    lin = 12 * (768 * 2304 + 768 * 768 + 768 * 3072 + 3072 * 768)
    total = 86.57e6
    other = total - lin
    sparse = other + lin * 2 / 8
    assert abs((1 - sparse / total) - (1 - 22.7 / 86.6)) < 0.005
