"""Pins of the RIA oracle (Eq. (1), §3) against what the paper / SPEC
and arithmetic fix — not against itself.

RIA_ij = ( |W_ij| / sum_r |W_rj| + |W_ij| / sum_c |W_ic| ) * ( ||X_j||_2 )^a   (channel reading S:165, zero
sums -> 0 S:152, default a = 0.5 S:166)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2410_16135_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ria_examples.json")


def bf(a):
    return synth.f32_to_bf16_bits(np.asarray(a, np.float32))


def exact_ria(Wint):
    """Exact rational RIA with activation factor 1, by the definition (Fractions)."""
    rows, cols = len(Wint), len(Wint[0])
    col = [sum(abs(Wint[r][j]) for r in range(rows)) for j in range(cols)]
    row = [sum(abs(Wint[i][c]) for c in range(cols)) for i in range(rows)]
    out = []
    for i in range(rows):
        out.append([(Fraction(abs(Wint[i][j]), col[j]) if col[j] else Fraction(0)) +
                    (Fraction(abs(Wint[i][j]), row[i]) if row[i] else Fraction(0)) for j in range(cols)])
    return out


def test_spec_worked_example():
    """w = [[1,2],[3,4]], act = [1,1], a = 0.5 -> scores[0][0] = 1/(1+3) + 1/(1+2) = 0.58333..."""
    g = json.load(open(GOLD))["spec_s155"]
    s = oracle.ria(bf(g["w"]), np.array(g["act"], np.float64), g["a"])
    assert abs(float(s[0, 0]) - g["expected_00"]) < 1e-6
    # the other three entries by hand from Eq. (1): 2/6 + 2/3, 3/4 + 3/7, 4/6 + 4/7
    assert np.allclose(s, [[1 / 4 + 1 / 3, 2 / 6 + 2 / 3], [3 / 4 + 3 / 7, 4 / 6 + 4 / 7]], rtol=1e-7)


@pytest.mark.parametrize("seed", range(6))
def test_exact_rationals(seed):
    """Small integer weights: the oracle equals float32(exact rational value) (fp64 evaluation, one rounding)."""
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    Wi = rng.integers(-5, 6, size=(rows, cols))
    if seed == 0:
        Wi[:, 0] = 0  # an all-zero input channel -> its scores are 0
    if seed == 1:
        Wi[0, :] = 0  # an all-zero output channel -> only the column fraction remains
    s = oracle.ria(bf(Wi))
    ex = exact_ria(Wi.tolist())
    for i in range(rows):
        for j in range(cols):
            want = np.float32(float(ex[i][j]))
            assert abs(float(s[i, j]) - float(want)) <= float(np.spacing(want)), (i, j, s[i, j], ex[i][j])


def test_activation_factor_and_exponent():
    """act^a with a = 0.5 on perfect squares is exact; a = 0 makes the factor 1."""
    Wi = np.array([[1, 2, 3], [4, 5, 6]])
    base = oracle.ria(bf(Wi))
    s = oracle.ria(bf(Wi), np.array([4.0, 9.0, 16.0]), 0.5)
    assert np.allclose(s, base * np.array([2.0, 3.0, 4.0]), rtol=1e-7)
    s0 = oracle.ria(bf(Wi), np.array([4.0, 9.0, 16.0]), 0.0)
    assert np.array_equal(s0, base)


def test_scale_invariance_a0():
    """with a = 0 both fractions are scale-free: ria(2^k W) == ria(W) (exact in bf16)."""
    W = synth.weights(40, 70, seed=3)
    Wf = synth.bf16_bits_to_f32(W)
    s = oracle.ria(W)
    for k in (-3, 4):
        assert np.array_equal(oracle.ria(bf(Wf * 2.0 ** k)), s)


def test_act_norms_exact():
    """||x||_2 of integer channels with integer norms (3,4 -> 5; 1,2,2 -> 3; zeros -> 0)."""
    XT = bf(np.array([[3, 4, 0, 0], [1, 2, 2, 0], [0, 0, 0, 0], [-6, 8, 0, 0]], np.float32))
    assert np.array_equal(oracle.act_norms(XT), np.array([5.0, 3.0, 0.0, 10.0]))
    assert np.array_equal(oracle.act_norms(XT, T=1), np.array([3.0, 1.0, 0.0, 6.0]))


def test_ria_feeds_the_prune():
    """A score matrix drives the mask (Q1): RIA with a huge activation on one channel keeps that column in
    every block that contains it (its L1 dominates the block)."""
    W = synth.weights(64, 40, seed=11)
    act = np.ones(40)
    act[7] = 1e6
    s = oracle.ria(W, act, 0.5)
    mask = oracle.prune(W, 64, 8, score=s)
    bits = np.unpackbits(mask.view(np.uint8), bitorder="little").reshape(64, -1)[:, :40]
    assert bits[:, 7].sum() > 0  # column 7 (block 0) is kept: some rows keep it
