"""GPU parity of the channel-permutation gain scores: input channels, Eq. (7) P:207-213,
DESIGN.md Q22, V up to 128 and M up to 32; output channels, Eq. (8) P:211-213 / P:198, Q23
through the C ABI, against the oracle (pinned in tests/test_oracle_permute.py).  Every keep / drop decision
uses the same fp32 L1 tree and tie rules, so entries differ only by fp32-vs-fp64 summation (rtol 1e-5)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols,V,M,kind", [(64, 40, 64, 5, "normal"), (128, 96, 64, 8, "normal"),
                                                (32, 23, 16, 4, "int"), (96, 50, 32, 7, "wide"),
                                                (70, 333, 64, 6, "normal"), (16, 20, 1, 5, "int"),
                                                (1152, 384, 64, 5, "outlier"), (256, 300, 128, 5, "normal"),
                                                (256, 200, 128, 8, "wide"), (128, 260, 64, 13, "normal"),
                                                (200, 190, 32, 16, "int"), (130, 230, 128, 11, "outlier")])
def test_permute_gain(rows, cols, V, M, kind):
    W = synth.weights(rows, cols, seed=rows * 7 + cols, kind=kind)
    score = synth.bf16_bits_to_f32(W).astype(np.float32)
    if kind == "normal":
        score = oracle.ria(W, None, 0.5)  # the CP objective uses RIA (Eq. 6-7)
    got = vnm.permute_gain(torch.tensor(score).cuda(), V, M).cpu().numpy().astype(np.float64)
    ref = oracle.permute_gain(score, V, M)
    assert np.allclose(got, ref, rtol=1e-5, atol=1e-30), float(np.max(np.abs(got - ref)))


def test_permute_gain_identity_is_retained_score():
    rows, cols, V, M = 256, 160, 64, 5
    W = synth.weights(rows, cols, seed=3)
    score = oracle.ria(W, None, 0.5)
    cost = vnm.permute_gain(torch.tensor(score).cuda(), V, M).cpu().numpy().astype(np.float64)
    mask = oracle.prune(W, V, M, score=score)
    assert abs(np.trace(cost) - oracle.retained_score(score, mask, V, M)) < 1e-4 * np.trace(cost)


@pytest.mark.parametrize("rows,cols,V,M,kind", [(64, 40, 64, 5, "normal"), (128, 96, 64, 8, "normal"),
                                                (48, 23, 16, 4, "int"), (96, 50, 32, 7, "wide"),
                                                (70, 333, 64, 6, "normal"), (16, 20, 1, 5, "int"),
                                                (256, 120, 128, 5, "outlier"), (130, 77, 64, 13, "normal"),
                                                (384, 385, 64, 5, "outlier")])
def test_permute_gain_out(rows, cols, V, M, kind):
    """Output-channel permutation gains (Eq. 8) vs the oracle (pinned by substitution through the pruning
    oracle): same fp32 L1 trees (the leaf-replaced tree is bit-identical to re-summing) and tie rules, so
    entries differ only by fp32-vs-fp64 accumulation over the column blocks."""
    W = synth.weights(rows, cols, seed=rows * 5 + cols, kind=kind)
    score = synth.bf16_bits_to_f32(W).astype(np.float32)
    if kind == "normal":
        score = oracle.ria(W, None, 0.5)
    got = vnm.permute_gain_out(torch.tensor(score).cuda(), V, M).cpu().numpy().astype(np.float64)
    ref = oracle.permute_gain_out(score, V, M)
    assert np.allclose(got, ref, rtol=1e-5, atol=1e-30), float(np.max(np.abs(got - ref)))


def test_permute_gain_out_identity_is_retained_score():
    rows, cols, V, M = 256, 160, 64, 5
    W = synth.weights(rows, cols, seed=4)
    score = oracle.ria(W, None, 0.5)
    cost = vnm.permute_gain_out(torch.tensor(score).cuda(), V, M).cpu().numpy().astype(np.float64)
    mask = oracle.prune(W, V, M, score=score)
    assert abs(np.trace(cost) - oracle.retained_score(score, mask, V, M)) < 1e-4 * np.trace(cost)
