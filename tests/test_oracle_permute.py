"""Pins of the channel-permutation gain oracle (Eq. (7) `eq:admm1` P:207, the LSA
modelling P:213; SPEC solve_input_perm S:372-389; reading Q22).

cost[j][b*M+s] = sum over V-stripes of the retained score channel j contributes in slot s of block b when it
replaces that slot's occupant (other columns frozen) and the block is re-pruned by S_{V:N:M}."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2410_16135_b200 import synth


def bf(a):
    return synth.f32_to_bf16_bits(np.asarray(a, np.float32))


def cost_by_substitution(score, V, M, j, slot):
    """The definition through the (pinned) pruning oracle: overwrite column `slot` with channel j, prune the
    whole matrix, add e_j over the rows that keep `slot`."""
    rows, cols = score.shape
    g = oracle.geometry(rows, cols, V, M)
    S = np.zeros((rows, g["cols_p"]), np.float32)
    S[:, :cols] = np.abs(score)
    Sp = S.copy()
    Sp[:, slot] = S[:, j]
    mask = oracle.prune(bf(np.zeros_like(Sp)), V, M, score=Sp)
    bits = np.unpackbits(mask.view(np.uint8), bitorder="little").reshape(g["rows_p"], -1)[:rows, :g["cols_p"]]
    return float(np.sum(bits[:, slot] * S[:, j].astype(np.float64)))


@pytest.mark.parametrize("rows,cols,V,M,seed", [(4, 10, 2, 5, 0), (8, 16, 4, 8, 1), (6, 12, 2, 6, 2), (3, 7, 1, 5, 3)])
def test_equals_substitution_through_the_prune(rows, cols, V, M, seed):
    """Every entry equals the retained contribution obtained by actually substituting the column and running
    the pruning oracle (pinned by brute force in test_oracle_prune.py)."""
    score = np.random.default_rng(seed).standard_normal((rows, cols)).astype(np.float32)
    cost = oracle.permute_gain(score, V, M)
    g = oracle.geometry(rows, cols, V, M)
    for j, slot in itertools.product(range(g["cols_p"]), range(g["cols_p"])):
        ref = cost_by_substitution(score, V, M, j, slot) if j < cols else 0.0
        assert abs(cost[j, slot] - ref) <= 1e-9 * max(1.0, ref), (j, slot, cost[j, slot], ref)


@pytest.mark.parametrize("rows,cols,V,M", [(64, 40, 64, 5), (128, 96, 64, 8), (32, 23, 16, 4), (96, 50, 32, 7)])
def test_identity_assignment_is_the_retained_score(rows, cols, V, M):
    """With every channel in its own slot the costs add up to the retained score of S_{V:N:M}."""
    score = synth.bf16_bits_to_f32(synth.weights(rows, cols, seed=rows + cols)).astype(np.float32)
    cost = oracle.permute_gain(score, V, M)
    mask = oracle.prune(bf(score), V, M, score=score)
    want = oracle.retained_score(score, mask, V, M)
    assert abs(np.trace(cost) - want) <= 1e-9 * want


def test_zero_channel_and_m4():
    """A zero channel contributes nothing anywhere; at M = 4 every slot is kept (P:9: 64:2:4 is plain 2:4), so a
    channel's cost in slot s is its 2:4 survivors against the block's other 3 columns."""
    score = np.random.default_rng(5).random((8, 12)).astype(np.float32) + 0.1
    score[:, 3] = 0.0
    cost = oracle.permute_gain(score, 4, 5)
    assert np.all(cost[3] == 0.0)
    s4 = np.random.default_rng(6).random((4, 8)).astype(np.float32)
    c4 = oracle.permute_gain(s4, 4, 4)
    for j in range(8):
        for slot in range(8):
            b = slot // 4
            others = [b * 4 + c for c in range(4) if b * 4 + c != slot]
            exp = 0.0
            for r in range(4):
                beat = sum(1 for o in others if s4[r, o] > s4[r, j] or (s4[r, o] == s4[r, j] and o % 4 < slot % 4))
                if beat <= 1:
                    exp += float(s4[r, j])
            assert abs(c4[j, slot] - exp) < 1e-9
