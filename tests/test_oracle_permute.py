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


# ---------------------------------------------------------------------------------- output permutation (Eq. 8)
def cost_out_by_substitution(score, V, M, i, slot):
    """Output-permutation cost through the (pinned) pruning oracle: overwrite ROW `slot` with row i, prune the
    whole matrix, add row `slot`'s kept e (block order, ascending columns within a block)."""
    rows, cols = score.shape
    g = oracle.geometry(rows, cols, V, M)
    S = np.zeros((g["rows_p"], g["cols_p"]), np.float32)
    S[:rows, :cols] = np.abs(score)
    Sp = S.copy()
    Sp[slot, :] = S[i, :]
    mask = oracle.prune(bf(np.zeros((g["rows_p"], cols), np.float32)), V, M, score=Sp[:, :cols].copy())
    bits = np.unpackbits(mask.view(np.uint8), bitorder="little").reshape(g["rows_p"], -1)[:, :g["cols_p"]]
    acc = 0.0
    for c in range(g["cols_p"]):
        if bits[slot, c]:
            acc += float(Sp[slot, c])
    return acc


@pytest.mark.parametrize("rows,cols,V,M,seed", [(4, 10, 2, 5, 0), (8, 16, 4, 8, 1), (6, 12, 2, 6, 2), (8, 9, 4, 4, 3),
                                                (7, 11, 4, 5, 4)])
def test_out_equals_substitution_through_the_prune(rows, cols, V, M, seed):
    """Every output-permutation entry equals the retained score of the slot's row after actually putting row i
    there and running the pruning oracle (exact: same decisions, same fp64 summation order)."""
    score = np.random.default_rng(seed).standard_normal((rows, cols)).astype(np.float32)
    cost = oracle.permute_gain_out(score, V, M)
    g = oracle.geometry(rows, cols, V, M)
    for i, slot in itertools.product(range(g["rows_p"]), range(g["rows_p"])):
        ref = cost_out_by_substitution(score, V, M, i, slot)
        assert cost[i, slot] == ref, (i, slot, cost[i, slot], ref)


@pytest.mark.parametrize("rows,cols,V,M", [(64, 40, 64, 5), (128, 96, 64, 8), (48, 23, 16, 4), (96, 50, 32, 7),
                                           (70, 33, 32, 13)])
def test_out_identity_assignment_is_the_retained_score(rows, cols, V, M):
    """With every row in its own slot the output costs add up to the retained score of S_{V:N:M}."""
    score = synth.bf16_bits_to_f32(synth.weights(rows, cols, seed=rows * cols)).astype(np.float32)
    cost = oracle.permute_gain_out(score, V, M)
    mask = oracle.prune(bf(score), V, M, score=score)
    want = oracle.retained_score(score, mask, V, M)
    assert abs(np.trace(cost) - want) <= 1e-9 * want


def test_out_v1_is_slot_independent():
    """V = 1: a stripe is a single row, so a row's contribution does not depend on where it goes."""
    score = np.random.default_rng(9).random((6, 20)).astype(np.float32)
    cost = oracle.permute_gain_out(score, 1, 5)
    for i in range(6):
        assert np.all(cost[i] == cost[i, 0])
    # ... and equals the row's own retained score
    mask = oracle.prune(bf(score), 1, 5, score=score)
    bits = np.unpackbits(mask.view(np.uint8), bitorder="little").reshape(6, -1)[:, :20]
    for i in range(6):
        assert abs(cost[i, 0] - float(np.sum(bits[i] * score[i].astype(np.float64)))) <= 1e-12


def test_out_permutation_changes_the_objective():
    """with V > 1 the output permutation changes the retained norm — the costs are not slot-independent,
    and the LSA optimum (brute force over all row orders of a 4 x 16 matrix, 2:2:8) beats or ties the identity."""
    score = np.random.default_rng(11).random((4, 16)).astype(np.float32)
    cost = oracle.permute_gain_out(score, 2, 8)
    assert not np.all(cost == cost[:, :1])
    best = max(sum(cost[i, p[i]] for i in range(4)) for p in itertools.permutations(range(4)))
    assert best >= np.trace(cost)
