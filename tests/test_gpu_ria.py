"""GPU parity of the RIA score pre-pass (Eq. (1)) through the C ABI.

fp32 on the GPU vs the fp64 oracle: sums of up to K terms in fp32 carry a relative error well below 1e-4
at these sizes (n u ~ 11008 x 6e-8 worst case); the mask built from the GPU scores is then bit-exact
against the oracle's prune of the same scores (the decision rules are exact, Q3-Q5)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import packed_np, to_dev_bf16, u32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cols,T", [(384, 197), (4096, 16), (1000, 1), (77, 300), (5, 0)])
def test_act_norms(cols, T):
    XT = synth.activations_t(cols, max(T, 1), seed=cols + T)
    n = vnm.act_norms(to_dev_bf16(XT), T=T).cpu().numpy().astype(np.float64)
    ref = oracle.act_norms(XT, T=T)
    assert np.allclose(n, ref, rtol=2e-6, atol=1e-30)


@pytest.mark.parametrize("rows,cols,kind,use_act", [(128, 64, "normal", True), (1152, 384, "normal", True),
                                                    (70, 23, "int", False), (300, 1000, "outlier", True),
                                                    (4096, 4096, "normal", True), (513, 777, "wide", False)])
def test_ria_scores(rows, cols, kind, use_act):
    W = synth.weights(rows, cols, seed=rows + cols, kind=kind)
    if kind == "int":
        W[3, :] = 0      # zero output channel
        W[:, 5] = 0      # zero input channel
    act = oracle.act_norms(synth.activations_t(cols, 64, seed=cols)) if use_act else None
    s = vnm.ria_score(to_dev_bf16(W), None if act is None else torch.tensor(act, dtype=torch.float32).cuda(), 0.5)
    s = s.cpu().numpy().astype(np.float64)
    ref = oracle.ria(W, None if act is None else act.astype(np.float32).astype(np.float64), 0.5)
    assert np.allclose(s, ref, rtol=1e-4, atol=0), float(np.max(np.abs(s - ref) / np.maximum(ref, 1e-30)))
    if kind == "int":
        assert np.all(s[:, 5] == 0)


def test_ria_deterministic():
    W = to_dev_bf16(synth.weights(2048, 1536, seed=4))
    a = vnm.ria_score(W)
    b = vnm.ria_score(W)
    assert torch.equal(a, b)


@pytest.mark.parametrize("rows,cols,V,M", [(1152, 384, 64, 5), (4096, 4100, 64, 5), (512, 1000, 128, 8)])
def test_ria_then_prune_compress_bitexact(rows, cols, V, M):
    """The TS1/TS3 path: RIA scores -> S_{V:N:M} -> A_n / A_i1 / A_i2, every byte vs the oracle
    given the same scores."""
    W = synth.weights(rows, cols, seed=V + M + rows, kind="outlier")
    act = torch.tensor(oracle.act_norms(synth.activations_t(cols, 128, seed=1)), dtype=torch.float32).cuda()
    Wd = to_dev_bf16(W)
    s = vnm.ria_score(Wd, act, 0.5)
    P, mask = vnm.prune_compress(Wd, V, M, score=s, want_mask=True)
    torch.cuda.synchronize()
    s_np = np.ascontiguousarray(s.cpu().numpy())
    mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, V, M, score=s_np)
    assert np.array_equal(u32(mask), mask_ref)
    v, c, m = packed_np(P)
    assert np.array_equal(v, v_ref) and np.array_equal(c, c_ref) and np.array_equal(m, m_ref)
