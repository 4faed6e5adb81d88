"""GPU parity of vnm_spmm_batched (the grouped small-T SpMM: up to 4 independent problems per launch) against the
oracle's fp64 product (step O8), every output compared; the tolerance of BASELINE.json (Q14).  Calls go
through the C ABI (vnm.spmm_batched marshals the arrays only)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


def _case(rows, cols, V, M, T, seed, kind="outlier"):
    W = synth.weights(rows, cols, seed=seed, kind=kind)
    XT = synth.activations_t(cols, T, seed=seed + 1)
    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, oracle.prune(W, V, M), V, M))
    return vnm.prune_compress(to_dev_bf16(W), V, M), to_dev_bf16(XT), Yref, Aref


def _check(Y, Yref, Aref, bf16):
    got = Y.float().cpu().numpy().astype(np.float64)
    tol = oracle.tolerance(Yref, Aref, y_is_bf16=bf16)
    bad = np.abs(got - Yref) > tol
    assert not bad.any(), f"{bad.sum()} / {bad.size} outside tolerance"


def test_llama_decode_trio_one_launch():
    """The bench's decode step: Llama q (4096x4096), up (11008x4096), down (4096x11008) at 64:2:5, T = 16, bf16 Y^T,
    as ONE launch (vnm_launch_count), every output against the oracle."""
    T = 16
    cases = [_case(r, c, 64, 5, T, seed=r + 3 * c) for r, c in [(4096, 4096), (11008, 4096), (4096, 11008)]]
    n0 = vnm.lib().vnm_launch_count()
    Ys = vnm.spmm_batched([x for _, x, _, _ in cases], [P for P, _, _, _ in cases], T, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert vnm.lib().vnm_launch_count() - n0 == 1
    for Y, (_, _, Yref, Aref) in zip(Ys, cases):
        _check(Y, Yref, Aref, bf16=True)


@pytest.mark.parametrize("T", [1, 7, 16, 32])
@pytest.mark.parametrize("specs", [
    [(300, 777, 64, 5), (1000, 333, 128, 13), (130, 1100, 64, 8)],          # mixed M, V = 64 / 128 (one V class)
    [(256, 640, 32, 5), (130, 500, 32, 7)],                                 # V = 32 (VSET 2)
    [(200, 300, 16, 5), (96, 257, 16, 8), (64, 100, 16, 11), (70, 23, 16, 9)],  # V = 16, four problems
    [(512, 1024, 256, 5), (600, 999, 64, 6), (384, 1000, 128, 9), (64, 4, 64, 4), (129, 2000, 64, 16)],  # 4 + 1
])
def test_batched_mixed_shapes(specs, T):
    """Ragged rows / channels / tokens, mixed M and V within a V class, fp32 Y^T; five problems run as a group of
    4 and a single launch."""
    cases = [_case(r, c, V, M, T, seed=7 * r + c + M + T) for r, c, V, M in specs]
    Ys = vnm.spmm_batched([x for _, x, _, _ in cases], [P for P, _, _, _ in cases], T)
    torch.cuda.synchronize()
    for Y, (_, _, Yref, Aref) in zip(Ys, cases):
        _check(Y, Yref, Aref, bf16=False)


def test_batched_mixed_v_classes_and_plans():
    """Problems that cannot share a launch (V = 32 next to V = 64; T > 32 goes through vnm_spmm one by one):
    still every output right."""
    for T, specs in [(16, [(256, 640, 32, 5), (300, 777, 64, 5)]), (40, [(300, 777, 64, 5), (200, 500, 64, 8)])]:
        cases = [_case(r, c, V, M, T, seed=r + c + T) for r, c, V, M in specs]
        Ys = vnm.spmm_batched([x for _, x, _, _ in cases], [P for P, _, _, _ in cases], T)
        torch.cuda.synchronize()
        for Y, (_, _, Yref, Aref) in zip(Ys, cases):
            _check(Y, Yref, Aref, bf16=False)


def test_batched_without_workspace():
    """No workspace: whole row groups per CTA across the problems (nothing cut)."""
    T = 16
    specs = [(4096, 4096, 64, 5), (1024, 11008, 64, 13), (700, 4096, 128, 8)]
    cases = [_case(r, c, V, M, T, seed=r + M) for r, c, V, M in specs]
    n = len(cases)
    Ys = [torch.empty((P.g.rows, T), dtype=torch.float32, device="cuda") for P, _, _, _ in cases]
    cps = [P.c() for P, _, _, _ in cases]
    arr = lambda ty, xs: (ty * n)(*xs)
    st = vnm.lib().vnm_spmm_batched(
        n, arr(ctypes.c_void_p, [x.data_ptr() for _, x, _, _ in cases]), arr(ctypes.c_int64, [x.stride(0) for _, x, _, _ in cases]),
        T, arr(ctypes.c_void_p, [ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps]),
        arr(ctypes.c_void_p, [Y.data_ptr() for Y in Ys]), arr(ctypes.c_int64, [Y.stride(0) for Y in Ys]), vnm.VNM_F32,
        0, None, 0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0, vnm.status_string(st)
    torch.cuda.synchronize()
    for Y, (_, _, Yref, Aref) in zip(Ys, cases):
        _check(Y, Yref, Aref, bf16=False)


def test_batched_deterministic_and_workspace_reusable():
    """20 batched calls on one workspace give bit-identical Y^T (the K pieces are summed in one fixed order and
    every call leaves the tickets zero); a single-problem vnm_spmm on the same workspace afterwards is right too."""
    T = 16
    cases = [_case(r, c, 64, 5, T, seed=r + c) for r, c in [(4096, 4096), (11008, 4096), (4096, 11008)]]
    Xs, Ps = [x for _, x, _, _ in cases], [P for P, _, _, _ in cases]
    ws = vnm.spmm_batched_workspace([P.g for P in Ps], T, "cuda")
    ref = [Y.clone() for Y in vnm.spmm_batched(Xs, Ps, T, workspace=ws)]
    for _ in range(20):
        Ys = vnm.spmm_batched(Xs, Ps, T, workspace=ws)
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(Ys, ref))
    Y1 = vnm.spmm(Xs[1], Ps[1], T=T, workspace=ws)
    torch.cuda.synchronize()
    _check(Y1, cases[1][2], cases[1][3], bf16=False)


def test_weights_ready_still_waits_for_x():
    """VNM_SPMM_WEIGHTS_READY lets the launch read the WEIGHTS before griddepcontrol.wait, never X^T: here X^T of
    both problems is written by a one-CTA probe kernel that releases its dependents at once and copies only after
    spinning ~0.5 ms, so the SpMM runs during the spin; reading X^T early would see the NaN fill."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    probe = os.path.join(root, "tests", "probes", "libvnm_probe.so")
    if not os.path.exists(probe):
        pytest.skip("tests/probes/libvnm_probe.so not built")
    PL = ctypes.CDLL(probe)
    PL.vnm_probe_delayed_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_longlong,
                                          ctypes.c_void_p]
    T = 16
    cases = [_case(r, c, 64, 5, T, seed=r + 11 * c) for r, c in [(4096, 4096), (11008, 4096)]]
    # one X^T buffer for both problems (same cols): the delayed copy fills it
    src = cases[0][1]
    X = torch.empty_like(src)
    Ps = [P for P, _, _, _ in cases]
    ws = vnm.spmm_batched_workspace([P.g for P in Ps], T, "cuda")
    Ys = [torch.empty((P.g.rows, T), dtype=torch.float32, device="cuda") for P in Ps]
    stream = torch.cuda.current_stream()
    for _ in range(3):
        X.fill_(float("nan"))
        for Y in Ys:
            Y.zero_()
        assert PL.vnm_probe_delayed_copy(X.data_ptr(), src.data_ptr(), X.numel() * 2, 1_000_000, stream.cuda_stream) == 0
        vnm.spmm_batched([X, X], Ps, T, outs=Ys, workspace=ws, weights_ready=True)
        torch.cuda.synchronize()
        for Y, (_, x0, Yref, Aref) in zip(Ys, cases):
            assert not torch.isnan(Y).any()
        _check(Ys[0], cases[0][2], cases[0][3], bf16=False)
        # problem 1 used X = problem 0's activations: compare against its own weights times those
        Yref1, Aref1 = oracle.gemm_ref(synth.activations_t(4096, T, seed=4096 + 11 * 4096 + 1),
                                       oracle.apply_mask(synth.weights(11008, 4096, seed=11008 + 11 * 4096, kind="outlier"),
                                                         oracle.prune(synth.weights(11008, 4096, seed=11008 + 11 * 4096, kind="outlier"), 64, 5), 64, 5))
        _check(Ys[1], Yref1, Aref1, bf16=False)


def test_weights_ready_sequence_in_a_graph():
    """The bench's decode-block sequence with the flag: prune (batched) -> [q k v] -> [o] (flag) -> [gate up] (flag)
    -> [down] (flag), captured once and replayed; every replay bit-identical to the first, which matches the
    oracle on the last group."""
    T = 16
    shapes = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]
    Ws = [to_dev_bf16(synth.weights(r, c, seed=5 * r + c + i, kind="outlier")) for i, (r, c) in enumerate(shapes)]
    Xs = [to_dev_bf16(synth.activations_t(c, T, seed=c + i)) for i, (r, c) in enumerate(shapes)]
    Ps = vnm.prune_compress_batched(Ws, 64, 5)
    Ys = [torch.empty((r, T), dtype=torch.bfloat16, device="cuda") for r, _ in shapes]
    groups = [[0, 1, 2], [3], [4, 5], [6]]
    wss = [vnm.spmm_batched_workspace([Ps[i].g for i in gr], T, "cuda") for gr in groups]
    cps = [P.c() for P in Ps]
    n = len(Ps)
    b_w = (ctypes.c_void_p * n)(*[W.data_ptr() for W in Ws])
    b_lw = (ctypes.c_int64 * n)(*[W.stride(0) for W in Ws])
    b_po = (ctypes.c_void_p * n)(*[ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps])

    def step():
        assert vnm.lib().vnm_prune_compress_batched(n, b_w, b_lw, None, None, b_po, None,
                                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        for gi, gr in enumerate(groups):
            vnm.spmm_batched([Xs[i] for i in gr], [Ps[i] for i in gr], T, outs=[Ys[i] for i in gr], workspace=wss[gi],
                             weights_ready=gi > 0)
    step()
    torch.cuda.synchronize()
    ref = [Y.clone() for Y in Ys]
    W6 = synth.weights(4096, 11008, seed=5 * 4096 + 11008 + 6, kind="outlier")
    Yref, Aref = oracle.gemm_ref(synth.activations_t(11008, T, seed=11008 + 6), oracle.apply_mask(W6, oracle.prune(W6, 64, 5), 64, 5))
    _check(Ys[6], Yref, Aref, bf16=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for i in range(600):
        g.replay()
        if i % 200 == 199:
            torch.cuda.synchronize()
            assert all(torch.equal(a.view(torch.int16), b.view(torch.int16)) for a, b in zip(Ys, ref)), i
