"""Full element-wise parity of the EXACT paths bench.py times, against the oracle.

* DeiT-S (BJ configs[1], the default bench workload): the same seeded weights / activations as bench.py, ONE
  vnm_prune_compress_batched launch over the 4 layers with the window form (exactly the bench's pass), every
  batched entry's mask / A_n / A_i1 / A_i2 compared byte for byte with the oracle's prune + pack, then every
  layer's vnm_spmm with the default plan and bf16 Y^T — every one of the 4 x (rows x 50,432) outputs compared
  with the oracle's fp64 product (O8) within the BASELINE.json tolerance (+ bf16 rounding, Q14).
* Llama2-7B prefill (BJ configs[3]): the up and down layers at T = 2048, same flow, every output.
* Llama2-7B decode (configs[3], T = 16): the bench's three layers, every output (the small-T plan).

PAPER.md P:80-84 (S_{V:N:M}), App. A P:547-548 (the packed form and the SpMM).  The oracle product runs over
token chunks so host memory stays bounded."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import packed_np, to_dev_bf16, u32

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (the workload table and the input recipe the bench uses)


def bench_inputs(name):
    """The bench's own host inputs for a workload (bench.run_gpu: kind="outlier" W, seeded per layer)."""
    wl = bench.WORKLOADS[name]
    T, cfg = wl["T"], wl["cfg"]
    ldx = -(-T // 8) * 8
    out = []
    for li, (lname, rows, cols) in enumerate(wl["layers"]):
        W = synth.weights(rows, cols, seed=synth.seed(cfg, 0) + 10 * li, kind="outlier")
        XT = synth.activations_t(cols, T, seed=synth.seed(cfg, 1) + 10 * li, ld=ldx)
        out.append((lname, W, XT))
    return wl, out


def check_full(Y_dev, XT, Wm, T, bf16, chunk=4096):
    """Every element of Y^T [rows][T] against O8, token chunk by token chunk."""
    worst = -np.inf
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        Yref, Aref = oracle.gemm_ref(np.ascontiguousarray(XT[:, t0:t1]), Wm)
        Y = Y_dev[:, t0:t1].float().cpu().numpy().astype(np.float64)
        tol = oracle.tolerance(Yref, Aref, y_is_bf16=bf16)
        err = np.abs(Y - Yref) - tol
        bad = err > 0
        assert not bad.any(), f"tokens [{t0},{t1}): {bad.sum()} outside tolerance, worst excess {err.max()}"
        worst = max(worst, float(err.max()))
    return worst


def run_workload(name, tc):
    wl, layers = bench_inputs(name)
    V, M, T = wl["V"], wl["M"], wl["T"]
    Wd = [to_dev_bf16(W) for _, W, _ in layers]
    Ps, masks = vnm.prune_compress_batched(Wd, V, M, want_mask=True, tc=tc)
    torch.cuda.synchronize()
    for (lname, W, XT), P, mk in zip(layers, Ps, masks):
        # every batched entry == the oracle's prune + pack, byte for byte
        mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, V, M)
        assert np.array_equal(u32(mk), mask_ref), f"{lname}: mask"
        v, c, m = packed_np(P)
        assert np.array_equal(v, v_ref), f"{lname}: A_n"
        assert np.array_equal(c, c_ref), f"{lname}: A_i1"
        assert np.array_equal(m, m_ref), f"{lname}: A_i2"
        Xd = to_dev_bf16(XT[:, :T] if XT.shape[1] != T else XT, ld=XT.shape[1])
        Y = torch.empty((W.shape[0], XT.shape[1]), dtype=torch.bfloat16, device="cuda")
        ws = vnm.spmm_workspace(P.g, T, "cuda")
        vnm.spmm(Xd, P, T=T, out=Y[:, :T], workspace=ws)
        torch.cuda.synchronize()
        check_full(Y[:, :T], np.ascontiguousarray(XT[:, :T]), oracle.apply_mask(W, mask_ref, V, M), T, bf16=True)


def test_deit_s_bench_step_full():
    """The default bench step (DeiT-S 64:2:5, T = 50,432): batched prune + window form, default SpMM plans
    (CTA-pair resident-A kernel for qkv / fc1, single-CTA window kernel for proj / fc2), every output of every
    layer — proj included."""
    run_workload("deit_s", tc=True)


def test_llama_prefill_up_down_full():
    """Llama2-7B 64:2:5 prefill, T = 2048, the bench's three layers (window form, CTA-pair kernel), every output."""
    run_workload("llama_prefill", tc=True)


def test_llama_decode_full_bench_inputs():
    """Llama2-7B 64:2:5 decode, T = 16, the bench's layers (small-T plan), every output."""
    run_workload("llama_decode", tc=False)


def test_deit_b_bench_step_full():
    """DeiT-B 64:2:8 (BJ configs[2]), T = 50,432, batched pass + window form, every output."""
    run_workload("deit_b", tc=True)
