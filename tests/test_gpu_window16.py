"""The window-16 tensor-core form (include/vnm.h; 8 < M < 16 with M % 4 != 0, e.g. the paper's 128:2:9 / 10 / 11 / 13
of tab:bs-sped): packing decoded back to the oracle's masked W, and the window-form
kernels running it against the oracle's fp64 GEMM (O8) within the BASELINE.json tolerance."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
from tests.test_gpu_spmm import assert_within

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def decode_window16(P, rows, cols):
    """Host decode of the window-16 form: MMA mi = 2j + h holds, per row, 16 values = for blocks 4j + i (i = 0..3)
    the 2:4 groups 2h and 2h + 1 of the block's 16-channel window (channels 4 (2h + s) .. + 3), 2 values each;
    K-group gi = 2i + s of the MMA; its nibble in meta_tc's M = 128 lane order (lane (r%8) + 16 (r/16) + 8 (gi/4),
    bits 16 (r%16 >= 8) + 4 (gi%4)).  Window positions past the block (channel >= M) and pad blocks must carry
    zero values; every value lands exactly once."""
    g = P.g
    M = g.M
    n_mma = g.nb_pad // 2
    n_stage = (n_mma + 3) // 4
    rows_w = (g.rows_p + 127) // 128 * 128
    vals = P.values_tc.view(torch.int16).cpu().numpy().view(np.uint16).reshape(rows_w, 16 * n_mma)
    mt = P.meta_tc.cpu().numpy().view(np.uint32).reshape(rows_w // 128, n_stage, 128, 4)
    dense = np.zeros((rows_w, g.cols_p + 16), np.uint16)
    for r in range(rows_w):
        t, rr = divmod(r, 128)
        jb = 0 if (rr % 16) < 8 else 1
        for mi in range(n_mma):
            j, h = divmod(mi, 2)
            st, k = divmod(mi, 4)
            for gi in range(8):
                i, s = divmod(gi, 2)
                b = 4 * j + i
                lane = (rr % 8) + 16 * (rr // 16) + 8 * (gi // 4)
                nib = (int(mt[t, st, lane, k]) >> (16 * jb + 4 * (gi % 4))) & 0xF
                for q, pos in enumerate((nib & 3, nib >> 2)):
                    v = vals[r, 16 * mi + 2 * gi + q]
                    ch = 4 * (2 * h + s) + pos
                    if ch >= M or b >= g.nb:
                        assert v & 0x7FFF == 0, (r, b, h, s, ch)
                        continue
                    c = b * M + ch
                    assert dense[r, c] == 0 or v & 0x7FFF == 0, (r, c)
                    if v & 0x7FFF:
                        dense[r, c] = v
    return dense[:rows, :cols]


@pytest.mark.parametrize("V", [32, 64, 128])
@pytest.mark.parametrize("M", [9, 10, 11, 13, 14, 15])
@pytest.mark.parametrize("rows,cols,kind", [(200, 333, "outlier"), (128, 100, "int")])
def test_window16_decodes_to_oracle(V, M, rows, cols, kind):
    """prune_compress(tc) == vnm_pack_tc of its canonical output == the batched pass, and the form holds exactly
    the oracle's masked W, value for value."""
    W = synth.weights(rows, cols, seed=rows + cols + M + V, kind=kind)
    Wd = to_dev_bf16(W)
    P = vnm.prune_compress(Wd, V, M, tc=True)
    Q = vnm.prune_compress(Wd, V, M)
    vnm.pack_tc(Q)
    B = vnm.prune_compress_batched([Wd, Wd], V, M, tc=True)
    torch.cuda.synchronize()
    for R in (Q, *B):
        assert torch.equal(P.values_tc.view(torch.int16), R.values_tc.view(torch.int16))
        assert torch.equal(P.meta_tc, R.meta_tc)
    Wm = oracle.apply_mask(W, oracle.prune(W, V, M), V, M)
    zero = lambda a: np.where((a & 0x7FFF) == 0, 0, a)
    assert np.array_equal(zero(decode_window16(P, rows, cols)), zero(Wm))


# (rows, cols, V, M, T, out): the plan the default choice takes is noted (n_stage = nb_pad / 8 4-MMA stages)
CASES = [
    (256, 1000, 64, 9, 300, "f32"),    # 14 stages, 2 row tiles -> pair kernel (tc2)
    (200, 333, 128, 13, 129, "bf16"),  # 4 stages -> 1-CTA kernel, ragged rows / K / tokens
    (384, 770, 32, 11, 264, "f32"),    # 3 row tiles -> 1-CTA kernel
    (130, 4096, 128, 13, 256, "bf16"),  # Llama-K, 40 stages -> tc2, half-empty row pair
    (256, 640, 64, 10, 301, "bf16"),   # Y^T row not a multiple of 16 B -> the gather plan
    (64, 50, 64, 15, 96, "f32"),       # one block group
    (512, 1000, 128, 14, 520, "bf16"),
]


@pytest.mark.parametrize("rows,cols,V,M,T,od", CASES)
def test_window16_spmm_matches_oracle(rows, cols, V, M, T, od):
    W = synth.weights(rows, cols, seed=rows * 7 + M, kind="outlier")
    XT = synth.activations_t(cols, T, seed=cols + T)
    Wm = oracle.apply_mask(W, oracle.prune(W, V, M), V, M)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=True)
    dt = torch.bfloat16 if od == "bf16" else torch.float32
    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=dt)
    torch.cuda.synchronize()
    assert_within(Y.float().cpu().numpy().astype(np.float64), Yref, Aref, bf16=od == "bf16")


def test_window16_ragged_rows_without_gather_plan_are_unsupported():
    """A Y^T row that is not a multiple of 16 bytes cannot take the window-form kernels (their TMA stores write
    whole 16-byte chunks, reading Q24); the window-16 form then needs the gather plan (V = 64 / 128 / 256) or the
    small-T plan (T <= 32) — V = 32 at T = 257 has neither and is refused before any launch, nothing written."""
    W = synth.weights(128, 200, seed=5)
    P = vnm.prune_compress(to_dev_bf16(W), 32, 11, tc=True)
    X = to_dev_bf16(synth.activations_t(200, 257, seed=6))
    with pytest.raises(vnm.VnmError) as e:
        vnm.spmm(X, P, T=257)
    assert e.value.status == vnm.VNM_ERR_UNSUPPORTED


def test_window16_integer_inputs_exact():
    """Small integers in W and X^T: every product and partial sum is exact in fp32, so the window-16 kernels must
    reproduce the oracle exactly (a misplaced window, step or nibble shows up as a wrong integer)."""
    for rows, cols, V, M, T in ((256, 1000, 64, 9, 256), (256, 777, 128, 13, 192), (384, 300, 64, 11, 128)):
        W = synth.weights(rows, cols, seed=rows + M, kind="int")
        XT = synth.activations_t(cols, T, seed=cols + M, kind="int")
        Wm = oracle.apply_mask(W, oracle.prune(W, V, M), V, M)
        Yref, _ = oracle.gemm_ref(XT, Wm)
        P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=True)
        Y = vnm.spmm(to_dev_bf16(XT), P, T=T).cpu().numpy().astype(np.float64)
        assert np.array_equal(Y, Yref), (rows, cols, V, M, T)


def test_window16_llama_up_v128_m13_sampled():
    """The bench's llama_prefill_v128_m13 up layer (11008 x 4096 at 128:2:13, T = 2048, bf16 Y^T) through the
    default plan, 3000 sampled outputs against the oracle computed one by one."""
    rows, cols, V, M, T = 11008, 4096, 128, 13, 2048
    W = synth.weights(rows, cols, seed=41, kind="outlier")
    XT = synth.activations_t(cols, T, seed=42)
    P, mask_d = vnm.prune_compress(to_dev_bf16(W), V, M, want_mask=True, tc=True)
    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=torch.bfloat16).float().cpu().numpy().astype(np.float64)
    mask = mask_d.cpu().numpy().view(np.uint32)
    assert np.array_equal(mask, oracle.prune(W, V, M))
    Wm = oracle.apply_mask(W, mask, V, M)
    g = synth.rng(43)
    o, t = g.integers(0, rows, 3000), g.integers(0, T, 3000)
    o[:4], t[:4] = [0, rows - 1, 0, rows - 1], [0, 0, T - 1, T - 1]
    Yref, Aref = oracle.gemm_ref_sampled(XT, Wm, o, t)
    tol = oracle.tolerance(Yref, Aref, y_is_bf16=True)
    assert np.all(np.abs(Y[o, t] - Yref) <= tol)
    assert np.isfinite(Y).all()


CHILD = r"""
import numpy as np, torch, oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
from tests.test_gpu_spmm import assert_within
for rows, cols, V, M, T, od in [(256, 1000, 64, 9, 300, 'f32'), (200, 333, 128, 13, 129, 'bf16'),
                                (384, 770, 32, 11, 264, 'f32'), (130, 4096, 128, 13, 256, 'bf16'),
                                (64, 50, 64, 15, 96, 'f32')]:
    W = synth.weights(rows, cols, seed=rows + T); XT = synth.activations_t(cols, T, seed=cols + T)
    Wm = oracle.apply_mask(W, oracle.prune(W, V, M), V, M)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=True)
    dt = torch.bfloat16 if od == 'bf16' else torch.float32
    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=dt).float().cpu().numpy().astype(np.float64)
    assert_within(Y, Yref, Aref, bf16=od == 'bf16')
print('ok')
"""


@pytest.mark.parametrize("plan", ["1", "2"])
def test_window16_each_kernel_forced(plan):
    """Both window-form kernels on the window-16 form — VNM_TC_PLAN=1 (single CTA, M = 128) and 2 (CTA pairs,
    M = 256) — in a child process (the plan switch is read once per process)."""
    env = dict(os.environ, VNM_TC_PLAN=plan, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
