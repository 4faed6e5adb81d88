"""GPU parity for the V:N:M SpMM (§8 rows a6-a8) against the oracle's fp64 product.

Bar (BASELINE.json): |Y - Y_ref| <= 1e-3 * sum_k |x w| + 1e-6 per element on fp32 Y; bf16 Y adds
2^-8 |Y_ref| (Q14).  Calls go through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


def make(rows, cols, V, M, T, seed, wkind="normal", xkind="normal"):
    W = synth.weights(rows, cols, seed=seed, kind=wkind)
    XT = synth.activations_t(cols, T, seed=seed + 1, kind=xkind)
    mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
    Wm = oracle.apply_mask(W, mask, V, M)
    return W, XT, Wm


def gpu_y(W, XT, V, M, T, out_dtype=torch.float32, tc=False):
    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=tc)
    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=out_dtype)
    torch.cuda.synchronize()
    return Y.float().cpu().numpy().astype(np.float64)


def assert_within(Y, Yref, Aref, bf16=False):
    tol = oracle.tolerance(Yref, Aref, y_is_bf16=bf16)
    err = np.abs(Y - Yref)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} / {bad.size} outside tolerance; worst {np.max(err - tol)}"


def test_config1_toy():
    """BJ config 1: 64:2:8, W 128x64, X 16x64 (T = 16)."""
    W, XT, Wm = make(128, 64, 64, 8, 16, seed=synth.seed(1, 0))
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, 8, 16), Yref, Aref)


@pytest.mark.parametrize("T", [1, 2, 7, 8, 15, 16, 33, 63, 64, 65, 100, 128, 129, 200, 256, 257, 300, 513])
def test_token_tails(T):
    W, XT, Wm = make(192, 300, 64, 5, T, seed=T)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, 5, T), Yref, Aref)


@pytest.mark.parametrize("rows,cols,M", [(70, 23, 5), (64, 4, 4), (128, 1, 5), (65, 1000, 7), (130, 257, 16),
                                         (64, 2048, 8), (256, 640, 6), (64, 5000, 5), (200, 333, 32)])
def test_shapes_and_k_tails(rows, cols, M):
    T = 96
    W, XT, Wm = make(rows, cols, 64, M, T, seed=rows + cols)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, M, T), Yref, Aref)


def test_bf16_output():
    W, XT, Wm = make(256, 512, 64, 5, 200, seed=3)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, 5, 200, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)


def test_identity_x_is_exact():
    """Pin P10: X = I  =>  Y^T = W' exactly (each output is one weight times 1.0)."""
    rows, cols, M = 128, 200, 5
    W = synth.weights(rows, cols, seed=11)
    XT = synth.f32_to_bf16_bits(np.eye(cols, dtype=np.float32))
    mask = oracle.prune(W, 64, M)
    Wm = synth.bf16_bits_to_f32(oracle.apply_mask(W, mask, 64, M)).astype(np.float64)
    Y = gpu_y(W, XT, 64, M, cols)
    assert np.array_equal(Y, Wm)


def test_integer_inputs_exact():
    """Integer W, X: every product and partial sum is exact in fp32 => Y equals the oracle exactly."""
    W, XT, Wm = make(128, 400, 64, 5, 64, seed=5, wkind="int", xkind="int")
    Yref, _ = oracle.gemm_ref(XT, Wm)
    assert np.array_equal(gpu_y(W, XT, 64, 5, 64), Yref)


def test_linearity():
    """spmm(x1 + x2) == spmm(x1) + spmm(x2) within the tolerance."""
    rows, cols, T, M = 128, 320, 80, 5
    W = synth.weights(rows, cols, seed=21)
    x1 = synth.activations_t(cols, T, seed=22, kind="int")
    x2 = synth.activations_t(cols, T, seed=23, kind="int")
    xs = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(x1) + synth.bf16_bits_to_f32(x2))
    y = lambda x: gpu_y(W, x, 64, M, T)
    mask = oracle.prune(W, 64, M)
    _, A = oracle.gemm_ref(xs, oracle.apply_mask(W, mask, 64, M))
    assert np.all(np.abs(y(xs) - (y(x1) + y(x2))) <= 2e-3 * A + 1e-6)


def test_m4_matches_dense_24():
    """Pin P6 on the GPU: 64:2:4 SpMM == the plain 2:4 product (W (.) M dense, fp64)."""
    W, XT, Wm = make(256, 512, 64, 4, 128, seed=31)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, 4, 128), Yref, Aref)


def sampled_check(rows, cols, M, T, seed, n=3000, out_dtype=torch.float32, tc=False):
    W = synth.weights(rows, cols, seed=seed, kind="outlier")
    XT = synth.activations_t(cols, T, seed=seed + 1)
    Wd, Xd = to_dev_bf16(W), to_dev_bf16(XT)
    P, mask_d = vnm.prune_compress(Wd, 64, M, want_mask=True, tc=tc)
    Y = vnm.spmm(Xd, P, T=T, out_dtype=out_dtype)
    torch.cuda.synchronize()
    mask = mask_d.cpu().numpy().view(np.uint32)
    Wm = oracle.apply_mask(W, mask, 64, M)
    g = synth.rng(seed + 2)
    o = g.integers(0, rows, n)
    t = g.integers(0, T, n)
    # always include the corners
    o[:4] = [0, rows - 1, 0, rows - 1]
    t[:4] = [0, 0, T - 1, T - 1]
    Yref, Aref = oracle.gemm_ref_sampled(XT, Wm, o, t)
    Ys = Y.float()[torch.from_numpy(o).cuda(), torch.from_numpy(t).cuda()].cpu().numpy().astype(np.float64)
    tol = oracle.tolerance(Yref, Aref, y_is_bf16=out_dtype == torch.bfloat16)
    assert np.all(np.abs(Ys - Yref) <= tol)
    # and a property that holds everywhere: finite
    assert torch.isfinite(Y).all()


@pytest.mark.parametrize("tc", [False, True])
@pytest.mark.parametrize("rows,cols", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_llama_prefill_sampled(rows, cols, tc):
    """BJ config 4a at full size (T = 2048, 64:2:5), both plans (bench.py times the window plan, tc=True)."""
    sampled_check(rows, cols, 5, 2048, seed=rows + cols, out_dtype=torch.bfloat16, tc=tc)


@pytest.mark.parametrize("T", [1, 2, 4, 8, 16])
def test_llama_decode_full(T):
    """BJ config 4b: decode batch 1-16 at 64:2:5, every output compared."""
    rows, cols = 11008, 4096
    W = synth.weights(rows, cols, seed=40 + T)
    XT = synth.activations_t(cols, T, seed=50 + T)
    mask = oracle.prune(W, 64, 5)
    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, mask, 64, 5))
    assert_within(gpu_y(W, XT, 64, 5, T), Yref, Aref)


@pytest.mark.parametrize("rows,cols,T,M", [(70, 23, 3, 5), (200, 333, 17, 7), (128, 1000, 32, 8), (64, 4, 1, 4),
                                           (130, 2048, 24, 6), (4096, 11008, 9, 5), (11008, 4096, 31, 4)])
def test_slab_plan(rows, cols, T, M):
    """The small-T plan (T <= 32): dense X^T slice per unit by TMA, the kept rows gathered by ldmatrix;
    ragged rows / channels / tokens, stream-K splits on the Llama shapes, every output compared."""
    W, XT, Wm = make(rows, cols, 64, M, T, seed=rows + cols + T)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, M, T), Yref, Aref)
    assert_within(gpu_y(W, XT, 64, M, T, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)


@pytest.mark.parametrize("T,ld", [(17, 32), (5, 16), (32, 40)])
def test_slab_plan_strided_x(T, ld):
    """X^T with a leading dimension past T rounded to 8: the slab comes from a 2-D TMA instead of one bulk copy."""
    rows, cols, M = 192, 700, 6
    W, XT, Wm = make(rows, cols, 64, M, T, seed=T + ld)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    P = vnm.prune_compress(to_dev_bf16(W), 64, M)
    Xd = to_dev_bf16(XT, ld=ld)
    assert Xd.stride(0) == ld
    Y = vnm.spmm(Xd, P, T=T)
    torch.cuda.synchronize()
    assert_within(Y.cpu().numpy().astype(np.float64), Yref, Aref)


@pytest.mark.parametrize("tc", [False, True])
@pytest.mark.parametrize("rows,cols,M", [(1152, 384, 5), (384, 1536, 5), (3072, 768, 8), (768, 3072, 8)])
def test_deit_sampled(rows, cols, M, tc):
    """BJ configs 2/3: DeiT-S @64:2:5 and DeiT-B @64:2:8 with T = 197 * 256 tokens (both plans)."""
    sampled_check(rows, cols, M, 197 * 256, seed=rows * 3 + cols, out_dtype=torch.bfloat16, tc=tc)


@pytest.mark.parametrize("M", [4, 5, 6, 7, 8])
@pytest.mark.parametrize("rows,cols,T", [(128, 512, 192), (70, 23, 65), (200, 333, 193), (384, 1000, 500),
                                         (64, 40, 100), (1000, 257, 384)])
def test_window_plan(rows, cols, T, M):
    """The tensor-core window form (values_tc / meta_tc, T > 64): ragged rows / cols / tokens, every M <= 8."""
    W, XT, Wm = make(rows, cols, 64, M, T, seed=rows + 7 * cols + M)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, 64, M, T, tc=True), Yref, Aref)


def test_window_plan_exact_integers():
    """Integer W and X: the window plan (extra zero-valued positions included) is exact."""
    W, XT, Wm = make(256, 640, 64, 5, 256, seed=9, wkind="int", xkind="int")
    Yref, _ = oracle.gemm_ref(XT, Wm)
    assert np.array_equal(gpu_y(W, XT, 64, 5, 256, tc=True), Yref)


def test_window_plan_bf16_out_and_identity():
    rows, cols, M = 192, 200, 6
    W = synth.weights(rows, cols, seed=13)
    XT = synth.f32_to_bf16_bits(np.eye(cols, dtype=np.float32))
    mask = oracle.prune(W, 64, M)
    Wm = synth.bf16_bits_to_f32(oracle.apply_mask(W, mask, 64, M)).astype(np.float64)
    assert np.array_equal(gpu_y(W, XT, 64, M, cols, tc=True), Wm)
    W2, X2, Wm2 = make(300, 700, 64, 7, 333, seed=14)
    Yref, Aref = oracle.gemm_ref(X2, Wm2)
    assert_within(gpu_y(W2, X2, 64, 7, 333, out_dtype=torch.bfloat16, tc=True), Yref, Aref, bf16=True)


def test_determinism():
    W, XT, _ = make(256, 1000, 64, 5, 300, seed=77)
    assert np.array_equal(gpu_y(W, XT, 64, 5, 300), gpu_y(W, XT, 64, 5, 300))


@pytest.mark.parametrize("V", [32, 128])
@pytest.mark.parametrize("rows,cols,T,M", [(256, 640, 300, 5), (384, 1000, 65, 8), (128, 333, 8, 6),
                                           (512, 4096, 256, 5), (640, 770, 1, 4)])
def test_window_plan_any_v(V, rows, cols, T, M):
    """NEXT-1: V != 64 (e.g. the paper's 128:2:M) runs in the window form at any T."""
    W, XT, Wm = make(rows, cols, V, M, T, seed=V + rows + cols + M)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, V, M, T, tc=True), Yref, Aref)


def test_v32_without_window_form_is_unsupported():
    """V = 32 past the small-T range needs the tensor-core form (the gather plan tiles 64-row V-blocks)."""
    W = synth.weights(256, 256, seed=3)
    P = vnm.prune_compress(to_dev_bf16(W), 32, 5)
    with pytest.raises(RuntimeError):
        vnm.spmm(to_dev_bf16(synth.activations_t(256, 128, seed=4)), P, T=128)


@pytest.mark.parametrize("V,M", [(128, 9), (128, 10), (128, 11), (128, 13), (128, 5), (256, 7)])
@pytest.mark.parametrize("rows,cols,T", [(384, 1500, 100), (300, 777, 257)])
def test_gather_plan_v128_any_m(V, M, rows, cols, T):
    """NEXT-1: the paper's 128:2:9 / 10 / 11 / 13 points (tab:bs-sped), which have no tensor-core form,
    at prefill-sized T through the gather plan (64-row tiles sharing their V-block's A_i1 row); V = 256 too."""
    W, XT, Wm = make(rows, cols, V, M, T, seed=V + M + rows + T, wkind="outlier")
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, V, M, T), Yref, Aref)
    assert_within(gpu_y(W, XT, V, M, T, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)


def test_pair_resident_kernel_forced():
    """The CTA-pair resident-A kernel (spmm_tc3.cu) on every shape class it accepts — fp32 and bf16 Y^T, ragged
    rows / K / tokens (T % 8 != 0 exercises the element-wise tail stores), every window-form M, V = 32 / 128 —
    forced with VNM_TC_PLAN=3 in a child process (the plan switch is read at library load).  By default it only
    runs for the DeiT-S-like shapes (test_deit_sampled covers that choice)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, oracle\n"
        "from paper_2410_16135_b200 import synth, vnm\n"
        "from tests.gpu_util import to_dev_bf16\n"
        "cases = [(1536, 384, 64, 5, 1000, 'f32'), (1152, 384, 64, 5, 677, 'bf16'), (200, 333, 64, 6, 193, 'f32'),\n"
        "         (70, 23, 64, 7, 65, 'bf16'), (384, 1000, 64, 8, 500, 'f32'), (256, 640, 64, 4, 300, 'bf16'),\n"
        "         (256, 640, 32, 5, 301, 'f32'), (384, 770, 128, 8, 129, 'bf16'), (1000, 257, 64, 5, 2049, 'f32'),\n"
        "         (512, 1000, 64, 16, 300, 'bf16'), (256, 333, 64, 12, 129, 'f32')]\n"
        "for rows, cols, V, M, T, od in cases:\n"
        "    W = synth.weights(rows, cols, seed=rows + T); XT = synth.activations_t(cols, T, seed=cols + T)\n"
        "    mask = oracle.prune(W, V, M)\n"
        "    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, mask, V, M))\n"
        "    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=True)\n"
        "    dt = torch.bfloat16 if od == 'bf16' else torch.float32\n"
        "    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=dt).float().cpu().numpy().astype(np.float64)\n"
        "    tol = oracle.tolerance(Yref, Aref, y_is_bf16=(od == 'bf16'))\n"
        "    assert np.all(np.abs(Y - Yref) <= tol), (rows, cols, V, M, T, od, float(np.max(np.abs(Y - Yref) - tol)))\n"
        "print('ok')\n")
    env = dict(os.environ, VNM_TC_PLAN="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("V", [64, 32, 128])
@pytest.mark.parametrize("rows,cols,T,M", [(256, 640, 300, 16), (200, 333, 65, 12), (384, 1000, 129, 16),
                                           (130, 4096, 256, 16), (64, 50, 100, 32)])
def test_natural_24_form(V, rows, cols, T, M):
    """M % 4 == 0, M > 8 (e.g. the 64:2:16 point of BJ config 5): the masked W is 2:4-sparse in channel order,
    and vnm_spmm runs its natural 2:4 tensor-core form through the window-form kernels (M = 4 view)."""
    W, XT, Wm = make(rows, cols, V, M, T, seed=V + rows + cols + M + T)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, V, M, T, tc=True), Yref, Aref)
    assert_within(gpu_y(W, XT, V, M, T, out_dtype=torch.bfloat16, tc=True), Yref, Aref, bf16=True)


@pytest.mark.parametrize("rows,cols", [(11008, 4096), (4096, 11008)])
def test_llama_m16_sampled(rows, cols):
    """BJ config 5 at M = 16, T = 2048 through the natural 2:4 form (sampled rows against the oracle)."""
    sampled_check(rows, cols, 16, 2048, seed=rows + cols + 16, out_dtype=torch.bfloat16, tc=True)


@pytest.mark.parametrize("graph", [False, True])
def test_chained_small_t_layers_see_the_previous_output(graph):
    """Two small-T SpMMs back to back on one stream, the second reading the first's Y^T as its X^T (a decode
    MLP), eagerly and replayed from a CUDA graph.  The small-T plan is launched with programmatic dependent
    launch; its griddepcontrol.wait (after the prologue) is what orders the second kernel's reads after the
    first's writes.  Y1's buffer is NaN-filled first, so a read of unwritten data shows as NaN / a mismatch.
    (The race itself is pinned by test_pdl_wait_orders_reads_after_a_delayed_producer.)"""
    T, M = 16, 5
    W1 = synth.weights(256, 512, seed=31)
    W2 = synth.weights(384, 256, seed=32)
    X = synth.activations_t(512, T, seed=33)
    P1 = vnm.prune_compress(to_dev_bf16(W1), 64, M)
    P2 = vnm.prune_compress(to_dev_bf16(W2), 64, M)
    Xd = to_dev_bf16(X)
    Y1 = torch.empty((256, T), dtype=torch.bfloat16, device="cuda")
    Y2 = torch.empty((384, T), dtype=torch.float32, device="cuda")
    ws1 = vnm.spmm_workspace(P1.g, T, "cuda")
    ws2 = vnm.spmm_workspace(P2.g, T, "cuda")

    def run():
        Y1.fill_(float("nan"))
        vnm.spmm(Xd, P1, T=T, out=Y1, workspace=ws1)
        vnm.spmm(Y1, P2, T=T, out=Y2, workspace=ws2)

    if graph:
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        for _ in range(3):
            g.replay()
    else:
        for _ in range(3):
            run()
    torch.cuda.synchronize()
    y1 = Y1.view(torch.int16).cpu().numpy().view(np.uint16)
    assert not torch.isnan(Y1).any()
    Wm2 = oracle.apply_mask(W2, oracle.prune(W2, 64, M), 64, M)
    Yref, Aref = oracle.gemm_ref(y1, Wm2)
    assert_within(Y2.cpu().numpy().astype(np.float64), Yref, Aref)


# ---------------------------------------------------------------------------------------------- small-T plan
@pytest.mark.parametrize("rows,cols,V,M,T", [
    (256, 640, 128, 5, 16), (384, 1000, 128, 8, 1), (300, 2000, 128, 9, 7), (512, 1500, 128, 10, 16),
    (200, 777, 128, 11, 24), (640, 3000, 128, 13, 32), (256, 640, 32, 5, 9), (130, 500, 32, 7, 16),
    (200, 300, 16, 5, 5), (96, 257, 16, 8, 32), (512, 1024, 256, 5, 16), (600, 999, 256, 6, 3),
    (192, 640, 64, 9, 16), (130, 1100, 64, 13, 8), (256, 4096, 64, 16, 16), (64, 100, 64, 32, 12),
    (1000, 333, 64, 4, 17)])
def test_smallt_any_v_any_m(rows, cols, V, M, T):
    """The small-T plan reads only the canonical arrays (A_n / A_i1 / A_i2), so it serves every V >= 16 and
    every M — incl. the paper's 128:2:9 / 10 / 11 / 13 points (tab:bs-sped) — at decode sizes;
    ragged rows, channels and tokens, fp32 and bf16 Y^T, every output compared."""
    W, XT, Wm = make(rows, cols, V, M, T, seed=rows + cols + V + M + T, wkind="outlier")
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    assert_within(gpu_y(W, XT, V, M, T), Yref, Aref)
    assert_within(gpu_y(W, XT, V, M, T, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)


@pytest.mark.parametrize("V,M", [(128, 5), (128, 8), (128, 13), (64, 16)])
@pytest.mark.parametrize("T", [1, 16])
def test_llama_decode_any_vm_full(V, M, T):
    """Llama up 11008 x 4096 at decode sizes for the paper's V = 128 points and 64:2:16, every output compared."""
    rows, cols = 11008, 4096
    W = synth.weights(rows, cols, seed=60 + T + M, kind="outlier")
    XT = synth.activations_t(cols, T, seed=70 + T)
    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, oracle.prune(W, V, M), V, M))
    assert_within(gpu_y(W, XT, V, M, T, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)


def _spmm_raw(Xd, P, T, Y, ws, ws_bytes):
    """vnm_spmm through the C ABI with an explicit (possibly NULL) workspace."""
    import ctypes
    cp = P.c()
    st = vnm.lib().vnm_spmm(ctypes.c_void_p(Xd.data_ptr()), Xd.stride(0), T, ctypes.byref(cp),
                            ctypes.c_void_p(Y.data_ptr()), Y.stride(0),
                            vnm.VNM_BF16 if Y.dtype == torch.bfloat16 else vnm.VNM_F32,
                            None if ws is None else ctypes.c_void_p(ws.data_ptr()), ws_bytes,
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0, vnm.status_string(st)


@pytest.mark.parametrize("rows,cols,M,T", [(11008, 4096, 5, 16), (4096, 11008, 5, 3), (300, 777, 9, 20),
                                           (1024, 11008, 13, 32), (512, 11008, 8, 16)])
def test_smallt_without_workspace(rows, cols, M, T):
    """No workspace: the small-T plan gives every CTA whole row groups (nothing is cut between CTAs).  The M = 13 /
    M = 8, T = 16 cases run a 3- / 6-slot ring with 3 phases in use over 27- / 43-unit pieces (4 / 6 A_i2 boxes:
    the idle phase's warps must not hold a box)."""
    W, XT, Wm = make(rows, cols, 64, M, T, seed=rows + M + T)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    P = vnm.prune_compress(to_dev_bf16(W), 64, M)
    Y = torch.empty((rows, (T + 7) // 8 * 8), dtype=torch.float32, device="cuda")[:, :T]
    _spmm_raw(to_dev_bf16(XT), P, T, Y, None, 0)
    torch.cuda.synchronize()
    assert_within(Y.cpu().numpy().astype(np.float64), Yref, Aref)


def test_workspace_reused_across_shapes():
    """ONE workspace (zeroed once, sized for the largest call) serves calls of different geometry and T in any
    order on a stream (include/vnm.h): the tickets sit at a fixed offset and every call leaves them zero, so
    the partials one call leaves behind never look like tickets to the next."""
    shapes = [(11008, 4096, 5, 32), (4096, 11008, 5, 16), (4096, 4096, 5, 8), (11008, 4096, 5, 1), (512, 3000, 11, 24)]
    cases = []
    for i, (rows, cols, M, T) in enumerate(shapes):
        W, XT, Wm = make(rows, cols, 64, M, T, seed=100 + i)
        Yref, Aref = oracle.gemm_ref(XT, Wm)
        cases.append((vnm.prune_compress(to_dev_bf16(W), 64, M), to_dev_bf16(XT), T, Yref, Aref))
    nws = max(vnm.spmm_workspace_bytes(P.g, T) for P, _, T, _, _ in cases)
    ws = torch.empty(nws // 4 + 4, dtype=torch.float32, device="cuda")
    assert vnm.lib().vnm_spmm_workspace_init(ctypes_ptr(ws), ws.numel() * 4, None) == 0
    for rep in range(2):
        for P, Xd, T, Yref, Aref in (cases if rep == 0 else cases[::-1]):
            Y = torch.empty((P.g.rows, (T + 7) // 8 * 8), dtype=torch.float32, device="cuda")[:, :T]
            _spmm_raw(Xd, P, T, Y, ws, ws.numel() * 4)
            torch.cuda.synchronize()
            assert_within(Y.cpu().numpy().astype(np.float64), Yref, Aref)


def ctypes_ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def test_pdl_wait_orders_reads_after_a_delayed_producer():
    """The small-T SpMM is launched with programmatic dependent launch and reads its X^T only after
    griddepcontrol.wait.  Here its producer is a one-CTA kernel (test-only probe library) that releases its
    dependents at once and writes X^T only after spinning ~0.5 ms, so the SpMM's CTAs run DURING the spin: a
    missing or misplaced wait reads the NaN-filled buffer and fails this test every time, not by chance."""
    import ctypes
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    probe = os.path.join(root, "tests", "probes", "libvnm_probe.so")
    if not os.path.exists(probe):
        pytest.skip("tests/probes/libvnm_probe.so not built")
    PL = ctypes.CDLL(probe)
    PL.vnm_probe_delayed_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_longlong,
                                          ctypes.c_void_p]
    rows, cols, M, T = 4096, 4096, 5, 16
    W, XT, Wm = make(rows, cols, 64, M, T, seed=321)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    P = vnm.prune_compress(to_dev_bf16(W), 64, M)
    src = to_dev_bf16(XT)
    assert src.stride(0) == T
    X = torch.empty_like(src)
    Y = torch.empty((rows, T), dtype=torch.float32, device="cuda")
    ws = vnm.spmm_workspace(P.g, T, "cuda")
    stream = torch.cuda.current_stream()
    for _ in range(3):
        X.fill_(float("nan"))
        Y.zero_()
        assert PL.vnm_probe_delayed_copy(X.data_ptr(), src.data_ptr(), X.numel() * 2, 1_000_000,
                                         stream.cuda_stream) == 0
        vnm.spmm(X, P, T=T, out=Y, workspace=ws)
        torch.cuda.synchronize()
        assert not torch.isnan(Y).any()
        assert_within(Y.cpu().numpy().astype(np.float64), Yref, Aref)


def test_binding_validates_out_and_xt():
    """vnm.spmm checks `out` / `XT` extents and strides before the call (an undersized or strided `out` would
    otherwise become an out-of-bounds device write)."""
    W = synth.weights(128, 64, seed=1)
    P = vnm.prune_compress(to_dev_bf16(W), 64, 8)
    X = to_dev_bf16(synth.activations_t(64, 16, seed=2))
    with pytest.raises(ValueError):
        vnm.spmm(X, P, T=16, out=torch.empty((127, 16), device="cuda"))
    with pytest.raises(ValueError):
        vnm.spmm(X, P, T=16, out=torch.empty((128, 8), device="cuda"))
    with pytest.raises(ValueError):
        vnm.spmm(X, P, T=16, out=torch.empty((16, 128), device="cuda").t())
    with pytest.raises(ValueError):
        vnm.spmm(X, P, T=17)
    with pytest.raises(ValueError):
        vnm.spmm(X.t().contiguous().t(), P, T=16)
