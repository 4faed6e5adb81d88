"""Out-of-bounds-write and determinism checks for every kernel / plan (the pool's compute-sanitizer is closed:
VERDICT r1 item 8 asked for memcheck / racecheck; these are the in-repo substitutes).

* Canaries: every output buffer (Y^T, the packed arrays, the split-K workspace) is allocated with guard space
  before and after the region the C ABI may write (include/vnm.h: only rows < g.rows and tokens < T of Y^T; the
  packed arrays' documented extents; the workspace's vnm_spmm_workspace_bytes), filled with a sentinel bit
  pattern, and compared bit for bit after the call.
* Determinism ("identical inputs give byte-identical outputs"): the small-T plan finishes row groups cut
  between CTAs through one of three paths decided by timing (the last piece with every other piece in, the last
  arriver after publishing, or the fix-up warp); the canonical right-fold order makes all of them bit-identical,
  so repeated calls must agree bit for bit."""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu

SENT16 = 0x7FA1   # a NaN bf16 pattern no kernel writes
SENT32 = 0x7FC0DEAD

PLANS = [
    # name, rows, cols, V, M, T, tc
    ("small-T 64:2:5", 4096, 4096, 64, 5, 16, False),
    ("small-T V=128 M=13 T=5", 300, 2000, 128, 13, 5, False),
    ("small-T V=16", 200, 300, 16, 5, 9, False),
    ("small-T T=32", 1000, 777, 64, 6, 32, False),
    ("gather 64:2:9", 192, 333, 64, 9, 48, False),
    ("window 1-CTA", 256, 640, 64, 5, 300, True),
    ("window pairs", 512, 4096, 64, 5, 512, True),
    ("window resident pairs", 1536, 384, 64, 5, 8200, True),
    ("natural 2:4", 256, 640, 64, 16, 200, True),
    ("window V=32", 256, 640, 32, 7, 129, True),
    ("window-16 1-CTA", 200, 333, 128, 13, 136, True),
    ("window-16 pairs", 256, 1000, 64, 9, 264, True),
    ("window-16 ragged -> gather", 200, 333, 128, 11, 129, True),
]


@pytest.mark.parametrize("name,rows,cols,V,M,T,tc", PLANS)
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_spmm_writes_only_its_region(name, rows, cols, V, M, T, tc, out_dtype):
    W = synth.weights(rows, cols, seed=rows + cols + M, kind="outlier")
    XT = synth.activations_t(cols, T, seed=T + 3)
    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=tc)
    gr, gc = 5, 24                                 # guard rows above / below, guard tokens right of T
    ldy = (T + gc + 7) // 8 * 8
    isz = 2 if out_dtype == torch.bfloat16 else 4
    it = torch.int16 if isz == 2 else torch.int32
    sent = SENT16 if isz == 2 else SENT32
    buf = torch.full(((rows + 2 * gr) * ldy + 64,), sent if isz == 4 else sent - 65536 if sent > 32767 else sent,
                     dtype=it, device="cuda")
    Y = buf[gr * ldy:(gr + rows) * ldy].view(rows, ldy).view(out_dtype)[:, :T]
    nws = vnm.spmm_workspace_bytes(P.g, T)
    ws = None
    if nws:
        ws_buf = torch.full((nws // 4 + 64,), SENT32 - 2**32 if SENT32 > 2**31 - 1 else SENT32, dtype=torch.int32,
                            device="cuda")
        ws_buf[:nws // 4].zero_()
        ws = ws_buf[:nws // 4].view(torch.float32)
    vnm.spmm(to_dev_bf16(XT), P, T=T, out=Y, workspace=ws)
    torch.cuda.synchronize()
    b = buf.cpu().numpy().view(np.uint16 if isz == 2 else np.uint32)
    full = b[:(rows + 2 * gr) * ldy].reshape(rows + 2 * gr, ldy)
    assert (full[:gr] == sent).all() and (full[gr + rows:] == sent).all(), f"{name}: rows outside [0, rows) written"
    assert (full[gr:gr + rows, T:] == sent).all(), f"{name}: tokens >= T written"
    assert (b[(rows + 2 * gr) * ldy:] == sent).all()
    if ws is not None:
        wb = ws_buf.cpu().numpy().view(np.uint32)
        assert (wb[nws // 4:] == SENT32).all(), f"{name}: written past the workspace"
    mask = oracle.prune(W, V, M)
    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, mask, V, M))
    Yg = full[gr:gr + rows, :T]
    Yg = (Yg.astype(np.uint32) << 16).view(np.float32) if isz == 2 else Yg.view(np.float32)
    assert np.all(np.abs(Yg.astype(np.float64) - Yref) <= oracle.tolerance(Yref, Aref, y_is_bf16=isz == 2))


@pytest.mark.parametrize("rows,cols,V,M,tc", [(1152, 384, 64, 5, True), (200, 333, 16, 7, False), (300, 1000, 128, 16, True),
                                              (70, 23, 64, 8, True), (96, 200, 32, 13, False), (300, 1000, 128, 13, True),
                                              (200, 500, 64, 9, True), (130, 700, 32, 11, True), (300, 1000, 64, 16, True)])
@pytest.mark.parametrize("with_mask", [True, False])
def test_prune_compress_writes_only_its_arrays(rows, cols, V, M, tc, with_mask):
    """The packed arrays (and the tensor-core form) are written exactly within their documented extents — with a
    mask output and without (for 8 < M <= 16 the two take different kernels: prune.cu + a pack, prune2 fused)."""
    W = synth.weights(rows, cols, seed=rows * M, kind="wide")
    g = vnm.geometry(rows, cols, V, M)
    sizes = {"values": g.rows_p * g.ld_val * 2, "col_idx": g.rows_p // V * g.nb_pad * 4, "meta": g.rows_p * g.ld_meta * 4,
             "mask": g.rows_p * g.ld_mask * 4}
    if tc:
        nv, nm = vnm.tc_bytes(g)
        sizes.update(values_tc=nv, meta_tc=nm)
    bufs = {k: torch.full((n // 4 + 32,), -559038737, dtype=torch.int32, device="cuda") for k, n in sizes.items()}
    view = lambda k, dt: bufs[k][:sizes[k] // 4].view(dt)
    P = vnm.Packed(g, view("values", torch.bfloat16).view(g.rows_p, g.ld_val),
                   view("col_idx", torch.uint8).view(g.rows_p // V, g.nb_pad, 4), view("meta", torch.int32).view(g.rows_p, g.ld_meta))
    if tc:
        P.values_tc, P.meta_tc = view("values_tc", torch.bfloat16), view("meta_tc", torch.int32)
    mask = view("mask", torch.int32).view(g.rows_p, g.ld_mask)
    import ctypes
    cp = P.c()
    Wd = to_dev_bf16(W)
    st = vnm.lib().vnm_prune_compress(ctypes.c_void_p(Wd.data_ptr()), Wd.stride(0), None, 0, ctypes.byref(g),
                                      ctypes.byref(cp), ctypes.c_void_p(mask.data_ptr()) if with_mask else None,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    for k, n in sizes.items():
        tail = bufs[k][n // 4:].cpu().numpy()
        assert (tail == -559038737).all(), f"{k}: written past its extent"
    mask_ref, v_ref, c_ref, m_ref = oracle.prune_pack(W, V, M)
    if with_mask:
        assert np.array_equal(mask.cpu().numpy().view(np.uint32), mask_ref)
    else:
        assert (bufs["mask"].cpu().numpy() == -559038737).all(), "mask written without a mask output"
    assert np.array_equal(P.values.view(torch.int16).cpu().numpy().view(np.uint16), v_ref)
    assert np.array_equal(P.meta.cpu().numpy().view(np.uint32), m_ref)
    assert np.array_equal(P.col_idx.cpu().numpy(), c_ref)


@pytest.mark.parametrize("rows,cols,M,T", [(11008, 4096, 5, 16), (4096, 11008, 5, 8), (4096, 4096, 8, 32), (300, 2000, 13, 3)])
def test_small_t_bitwise_deterministic(rows, cols, M, T):
    """20 calls of the stream-K small-T plan (row groups cut between CTAs) give bit-identical Y^T."""
    W = synth.weights(rows, cols, seed=rows + T)
    XT = synth.activations_t(cols, T, seed=cols + T)
    P = vnm.prune_compress(to_dev_bf16(W), 64, M)
    Xd = to_dev_bf16(XT)
    ws = vnm.spmm_workspace(P.g, T, "cuda")
    outs = []
    for _ in range(20):
        Y = vnm.spmm(Xd, P, T=T, out_dtype=torch.float32, workspace=ws)
        outs.append(Y.view(torch.int32).clone())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
