"""The C-ABI library loads and exports every symbol include/vnm.h declares; host-side validation
(geometry arithmetic, status codes for bad arguments) — no kernel launches, no GPU needed."""
import ctypes
import os
import re

import pytest

import oracle
from paper_2410_16135_b200 import vnm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vnm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:vnm_status|size_t|const char\*|uint64_t)\s+(vnm_\w+)\(", src, re.M)))


def test_exports_every_declared_symbol():
    L = vnm.lib()
    syms = declared_symbols()
    assert len(syms) >= 9, syms
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(vnm.EXPORTS) == syms


@pytest.mark.parametrize("rows,cols,V,M", [(128, 64, 64, 8), (1152, 384, 64, 5), (11008, 4096, 64, 5),
                                           (5, 7, 2, 5), (1, 1, 16, 5), (70, 23, 64, 5), (0, 0, 1, 4),
                                           (4096, 11008, 64, 7), (300, 1000, 256, 32)])
def test_geometry_matches_oracle(rows, cols, V, M):
    g = vnm.geometry(rows, cols, V, M).as_dict()
    assert g == oracle.geometry(rows, cols, V, M)


@pytest.mark.parametrize("V,M", [(3, 5), (0, 5), (512, 5), (64, 3), (64, 33), (-64, 5)])
def test_geometry_rejects(V, M):
    with pytest.raises(vnm.VnmError) as e:
        vnm.geometry(128, 64, V, M)
    assert e.value.status == vnm.VNM_ERR_SHAPE


def test_bytes():
    g = vnm.geometry(11008, 4096, 64, 5)
    L = vnm.lib()
    assert L.vnm_bytes(ctypes.byref(g), 0) == g.rows_p * g.ld_val * 2
    assert L.vnm_bytes(ctypes.byref(g), 1) == g.rows_p // 64 * g.nb_pad * 4
    assert L.vnm_bytes(ctypes.byref(g), 2) == g.rows_p * g.ld_meta * 4
    assert L.vnm_bytes(ctypes.byref(g), 3) == g.rows_p * g.ld_mask * 4
    assert L.vnm_bytes(ctypes.byref(g), 9) == 0


def test_status_codes_without_launch():
    L = vnm.lib()
    g = vnm.geometry(128, 64, 64, 8)
    fake = ctypes.c_void_p(1 << 20)          # never dereferenced: validation fails first
    odd = ctypes.c_void_p((1 << 20) + 2)     # misaligned
    # null W
    assert L.vnm_prune(None, 64, None, 0, ctypes.byref(g), fake, None) == vnm.VNM_ERR_ARG
    # ldw < cols
    assert L.vnm_prune(fake, 32, None, 0, ctypes.byref(g), fake, None) == vnm.VNM_ERR_SHAPE
    # misaligned W / ld not multiple of 8
    assert L.vnm_prune(odd, 64, None, 0, ctypes.byref(g), fake, None) == vnm.VNM_ERR_ALIGN
    assert L.vnm_prune(fake, 68, None, 0, ctypes.byref(g), fake, None) == vnm.VNM_ERR_ALIGN
    # geometry struct inconsistent with its own fields
    bad = vnm.geometry(128, 64, 64, 8)
    bad.nb_pad = 7
    assert L.vnm_prune(fake, 64, None, 0, ctypes.byref(bad), fake, None) == vnm.VNM_ERR_SHAPE
    # spmm: V = 16 runs only in the small-T plan (T <= 32); V = 8 nowhere; both rejected before any launch
    g16 = vnm.geometry(128, 64, 16, 8)
    P = vnm.CPacked(g16, 1 << 20, 1 << 20, 1 << 20)
    assert L.vnm_spmm(fake, 128, 128, ctypes.byref(P), fake, 128, 0, None, 0, None) == vnm.VNM_ERR_UNSUPPORTED
    g8 = vnm.geometry(128, 64, 8, 8)
    P8 = vnm.CPacked(g8, 1 << 20, 1 << 20, 1 << 20)
    assert L.vnm_spmm(fake, 16, 16, ctypes.byref(P8), fake, 16, 0, None, 0, None) == vnm.VNM_ERR_UNSUPPORTED
    P = vnm.CPacked(g, 1 << 20, 1 << 20, 1 << 20)
    assert L.vnm_spmm(fake, 16, 16, ctypes.byref(P), fake, 16, 7, None, 0, None) == vnm.VNM_ERR_ARG
    assert L.vnm_spmm(fake, 8, 16, ctypes.byref(P), fake, 16, 0, None, 0, None) == vnm.VNM_ERR_SHAPE
    assert L.vnm_spmm(fake, 12, 12, ctypes.byref(P), fake, 16, 0, None, 0, None) == vnm.VNM_ERR_ALIGN
    assert L.vnm_spmm(None, 16, 16, None, fake, 16, 0, None, 0, None) == vnm.VNM_ERR_ARG
    # compress: packed geometry must equal g
    P2 = vnm.CPacked(vnm.geometry(128, 64, 64, 5), 1 << 20, 1 << 20, 1 << 20)
    assert L.vnm_compress(fake, 64, fake, ctypes.byref(g), ctypes.byref(P2), None, None) == vnm.VNM_ERR_SHAPE
    # T = 0 is a no-op
    assert L.vnm_spmm(fake, 16, 0, ctypes.byref(P), fake, 16, 0, None, 0, None) == vnm.VNM_OK
    # batched prune: n out of range / NULL arrays are argument errors; an entry's error is returned before launch
    assert L.vnm_prune_compress_batched(0, None, None, None, None, None, None, None) == vnm.VNM_ERR_ARG
    assert L.vnm_prune_compress_batched(65, None, None, None, None, None, None, None) == vnm.VNM_ERR_ARG
    Pg = vnm.CPacked(g, 1 << 20, 1 << 20, 1 << 20)
    pw = (ctypes.c_void_p * 2)(fake, odd)
    lw = (ctypes.c_int64 * 2)(64, 64)
    po = (ctypes.c_void_p * 2)(ctypes.cast(ctypes.pointer(Pg), ctypes.c_void_p),
                               ctypes.cast(ctypes.pointer(Pg), ctypes.c_void_p))
    assert L.vnm_prune_compress_batched(2, pw, lw, None, None, po, None, None) == vnm.VNM_ERR_ALIGN
    # workspace init: nothing to do for 0 bytes; NULL with bytes is an argument error (no launch)
    assert L.vnm_spmm_workspace_init(None, 0, None) == vnm.VNM_OK
    assert L.vnm_spmm_workspace_init(None, 64, None) == vnm.VNM_ERR_ARG
    # the tensor-core form exists for M <= 8 (window), M % 4 == 0 (natural 2:4) and the other M < 16 (window-16),
    # not for M = 17 / 18; V outside [32, 128] never
    for M, has in [(5, True), (8, True), (12, True), (16, True), (9, True), (13, True), (15, True), (17, False),
                   (18, False), (20, True)]:
        gm = vnm.geometry(256, 1000, 64, M)
        assert (L.vnm_bytes(ctypes.byref(gm), 4) > 0) == has and (L.vnm_bytes(ctypes.byref(gm), 5) > 0) == has
        assert vnm.tc_applies(64, M) == has
    assert L.vnm_bytes(ctypes.byref(vnm.geometry(256, 1000, 256, 13)), 4) == 0
    # window-16 form: 8 values per block (two MMAs of 16 values per 4 blocks), meta_tc one word per MMA and lane
    g13 = vnm.geometry(300, 1000, 128, 13)  # cols_p 1001, nb 77, nb_pad 80, rows_w 384
    assert L.vnm_bytes(ctypes.byref(g13), 4) == 384 * 16 * 40 * 2
    assert L.vnm_bytes(ctypes.byref(g13), 5) == 3 * 10 * 128 * 4 * 4
    for s in (0, -1, -2, -3, -4, -5):
        assert vnm.status_string(s)


def test_no_cpu_path():
    import torch
    W = torch.zeros(128, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        vnm.prune(W, 64, 8)


def test_ria_argument_errors():
    """vnm_act_norms / vnm_ria_score reject bad arguments on the host, before any launch (NEXT-2)."""
    L = vnm.lib()
    assert L.vnm_ria_workspace_bytes(-1, 4) == 0
    assert L.vnm_ria_workspace_bytes(64, 512) == (1 * 512 + 1 * 64 + 2 * 512 + 64) * 4
    P = ctypes.c_void_p
    # negative shape, ld < cols, negative exponent
    assert L.vnm_ria_score(P(16), 8, -1, 4, None, 0.5, P(16), 8, P(16), 1 << 20, None) == vnm.VNM_ERR_SHAPE
    assert L.vnm_ria_score(P(16), 2, 4, 4, None, 0.5, P(16), 8, P(16), 1 << 20, None) == vnm.VNM_ERR_SHAPE
    assert L.vnm_ria_score(P(16), 8, 4, 4, None, -1.0, P(16), 8, P(16), 1 << 20, None) == vnm.VNM_ERR_SHAPE
    # missing workspace / too small, misaligned pointers
    assert L.vnm_ria_score(P(16), 8, 4, 4, None, 0.5, P(16), 8, None, 0, None) == vnm.VNM_ERR_ARG
    assert L.vnm_ria_score(P(16), 8, 4, 4, None, 0.5, P(16), 8, P(16), 8, None) == vnm.VNM_ERR_SHAPE
    assert L.vnm_ria_score(P(18), 8, 4, 4, None, 0.5, P(16), 8, P(16), 1 << 20, None) == vnm.VNM_ERR_ALIGN
    assert L.vnm_ria_score(P(16), 8, 0, 4, None, 0.5, None, 8, None, 0, None) == vnm.VNM_OK
    assert L.vnm_act_norms(P(16), 4, 3, 8, P(16), None) == vnm.VNM_ERR_SHAPE  # ldx < T
    assert L.vnm_act_norms(P(16), 8, 3, 8, None, None) == vnm.VNM_ERR_ARG
    assert L.vnm_act_norms(P(18), 8, 3, 8, P(16), None) == vnm.VNM_ERR_ALIGN


def test_spmm_batched_argument_errors_and_workspace():
    """vnm_spmm_batched validates before launching (no GPU needed) and sizes one workspace for the whole call."""
    L = vnm.lib()
    g = vnm.geometry(4096, 4096, 64, 5)
    fake = 1 << 20  # never dereferenced: validation fails first (array pointers fake and aligned)
    c = vnm.CPacked()
    c.g = g
    c.values = c.col_idx = c.meta = fake
    arr = lambda ty, xs: (ty * len(xs))(*xs)
    P = arr(ctypes.c_void_p, [ctypes.cast(ctypes.pointer(c), ctypes.c_void_p).value])
    X = arr(ctypes.c_void_p, [fake])
    Y = arr(ctypes.c_void_p, [fake])
    ld = arr(ctypes.c_int64, [16])
    # n out of range, NULL arrays, unknown flag bits
    assert L.vnm_spmm_batched(0, X, ld, 16, P, Y, ld, vnm.VNM_BF16, 0, None, 0, None) == vnm.VNM_ERR_ARG
    assert L.vnm_spmm_batched(65, X, ld, 16, P, Y, ld, vnm.VNM_BF16, 0, None, 0, None) == vnm.VNM_ERR_ARG
    assert L.vnm_spmm_batched(1, None, ld, 16, P, Y, ld, vnm.VNM_BF16, 0, None, 0, None) == vnm.VNM_ERR_ARG
    assert L.vnm_spmm_batched(1, X, ld, 16, P, Y, ld, vnm.VNM_BF16, 2, None, 0, None) == vnm.VNM_ERR_ARG
    # per-entry checks as vnm_spmm: T > ldx, misaligned Y
    assert L.vnm_spmm_batched(1, X, arr(ctypes.c_int64, [8]), 16, P, Y, ld, vnm.VNM_BF16, 0, None, 0, None) == vnm.VNM_ERR_SHAPE
    assert L.vnm_spmm_batched(1, X, ld, 16, P, arr(ctypes.c_void_p, [fake + 2]), ld, vnm.VNM_BF16, 0, None, 0,
                              None) == vnm.VNM_ERR_ALIGN
    # one workspace for the group >= every member's own
    gs = [vnm.geometry(4096, 4096, 64, 5), vnm.geometry(11008, 4096, 64, 5), vnm.geometry(4096, 11008, 64, 5)]
    b = vnm.spmm_batched_workspace_bytes(gs, 16)
    assert b >= max(vnm.spmm_workspace_bytes(x, 16) for x in gs) > 0
