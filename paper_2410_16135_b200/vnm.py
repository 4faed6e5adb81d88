"""Python binding of the C ABI in include/vnm.h (libvnm.so).  Argument marshalling only.

Every step of the V:N:M path runs in the CUDA kernels of ``csrc/``; this module turns torch CUDA
tensors into the device pointers / leading dimensions / stream the ABI takes, allocates the outputs
with torch (the library owns no device memory), and raises on any non-OK status.  There is no CPU
fallback: if ``libvnm.so`` is missing or a tensor is not on a CUDA device, the call raises.

Names follow the paper: ``prune`` is S_{V:N:M} (§3), ``compress`` produces
A_n / A_i1 / A_i2 (App. A), ``spmm`` is the V:N:M-sparse MM.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# VNM_LIB: an alternative build of the same library (experiments, e.g. the -DVNM_ABLATIONS libvnm_abl.so)
LIB_PATH = os.environ.get("VNM_LIB") or os.path.join(HERE, "libvnm.so")

VNM_OK, VNM_ERR_ARG, VNM_ERR_SHAPE, VNM_ERR_ALIGN, VNM_ERR_UNSUPPORTED, VNM_ERR_CUDA = 0, -1, -2, -3, -4, -5
VNM_F32, VNM_BF16 = 0, 1


class VnmError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


class Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("rows", "cols", "V", "M", "rows_p", "cols_p", "nb", "nb_pad", "ld_val", "ld_meta", "ld_mask")]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


class CPacked(ctypes.Structure):
    _fields_ = [("g", Geom), ("values", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("meta", ctypes.c_void_p),
                ("values_tc", ctypes.c_void_p), ("meta_tc", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None

EXPORTS = ["vnm_geometry", "vnm_bytes", "vnm_prune", "vnm_compress", "vnm_prune_compress",
           "vnm_prune_compress_batched", "vnm_pack_tc",
           "vnm_spmm", "vnm_spmm_workspace_bytes", "vnm_spmm_workspace_init", "vnm_spmm_batched",
           "vnm_spmm_batched_workspace_bytes", "vnm_act_norms", "vnm_ria_workspace_bytes", "vnm_ria_score",
           "vnm_permute_gain_workspace_bytes", "vnm_permute_gain", "vnm_permute_gain_out", "vnm_status_string",
           "vnm_launch_count"]


def lib():
    """Load libvnm.so (built by paper_2410_16135_b200/build.py / __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
            GP, PP = ctypes.POINTER(Geom), ctypes.POINTER(CPacked)
            L.vnm_geometry.argtypes = [i32, i32, i32, i32, GP]
            L.vnm_geometry.restype = ctypes.c_int
            L.vnm_bytes.argtypes = [GP, ctypes.c_int]
            L.vnm_bytes.restype = sz
            L.vnm_prune.argtypes = [P, i64, P, i64, GP, P, P]
            L.vnm_prune.restype = ctypes.c_int
            L.vnm_compress.argtypes = [P, i64, P, GP, PP, P, P]
            L.vnm_compress.restype = ctypes.c_int
            L.vnm_prune_compress.argtypes = [P, i64, P, i64, GP, PP, P, P]
            L.vnm_prune_compress.restype = ctypes.c_int
            L.vnm_prune_compress_batched.argtypes = [i32, P, P, P, P, P, P, P]
            L.vnm_prune_compress_batched.restype = ctypes.c_int
            L.vnm_pack_tc.argtypes = [PP, P]
            L.vnm_pack_tc.restype = ctypes.c_int
            L.vnm_spmm.argtypes = [P, i64, i32, PP, P, i64, ctypes.c_int, P, sz, P]
            L.vnm_spmm.restype = ctypes.c_int
            L.vnm_spmm_workspace_bytes.argtypes = [GP, i32]
            L.vnm_spmm_workspace_bytes.restype = sz
            L.vnm_spmm_workspace_init.argtypes = [P, sz, P]
            L.vnm_spmm_workspace_init.restype = ctypes.c_int
            L.vnm_spmm_batched.argtypes = [i32, P, P, i32, P, P, P, ctypes.c_int, ctypes.c_uint32, P, sz, P]
            L.vnm_spmm_batched.restype = ctypes.c_int
            L.vnm_spmm_batched_workspace_bytes.argtypes = [i32, P, i32]
            L.vnm_spmm_batched_workspace_bytes.restype = sz
            L.vnm_act_norms.argtypes = [P, i64, i32, i32, P, P]
            L.vnm_act_norms.restype = ctypes.c_int
            L.vnm_ria_workspace_bytes.argtypes = [i32, i32]
            L.vnm_ria_workspace_bytes.restype = sz
            L.vnm_ria_score.argtypes = [P, i64, i32, i32, P, ctypes.c_float, P, i64, P, sz, P]
            L.vnm_ria_score.restype = ctypes.c_int
            L.vnm_permute_gain_workspace_bytes.argtypes = [GP]
            L.vnm_permute_gain_workspace_bytes.restype = sz
            L.vnm_permute_gain.argtypes = [P, i64, GP, P, i64, P, sz, P]
            L.vnm_permute_gain.restype = ctypes.c_int
            L.vnm_permute_gain_out.argtypes = [P, i64, GP, P, i64, P]
            L.vnm_permute_gain_out.restype = ctypes.c_int
            L.vnm_status_string.argtypes = [ctypes.c_int]
            L.vnm_status_string.restype = ctypes.c_char_p
            L.vnm_launch_count.argtypes = []
            L.vnm_launch_count.restype = ctypes.c_uint64
            _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().vnm_status_string(s).decode()


def launch_count() -> int:
    return int(lib().vnm_launch_count())


def _check(st: int, what: str) -> None:
    if st != VNM_OK:
        raise VnmError(st, what)


def geometry(rows: int, cols: int, V: int, M: int) -> Geom:
    g = Geom()
    _check(lib().vnm_geometry(rows, cols, V, M, ctypes.byref(g)), "vnm_geometry")
    return g


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _as_bits16(t: torch.Tensor) -> torch.Tensor:
    if t.dtype in (torch.bfloat16, torch.int16, torch.uint16):
        return t
    raise TypeError(f"expected bf16 (or its int16 bits), got {t.dtype}")


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("vnm kernels take CUDA tensors (there is no CPU path)")


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("expected a 2-D row-major tensor with unit inner stride")
    return t.stride(0)


@dataclass
class Packed:
    """The compressed V:N:M weight (App. A): A_n = values, A_i1 = col_idx, A_i2 = meta, plus the optional
    tensor-core window form (values_tc / meta_tc, include/vnm.h) used by vnm_spmm for large T."""
    g: Geom
    values: torch.Tensor   # bf16 [rows_p][ld_val]
    col_idx: torch.Tensor  # uint8 [rows_p/V][nb_pad][4]
    meta: torch.Tensor     # int32 (u32 bits) [rows_p][ld_meta]
    values_tc: torch.Tensor | None = None  # bf16 [rows_w * ld_tc]
    meta_tc: torch.Tensor | None = None    # int32 (u32 bits)

    def c(self) -> CPacked:
        return CPacked(self.g, self.values.data_ptr(), self.col_idx.data_ptr(), self.meta.data_ptr(),
                       self.values_tc.data_ptr() if self.values_tc is not None else None,
                       self.meta_tc.data_ptr() if self.meta_tc is not None else None)

    @staticmethod
    def empty(g: Geom, device) -> "Packed":
        return Packed(g,
                      torch.empty((g.rows_p, g.ld_val), dtype=torch.bfloat16, device=device),
                      torch.empty((g.rows_p // g.V, g.nb_pad, 4), dtype=torch.uint8, device=device),
                      torch.empty((g.rows_p, g.ld_meta), dtype=torch.int32, device=device))


def tc_applies(V: int, M: int) -> bool:
    """The tensor-core form exists for this (V, M): window form (M <= 8), natural 2:4 form (M % 4 == 0) or
    window-16 form (8 < M < 16)."""
    return 32 <= V <= 128 and (M <= 8 or M % 4 == 0 or M < 16)


def tc_bytes(g: Geom) -> tuple[int, int]:
    L = lib()
    return int(L.vnm_bytes(ctypes.byref(g), 4)), int(L.vnm_bytes(ctypes.byref(g), 5))


def pack_tc(P: Packed) -> Packed:
    """Fill the tensor-core form of P (allocating it on P's device): the window form for 4 <= M <= 8, the
    natural 2:4 form for M % 4 == 0, the window-16 form for the other M < 16 (include/vnm.h); 32 <= V <= 128 only."""
    _require_cuda(P.values)
    nv, nm = tc_bytes(P.g)
    if nv == 0:
        raise VnmError(VNM_ERR_UNSUPPORTED, "vnm_pack_tc")
    if P.values_tc is None or P.values_tc.numel() * 2 < nv:
        P.values_tc = torch.empty(nv // 2, dtype=torch.bfloat16, device=P.values.device)
    if P.meta_tc is None or P.meta_tc.numel() * 4 < nm:
        P.meta_tc = torch.empty(nm // 4, dtype=torch.int32, device=P.values.device)
    cp = P.c()
    _check(lib().vnm_pack_tc(ctypes.byref(cp), _stream(P.values.device)), "vnm_pack_tc")
    return P


def prune(W: torch.Tensor, V: int, M: int, score: torch.Tensor | None = None) -> torch.Tensor:
    """S_{V:N:M}(score or |W|) -> mask bits, int32 (u32 bits) [rows_p][ld_mask]."""
    W = _as_bits16(W)
    _require_cuda(W, score)
    g = geometry(W.shape[0], W.shape[1], V, M)
    mask = torch.empty((g.rows_p, g.ld_mask), dtype=torch.int32, device=W.device)
    _check(lib().vnm_prune(_ptr(W), _ld(W), _ptr(score), _ld(score) if score is not None else 0, ctypes.byref(g),
                           _ptr(mask), _stream(W.device)), "vnm_prune")
    return mask


def compress(W: torch.Tensor, mask: torch.Tensor, V: int, M: int, status: torch.Tensor | None = None) -> Packed:
    """A_n / A_i1 / A_i2 from W and a V:N:M mask.  If `status` (int32[1], CUDA) is given it receives 0 or
    1 + the index of the first invalid block (see include/vnm.h)."""
    W = _as_bits16(W)
    _require_cuda(W, mask, status)
    g = geometry(W.shape[0], W.shape[1], V, M)
    P = Packed.empty(g, W.device)
    cp = P.c()
    _check(lib().vnm_compress(_ptr(W), _ld(W), _ptr(mask), ctypes.byref(g), ctypes.byref(cp), _ptr(status),
                              _stream(W.device)), "vnm_compress")
    return P


def prune_compress(W: torch.Tensor, V: int, M: int, score: torch.Tensor | None = None, want_mask: bool = False,
                   tc: bool = False):
    """Fused S_{V:N:M} + compression in one pass over W.  Returns Packed (and the mask if asked); with tc=True
    the tensor-core form is also filled when it applies (32 <= V <= 128; M <= 8 or M % 4 == 0)."""
    W = _as_bits16(W)
    _require_cuda(W, score)
    g = geometry(W.shape[0], W.shape[1], V, M)
    P = Packed.empty(g, W.device)
    if tc and tc_applies(V, M):
        nv, nm = tc_bytes(g)
        P.values_tc = torch.empty(nv // 2, dtype=torch.bfloat16, device=W.device)
        P.meta_tc = torch.empty(nm // 4, dtype=torch.int32, device=W.device)
    mask = torch.empty((g.rows_p, g.ld_mask), dtype=torch.int32, device=W.device) if want_mask else None
    cp = P.c()
    _check(lib().vnm_prune_compress(_ptr(W), _ld(W), _ptr(score), _ld(score) if score is not None else 0,
                                    ctypes.byref(g), ctypes.byref(cp), _ptr(mask), _stream(W.device)),
           "vnm_prune_compress")
    return (P, mask) if want_mask else P


def prune_compress_batched(Ws: list, V: int, M: int, scores: list | None = None, want_mask: bool = False,
                           tc: bool = False):
    """vnm_prune_compress_batched: prune + compress several weights of one (V, M) in one launch (byte-identical
    to one prune_compress per weight).  Returns the list of Packed (and the list of masks if asked)."""
    n = len(Ws)
    Ws = [_as_bits16(W) for W in Ws]
    scores = scores if scores is not None else [None] * n
    _require_cuda(*Ws, *scores)
    Ps, masks, cps = [], [], []
    for W in Ws:
        g = geometry(W.shape[0], W.shape[1], V, M)
        P = Packed.empty(g, W.device)
        if tc and tc_applies(V, M):
            nv, nm = tc_bytes(g)
            P.values_tc = torch.empty(nv // 2, dtype=torch.bfloat16, device=W.device)
            P.meta_tc = torch.empty(nm // 4, dtype=torch.int32, device=W.device)
        Ps.append(P)
        masks.append(torch.empty((g.rows_p, g.ld_mask), dtype=torch.int32, device=W.device) if want_mask else None)
        cps.append(P.c())
    arr = lambda ty, xs: (ty * n)(*xs)
    pw = arr(ctypes.c_void_p, [_ptr(W) for W in Ws])
    lw = arr(ctypes.c_int64, [_ld(W) for W in Ws])
    ps = arr(ctypes.c_void_p, [_ptr(s) for s in scores])
    ls = arr(ctypes.c_int64, [_ld(s) if s is not None else 0 for s in scores])
    po = arr(ctypes.c_void_p, [ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps])
    pm = arr(ctypes.c_void_p, [_ptr(m) for m in masks])
    _check(lib().vnm_prune_compress_batched(n, pw, lw, ps, ls, po, pm, _stream(Ws[0].device)),
           "vnm_prune_compress_batched")
    return (Ps, masks) if want_mask else Ps


def spmm(XT: torch.Tensor, P: Packed, T: int | None = None, out: torch.Tensor | None = None,
         out_dtype: torch.dtype = torch.float32, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Y^T = W' X^T on the sparse tensor cores.  XT: bf16 [cols][ldx] (feature-major, tokens contiguous).
    Returns Y^T [rows][T] (fp32 or bf16), or writes into `out` ([rows][ldy], ldy >= T)."""
    XT = _as_bits16(XT)
    _require_cuda(XT, out, workspace)
    T = XT.shape[1] if T is None else T
    g = P.g
    _ld(XT)
    if XT.shape[0] != g.cols:
        raise ValueError(f"XT has {XT.shape[0]} rows, the packed weight has {g.cols} input channels")
    if not 0 <= T <= XT.shape[1]:
        raise ValueError(f"T = {T} outside [0, {XT.shape[1]}] (the columns of XT)")
    if out is not None:
        # the kernels write rows [0, g.rows) x tokens [0, T) through out.stride(0): check the extent here
        _ld(out)
        if out.shape[0] < g.rows or out.shape[1] < T:
            raise ValueError(f"out is {tuple(out.shape)}, needs at least ({g.rows}, {T})")
        if out.device != XT.device:
            raise ValueError("out and XT must be on the same device")
    if workspace is not None and workspace.device != XT.device:
        raise ValueError("workspace and XT must be on the same device")
    if out is None:
        ldy = (T + 7) // 8 * 8
        out = torch.empty((g.rows, ldy), dtype=out_dtype, device=XT.device)[:, :T] if ldy != T else \
            torch.empty((g.rows, T), dtype=out_dtype, device=XT.device)
    ydt = VNM_BF16 if out.dtype == torch.bfloat16 else VNM_F32
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError("Y^T must be fp32 or bf16")
    cp = P.c()
    if workspace is None:  # split-K scratch for the small-T plan (the library allocates no device memory)
        nws = spmm_workspace_bytes(g, T)
        if nws:
            workspace = spmm_workspace(g, T, XT.device)
    ws_ptr, ws_bytes = (_ptr(workspace), workspace.numel() * workspace.element_size()) if workspace is not None \
        else (None, 0)
    _check(lib().vnm_spmm(_ptr(XT), XT.stride(0), T, ctypes.byref(cp), _ptr(out), out.stride(0), ydt, ws_ptr,
                          ws_bytes, _stream(XT.device)), "vnm_spmm")
    return out


VNM_SPMM_WEIGHTS_READY = 1


def spmm_batched(XTs: list, Ps: list, T: int, outs: list | None = None, out_dtype: torch.dtype = torch.float32,
                 workspace: torch.Tensor | None = None, weights_ready: bool = False) -> list:
    """vnm_spmm_batched: Y_i^T = W'_i X_i^T for independent problems sharing T (up to 4 small-T problems per
    launch).  XTs[i]: bf16 [cols_i][ldx_i]; returns the list of Y_i^T (or writes into outs[i]).  weights_ready:
    VNM_SPMM_WEIGHTS_READY (the packed weights were written before the previous kernel on the stream began)."""
    n = len(Ps)
    if len(XTs) != n or (outs is not None and len(outs) != n):
        raise ValueError("XTs, Ps (and outs) must have the same length")
    XTs = [_as_bits16(X) for X in XTs]
    _require_cuda(*XTs, *(outs or []), workspace)
    dev = XTs[0].device
    if outs is None:
        ldy = (T + 7) // 8 * 8
        outs = [torch.empty((P.g.rows, ldy), dtype=out_dtype, device=dev)[:, :T] for P in Ps]
    for X, P, Y in zip(XTs, Ps, outs):
        _ld(X)
        _ld(Y)
        if X.shape[0] != P.g.cols or not 0 <= T <= X.shape[1]:
            raise ValueError(f"XT {tuple(X.shape)} does not fit the weight ({P.g.cols} channels) and T = {T}")
        if Y.shape[0] < P.g.rows or Y.shape[1] < T:
            raise ValueError(f"out is {tuple(Y.shape)}, needs at least ({P.g.rows}, {T})")
        if X.device != dev or Y.device != dev:
            raise ValueError("every XT / out must be on the same device")
        if Y.dtype != outs[0].dtype or Y.dtype not in (torch.bfloat16, torch.float32):
            raise TypeError("Y^T must be fp32 or bf16, the same for every problem")
    if workspace is None:
        workspace = spmm_batched_workspace([P.g for P in Ps], T, dev)
    ws_ptr, ws_bytes = (_ptr(workspace), workspace.numel() * workspace.element_size()) if workspace is not None \
        else (None, 0)
    cps = [P.c() for P in Ps]
    arr = lambda ty, xs: (ty * n)(*xs)
    ydt = VNM_BF16 if outs[0].dtype == torch.bfloat16 else VNM_F32
    _check(lib().vnm_spmm_batched(n, arr(ctypes.c_void_p, [_ptr(X) for X in XTs]),
                                  arr(ctypes.c_int64, [X.stride(0) for X in XTs]), T,
                                  arr(ctypes.c_void_p, [ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps]),
                                  arr(ctypes.c_void_p, [_ptr(Y) for Y in outs]),
                                  arr(ctypes.c_int64, [Y.stride(0) for Y in outs]), ydt,
                                  VNM_SPMM_WEIGHTS_READY if weights_ready else 0, ws_ptr, ws_bytes,
                                  _stream(dev)), "vnm_spmm_batched")
    return outs


def spmm_batched_workspace_bytes(gs: list, T: int) -> int:
    n = len(gs)
    arr = (ctypes.c_void_p * n)(*[ctypes.cast(ctypes.pointer(g), ctypes.c_void_p) for g in gs])
    return int(lib().vnm_spmm_batched_workspace_bytes(n, arr, T))


def spmm_batched_workspace(gs: list, T: int, device) -> torch.Tensor | None:
    """An initialised workspace for vnm_spmm_batched over geometries gs at T (None if not used)."""
    nws = spmm_batched_workspace_bytes(gs, T)
    if not nws:
        return None
    ws = torch.empty(max(nws, 16) // 4, dtype=torch.float32, device=device)
    _check(lib().vnm_spmm_workspace_init(_ptr(ws), ws.numel() * 4, _stream(device)), "vnm_spmm_workspace_init")
    return ws


def spmm_workspace_bytes(g: Geom, T: int) -> int:
    return int(lib().vnm_spmm_workspace_bytes(ctypes.byref(g), T))


def spmm_workspace(g: Geom, T: int, device) -> torch.Tensor | None:
    """A vnm_spmm workspace for (g, T), initialised with vnm_spmm_workspace_init (zero flags; every vnm_spmm
    call leaves it initialised, so it can be reused by later calls on the same stream).  None if not used."""
    nws = spmm_workspace_bytes(g, T)
    if not nws:
        return None
    ws = torch.empty(max(nws, 16) // 4, dtype=torch.float32, device=device)
    _check(lib().vnm_spmm_workspace_init(_ptr(ws), ws.numel() * 4, _stream(device)), "vnm_spmm_workspace_init")
    return ws


def act_norms(XT: torch.Tensor, T: int | None = None) -> torch.Tensor:
    """||X_j||_2 over the tokens of every input channel (Eq. 1).  XT bf16 [cols][ldx]."""
    XT = _as_bits16(XT)
    _require_cuda(XT)
    T = XT.shape[1] if T is None else T
    out = torch.empty(XT.shape[0], dtype=torch.float32, device=XT.device)
    _check(lib().vnm_act_norms(_ptr(XT), XT.stride(0), XT.shape[0], T, _ptr(out), _stream(XT.device)), "vnm_act_norms")
    return out


def ria_score(W: torch.Tensor, act: torch.Tensor | None = None, a: float = 0.5) -> torch.Tensor:
    """RIA importance, Eq. (1), fp32 [rows][cols]; pass it as `score` to
    prune / prune_compress.  act: fp32 [cols] activation norms (act_norms) or None (factor 1)."""
    W = _as_bits16(W)
    _require_cuda(W, act)
    rows, cols = W.shape
    lds = (cols + 3) // 4 * 4
    score = torch.empty((rows, lds), dtype=torch.float32, device=W.device)[:, :cols]
    nws = int(lib().vnm_ria_workspace_bytes(rows, cols))
    ws = torch.empty(max(nws, 16) // 4 + 4, dtype=torch.float32, device=W.device)
    _check(lib().vnm_ria_score(_ptr(W), _ld(W), rows, cols, _ptr(act), float(a), _ptr(score), score.stride(0),
                               _ptr(ws), ws.numel() * 4, _stream(W.device)), "vnm_ria_score")
    return score


def permute_gain(score: torch.Tensor, V: int, M: int) -> torch.Tensor:
    """LSA cost matrix of the input-channel permutation step (Eq. 7): fp32
    [cols_p][cols_p], cost[j][b*M + s] = retained score channel j contributes in slot s of block b."""
    _require_cuda(score)
    if score.dtype != torch.float32:
        raise TypeError("score must be fp32")
    rows, cols = score.shape
    g = geometry(rows, cols, V, M)
    cost = torch.empty((g.cols_p, g.cols_p), dtype=torch.float32, device=score.device)
    nws = int(lib().vnm_permute_gain_workspace_bytes(ctypes.byref(g)))
    ws = torch.empty(max(nws, 16) // 4 + 4, dtype=torch.float32, device=score.device)
    _check(lib().vnm_permute_gain(_ptr(score), _ld(score), ctypes.byref(g), _ptr(cost), cost.stride(0), _ptr(ws),
                                  ws.numel() * 4, _stream(score.device)), "vnm_permute_gain")
    return cost


def permute_gain_out(score: torch.Tensor, V: int, M: int) -> torch.Tensor:
    """LSA cost matrix of the OUTPUT-channel permutation step (Eq. 8 `eq:admm2`):
    fp32 [rows_p][rows_p], cost[i][g*V + s] = retained score row i contributes in slot s of V-row stripe g."""
    _require_cuda(score)
    if score.dtype != torch.float32:
        raise TypeError("score must be fp32")
    rows, cols = score.shape
    g = geometry(rows, cols, V, M)
    cost = torch.empty((g.rows_p, g.rows_p), dtype=torch.float32, device=score.device)
    _check(lib().vnm_permute_gain_out(_ptr(score), _ld(score), ctypes.byref(g), _ptr(cost), cost.stride(0),
                                      _stream(score.device)), "vnm_permute_gain_out")
    return cost
