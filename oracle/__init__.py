"""CPU oracle for the V:N:M sparse linear layer (arXiv 2410.16135).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_2410_16135_b200`` never imports it, and the oracle shares no code with ``csrc/``.

The arithmetic lives in ``vnm_oracle.c`` (plain C, fp32 for the mask decisions in the canonical
stride-halving tree order of DESIGN.md reading Q3, fp64 for Y).  This module only marshals numpy
arrays through ctypes.  Every function cites the passage it follows (P:n = PAPER.md line n,
S:n = SPEC.md line n); the steps O1..O9 are those of DESIGN.md §3.

Parity pins (tests/test_oracle_*.py): brute force over C(M,4) x C(4,2) with exact rational sums,
SPEC worked examples, SparseMask invariants, density 2/M, 64:2:4 == textbook 2:4, exact sums on
integer weights, pack/unpack round trip, identity-X, fp64 GEMM vs exact rational products.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vnm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("rows", "cols", "V", "M", "rows_p", "cols_p", "nb", "nb_pad", "ld_val", "ld_meta", "ld_mask")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64 = ctypes.c_int32, ctypes.c_int64
            L.vnmo_geometry.argtypes = [i32, i32, i32, i32, ctypes.POINTER(Geom)]
            L.vnmo_prune.argtypes = [P, i64, P, i64, i32, i32, i32, i32, P, P, P]
            L.vnmo_pack.argtypes = [P, i64, P, i32, i32, i32, i32, P, P, P]
            L.vnmo_unpack.argtypes = [P, P, P, i32, i32, i32, i32, P]
            L.vnmo_gemm_ref.argtypes = [P, i64, i32, P, i64, i32, i32, P, P]
            L.vnmo_gemm_ref_sampled.argtypes = [P, i64, P, i64, i32, P, P, i64, P, P]
            L.vnmo_spmm_packed.argtypes = [P, i64, i32, P, P, P, i32, i32, i32, i32, P]
            L.vnmo_apply_mask.argtypes = [P, i64, P, i32, i32, i32, i32, P]
            L.vnmo_retained_score.argtypes = [P, i64, P, i32, i32, i32, i32]
            L.vnmo_retained_score.restype = ctypes.c_double
            L.vnmo_act_norms.argtypes = [P, i64, i32, i32, P]
            L.vnmo_ria.argtypes = [P, i64, i32, i32, P, ctypes.c_double, P, i64, P]
            L.vnmo_permute_gain.argtypes = [P, i64, i32, i32, i32, i32, P]
            L.vnmo_permute_gain_out.argtypes = [P, i64, i32, i32, i32, i32, P]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    """OpenMP thread count for the oracle (bench cpu_baseline)."""
    os.environ["OMP_NUM_THREADS"] = str(n)


def geometry(rows: int, cols: int, V: int, M: int) -> dict:
    """Padded geometry (§3 "Acceleration": pad inputs to a multiple of M, outputs of V)."""
    g = Geom()
    st = lib().vnmo_geometry(rows, cols, V, M, ctypes.byref(g))
    if st:
        raise ValueError(f"vnmo_geometry status {st}")
    return g.as_dict()


def prune(W: np.ndarray, V: int, M: int, score: np.ndarray | None = None, want_decisions: bool = False):
    """S_{V:N:M} (§3), steps O1-O5.  W: uint16 bf16 bits [rows][cols]; score: float32 or None (ABS).

    Returns mask uint32 [rows_p][ld_mask]; with want_decisions also kept [rows_p/V][nb][4] and
    pos [rows_p][nb][2]."""
    W = np.ascontiguousarray(W, dtype=np.uint16)
    rows, cols = W.shape
    g = geometry(rows, cols, V, M)
    if score is not None:
        score = np.ascontiguousarray(score, dtype=np.float32)
        assert score.shape == W.shape
    mask = np.zeros((g["rows_p"], g["ld_mask"]), dtype=np.uint32)
    kept = np.zeros((g["rows_p"] // V, g["nb"], 4), dtype=np.uint8) if want_decisions else None
    pos = np.zeros((g["rows_p"], g["nb"], 2), dtype=np.uint8) if want_decisions else None
    st = lib().vnmo_prune(_p(W), cols, _p(score), cols, rows, cols, V, M, _p(mask), _p(kept), _p(pos))
    if st:
        raise ValueError(f"vnmo_prune status {st}")
    return (mask, kept, pos) if want_decisions else mask


def pack(W: np.ndarray, mask: np.ndarray, V: int, M: int):
    """A_n / A_i1 / A_i2 (App. A), step O6.  Returns (status, values, col_idx, meta)."""
    W = np.ascontiguousarray(W, dtype=np.uint16)
    rows, cols = W.shape
    g = geometry(rows, cols, V, M)
    mask = np.ascontiguousarray(mask, dtype=np.uint32)
    assert mask.shape == (g["rows_p"], g["ld_mask"])
    values = np.zeros((g["rows_p"], g["ld_val"]), dtype=np.uint16)
    col_idx = np.zeros((g["rows_p"] // V, g["nb_pad"], 4), dtype=np.uint8)
    meta = np.zeros((g["rows_p"], g["ld_meta"]), dtype=np.uint32)
    st = lib().vnmo_pack(_p(W), cols, _p(mask), rows, cols, V, M, _p(values), _p(col_idx), _p(meta))
    return st, values, col_idx, meta


def prune_pack(W, V, M, score=None):
    mask = prune(W, V, M, score)
    st, values, col_idx, meta = pack(W, mask, V, M)
    if st:
        raise AssertionError(f"oracle produced an invalid mask (pack status {st})")
    return mask, values, col_idx, meta


def unpack(values, col_idx, meta, rows, cols, V, M):
    """Inverse of pack (App. A), step O7.  Returns bf16 bits [rows_p][cols_p]."""
    g = geometry(rows, cols, V, M)
    out = np.zeros((g["rows_p"], g["cols_p"]), dtype=np.uint16)
    st = lib().vnmo_unpack(_p(np.ascontiguousarray(values)), _p(np.ascontiguousarray(col_idx)),
                           _p(np.ascontiguousarray(meta)), rows, cols, V, M, _p(out))
    if st:
        raise ValueError(f"vnmo_unpack status {st}")
    return out


def apply_mask(W, mask, V, M):
    """W' = W (.) M, bf16 bits [rows][cols]."""
    W = np.ascontiguousarray(W, dtype=np.uint16)
    rows, cols = W.shape
    out = np.zeros((rows, cols), dtype=np.uint16)
    st = lib().vnmo_apply_mask(_p(W), cols, _p(np.ascontiguousarray(mask)), rows, cols, V, M, _p(out))
    if st:
        raise ValueError(st)
    return out


def gemm_ref(XT: np.ndarray, Wm: np.ndarray, want_abs: bool = True):
    """Step O8: Y^T = W' X^T in fp64.  XT bf16 bits [cols][T]; Wm bf16 bits [rows][cols].
    Returns (YT, AT) fp64 [rows][T], AT = sum_k |x w'| for the tolerance of BASELINE.json."""
    XT = np.ascontiguousarray(XT, dtype=np.uint16)
    Wm = np.ascontiguousarray(Wm, dtype=np.uint16)
    cols, T = XT.shape
    rows = Wm.shape[0]
    assert Wm.shape[1] >= cols
    YT = np.zeros((rows, T), dtype=np.float64)
    AT = np.zeros((rows, T), dtype=np.float64) if want_abs else None
    lib().vnmo_gemm_ref(_p(XT), T, T, _p(Wm), Wm.shape[1], rows, cols, _p(YT), _p(AT))
    return YT, AT


def gemm_ref_sampled(XT, Wm, o_idx, t_idx):
    """Step O8 at sampled outputs (o_i, t_i)."""
    XT = np.ascontiguousarray(XT, dtype=np.uint16)
    Wm = np.ascontiguousarray(Wm, dtype=np.uint16)
    o_idx = np.ascontiguousarray(o_idx, dtype=np.int32)
    t_idx = np.ascontiguousarray(t_idx, dtype=np.int32)
    n = len(o_idx)
    Y = np.zeros(n, dtype=np.float64)
    A = np.zeros(n, dtype=np.float64)
    lib().vnmo_gemm_ref_sampled(_p(XT), XT.shape[1], _p(Wm), Wm.shape[1], XT.shape[0],
                                _p(o_idx), _p(t_idx), n, _p(Y), _p(A))
    return Y, A


def spmm_packed(XT, values, col_idx, meta, rows, cols, V, M):
    """Step O9: Y^T from the packed arrays only, gathering x rows (App. A)."""
    XT = np.ascontiguousarray(XT, dtype=np.uint16)
    T = XT.shape[1]
    YT = np.zeros((rows, T), dtype=np.float64)
    st = lib().vnmo_spmm_packed(_p(XT), T, T, _p(np.ascontiguousarray(values)),
                                _p(np.ascontiguousarray(col_idx)), _p(np.ascontiguousarray(meta)),
                                rows, cols, V, M, _p(YT))
    if st:
        raise ValueError(st)
    return YT


def retained_score(score, mask, V, M):
    """Sum of scores over mask positions."""
    score = np.ascontiguousarray(score, dtype=np.float32)
    rows, cols = score.shape
    return lib().vnmo_retained_score(_p(score), cols, _p(np.ascontiguousarray(mask)), rows, cols, V, M)


def tolerance(YT_ref: np.ndarray, AT_ref: np.ndarray, y_is_bf16: bool = False) -> np.ndarray:
    """BASELINE.json: |Y - Y_ref| <= 1e-3 * sum|x w| + 1e-6 (fp32 Y).  A bf16 Y adds the RNE
    rounding of the output, 2^-8 |Y_ref| (reading Q14)."""
    tol = 1e-3 * AT_ref + 1e-6
    if y_is_bf16:
        tol = tol + np.abs(YT_ref) * 2.0 ** -8
    return tol


def act_norms(XT: np.ndarray, T: int | None = None) -> np.ndarray:
    """||X_j||_2 over the tokens of every input channel j (Eq. 1; channel reading S:165), fp64.
    XT: bf16 bits [cols][ldx] (feature-major)."""
    XT = np.ascontiguousarray(XT, dtype=np.uint16)
    cols, ldx = XT.shape
    T = ldx if T is None else T
    out = np.zeros(cols, np.float64)
    st = lib().vnmo_act_norms(_p(XT), ldx, cols, T, _p(out))
    if st:
        raise ValueError(f"vnmo_act_norms status {st}")
    return out


def ria(W: np.ndarray, act: np.ndarray | None = None, a: float = 0.5, want_f64: bool = False):
    """RIA importance, Eq. (1): (|W_ij| / sum_r |W_rj| + |W_ij| / sum_c |W_ic|) * act_j^a, fp64 rounded
    to fp32 once; zero sums give a zero fraction; act None = all ones."""
    W = np.ascontiguousarray(W, dtype=np.uint16)
    rows, cols = W.shape
    out = np.zeros((rows, cols), np.float32)
    s64 = np.zeros((rows, cols), np.float64) if want_f64 else None
    actv = None if act is None else np.ascontiguousarray(act, dtype=np.float64)
    st = lib().vnmo_ria(_p(W), cols, rows, cols, _p(actv), float(a), _p(out), cols, _p(s64))
    if st:
        raise ValueError(f"vnmo_ria status {st}")
    return (out, s64) if want_f64 else out


def permute_gain(score: np.ndarray, V: int, M: int) -> np.ndarray:
    """LSA cost of the input-channel permutation step (Eq. 7, Q22):
    cost[j][b*M + s] = retained score channel j contributes in slot s of block b (others frozen), summed over
    the V-row stripes.  score fp32 [rows][cols]; returns fp64 [cols_p][cols_p]."""
    score = np.ascontiguousarray(score, dtype=np.float32)
    rows, cols = score.shape
    g = geometry(rows, cols, V, M)
    K = g["cols_p"]
    cost = np.zeros((K, K), np.float64)
    st = lib().vnmo_permute_gain(_p(score), cols, rows, cols, V, M, _p(cost))
    if st:
        raise ValueError(f"vnmo_permute_gain status {st}")
    return cost


def permute_gain_out(score: np.ndarray, V: int, M: int) -> np.ndarray:
    """LSA cost of the OUTPUT-channel permutation step (Eq. 8 `eq:admm2`; SURVEY NEXT-3;
    DESIGN.md Q23): cost[i][g*V + s] = retained score row i contributes in slot s of V-row stripe g (other rows
    frozen, the stripe re-pruned by S_{V:N:M}).  score fp32 [rows][cols]; returns fp64 [rows_p][rows_p]."""
    score = np.ascontiguousarray(score, dtype=np.float32)
    rows, cols = score.shape
    g = geometry(rows, cols, V, M)
    R = g["rows_p"]
    cost = np.zeros((R, R), np.float64)
    st = lib().vnmo_permute_gain_out(_p(score), cols, rows, cols, V, M, _p(cost))
    if st:
        raise ValueError(f"vnmo_permute_gain_out status {st}")
    return cost
