"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no pruning, packing or products): it only draws
random weights / activations / scores with the shapes and value distributions of the paper's
workloads (DESIGN.md §5 "input recipe") and returns them as host numpy arrays:

  * bf16 tensors are returned as uint16 bit patterns (round-to-nearest-even from fp32);
  * W  [rows][cols]  (out-features x in-features, nn.Linear.weight layout);
  * XT [cols][T]     (feature-major activations: X^T, tokens contiguous).

Seeds follow SURVEY.md §8(d): seed = 1000*cfg + role (role 0 = W, 1 = X, 2 = score).
"""
from __future__ import annotations

import numpy as np


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bits (finite inputs)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def weights(rows: int, cols: int, seed: int, kind: str = "normal") -> np.ndarray:
    """Weight matrix W as bf16 bits.

    kind:
      normal   N(0, 0.02^2)  (trained-Transformer scale)
      outlier  N(0, 0.02^2) with 1% of input channels scaled x10 (non-uniform column L1, like LLMs)
      int      integers in {-3..3} (exact sums: isolates the tie rules; tie-heavy)
      wide     sign * 2^U(-24, 4) * U(1, 2)  (wide exponent range: exercises the summation order)
      ones     all ones (every L1 ties)
    """
    g = rng(seed)
    if kind == "normal":
        w = g.standard_normal((rows, cols), dtype=np.float32) * np.float32(0.02)
    elif kind == "outlier":
        w = g.standard_normal((rows, cols), dtype=np.float32) * np.float32(0.02)
        n_out = max(1, cols // 100)
        ch = g.choice(cols, size=n_out, replace=False)
        w[:, ch] *= np.float32(10.0)
    elif kind == "int":
        w = g.integers(-3, 4, size=(rows, cols)).astype(np.float32)
    elif kind == "wide":
        e = g.uniform(-24.0, 4.0, size=(rows, cols))
        m = g.uniform(1.0, 2.0, size=(rows, cols))
        s = np.where(g.random((rows, cols)) < 0.5, -1.0, 1.0)
        w = (s * m * np.exp2(np.floor(e))).astype(np.float32)
    elif kind == "ones":
        w = np.ones((rows, cols), dtype=np.float32)
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(w)


def activations_t(cols: int, T: int, seed: int, kind: str = "normal", ld: int | None = None) -> np.ndarray:
    """X^T as bf16 bits [cols][ld] (ld >= T, tokens contiguous); entries N(0,1) (or ints / ones)."""
    g = rng(seed)
    ld = T if ld is None else ld
    if kind == "normal":
        x = g.standard_normal((cols, ld), dtype=np.float32)
    elif kind == "int":
        x = g.integers(-4, 5, size=(cols, ld)).astype(np.float32)
    elif kind == "ones":
        x = np.ones((cols, ld), dtype=np.float32)
    else:
        raise ValueError(kind)
    if ld > T:
        x[:, T:] = 0.0
    return f32_to_bf16_bits(x)


def scores(rows: int, cols: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """An fp32 importance-score matrix (stand-in for RIA, Eq. (1); the path accepts any score).

    kind: uniform U[0,1) ; signed N(0,1) (|s| is taken) ; int integers 0..4 (ties)."""
    g = rng(seed)
    if kind == "uniform":
        return g.random((rows, cols), dtype=np.float32)
    if kind == "signed":
        return g.standard_normal((rows, cols), dtype=np.float32)
    if kind == "int":
        return g.integers(0, 5, size=(rows, cols)).astype(np.float32)
    raise ValueError(kind)


def seed(cfg: int, role: int) -> int:
    return 1000 * cfg + role
