"""Multi-GPU partitioning of the V:N:M linear layer; one process per GPU.

Two modes, both from the path's own structure (V-blocks and tokens are independent units):

* output-feature sharding — rank r owns V-blocks [r*S, (r+1)*S), S = ceil((rows_p/V)/G).  Its packed
  shard is a zero-copy row slice of A_n / A_i1 / A_i2; it computes Y^T rows [r*S*V, (r+1)*S*V) and one
  all_gather_into_tensor (NCCL over NVLink/NVSwitch) concatenates the feature-major shards — contiguous
  because Y^T is [rows][T].  The tail rank's shard is padded to S*V rows so every message has the same
  size; padded rows are dropped after the gather.
* token sharding — rank r owns tokens [r*T/G, (r+1)*T/G) of X^T (a column slice) and a full packed
  replica; no collective on the data path.

The per-rank product is `vnm.spmm` (the CUDA kernel); tests on CPU inject the oracle product through
`spmm_fn` to exercise the partitioning logic with the gloo backend.
"""
from __future__ import annotations

import math
import torch
import torch.distributed as dist

from . import vnm


def vblocks_per_rank(rows_p: int, V: int, world: int, align: int = 1) -> int:
    """V-blocks per rank, rounded up to a multiple of `align` (the window form needs 128-row shards)."""
    if not rows_p:
        return 0
    s = math.ceil((rows_p // V) / world)
    return math.ceil(s / align) * align


def shard_packed(P: vnm.Packed, rank: int, world: int) -> tuple[vnm.Packed, int, int]:
    """Rows [r0, r0 + rows_local) of the packed weight as a zero-copy view (A_n / A_i1 / A_i2 and, when
    present, the window form: then shards hold whole 128-row tiles, the unit of its metadata layout).

    Returns (packed shard, r0, padded shard rows S*V)."""
    g = P.g
    V = g.V
    tc = P.values_tc is not None and P.meta_tc is not None
    S = vblocks_per_rank(g.rows_p, V, world, max(1, 128 // V) if tc else 1)
    vb0 = min(rank * S, g.rows_p // V)
    vb1 = min(vb0 + S, g.rows_p // V)
    r0 = vb0 * V
    rows_local = max(0, min(g.rows, vb1 * V) - r0)
    gl = vnm.geometry(rows_local, g.cols, V, g.M)
    sub = vnm.Packed(gl, P.values[r0:r0 + gl.rows_p], P.col_idx[vb0:vb0 + gl.rows_p // V], P.meta[r0:r0 + gl.rows_p])
    if tc and gl.rows_p > 0:
        # include/vnm.h tensor-core form: values_tc [rows_w][ld_tc], meta_tc [rows_w/128][per-tile words]; both
        # strides are taken from the library's own byte counts of the FULL geometry, so the window form (M <= 8)
        # and the natural 2:4 form (M % 4 == 0, laid out over 4-channel groups) slice alike
        nv, nm = vnm.tc_bytes(g)
        rows_w_full = math.ceil(g.rows_p / 128) * 128
        ld_tc = nv // 2 // rows_w_full
        meta_tile = nm // 4 // (rows_w_full // 128)
        rows_w = math.ceil(gl.rows_p / 128) * 128
        sub.values_tc = P.values_tc[r0 * ld_tc:(r0 + rows_w) * ld_tc]
        t0 = r0 // 128
        sub.meta_tc = P.meta_tc[t0 * meta_tile:(t0 + rows_w // 128) * meta_tile]
    return sub, r0, S * V


def spmm_out_sharded(XT: torch.Tensor, P: vnm.Packed, T: int | None = None, group=None,
                     out_dtype: torch.dtype = torch.bfloat16, spmm_fn=None) -> torch.Tensor:
    """Output-feature-sharded SpMM: local shard product + all-gather of Y^T.  P is the FULL packed
    weight (every rank holds it or at least its own rows; only the local rows are read).
    Returns the full Y^T [rows][T] on every rank."""
    spmm_fn = spmm_fn or vnm.spmm
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T = XT.shape[1] if T is None else T
    sub, r0, rows_shard = shard_packed(P, rank, world)
    ldy = (T + 7) // 8 * 8  # the kernel's Y^T leading dimension must be a multiple of 8
    y_local = torch.zeros((rows_shard, ldy), dtype=out_dtype, device=XT.device)
    if sub.g.rows > 0:
        spmm_fn(XT, sub, T=T, out=y_local[:sub.g.rows, :T])
    y_full = torch.empty((world * rows_shard, ldy), dtype=out_dtype, device=XT.device)
    dist.all_gather_into_tensor(y_full, y_local, group=group)
    return y_full[:P.g.rows, :T]


def token_range(T: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range of a rank; chunk starts are multiples of 8 tokens (16-B aligned X^T view)."""
    per = math.ceil(math.ceil(T / world) / 8) * 8
    t0 = min(rank * per, T)
    return t0, min(t0 + per, T)


def spmm_token_sharded(XT: torch.Tensor, P: vnm.Packed, rank: int, world: int,
                       out_dtype: torch.dtype = torch.bfloat16, spmm_fn=None) -> tuple[torch.Tensor, int]:
    """Token-sharded SpMM: this rank's tokens only, no collective.  XT is the full [cols][T] activation
    (or any tensor whose columns are tokens); returns (Y^T for tokens [t0, t1), t0)."""
    spmm_fn = spmm_fn or vnm.spmm
    t0, t1 = token_range(XT.shape[1], rank, world)
    x = XT[:, t0:t1]
    ldy = (t1 - t0 + 7) // 8 * 8
    y = torch.empty((P.g.rows, max(ldy, 8)), dtype=out_dtype, device=XT.device)[:, :t1 - t0]
    if t1 > t0:
        spmm_fn(x, P, T=t1 - t0, out=y)
    return y, t0


def shard_rows_for_prune(rows: int, V: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """Mask/compress pass partitioned by V-stripes (no collective): rows [r0, r1) of W for this rank
    (align: V-blocks per shard rounded to a multiple of it, e.g. 128 / V for window-form shards)."""
    rows_p = math.ceil(rows / V) * V if rows else 0
    S = vblocks_per_rank(rows_p, V, world, align)
    r0 = min(rank * S * V, rows)
    return r0, min(r0 + S * V, rows)


__all__ = ["shard_packed", "spmm_out_sharded", "spmm_token_sharded", "token_range", "shard_rows_for_prune",
           "vblocks_per_rank"]
