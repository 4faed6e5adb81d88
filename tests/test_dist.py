"""Multi-process (world_size 2, 3, 4 and 8, gloo, CPU) tests of the partitioning layer.

The per-rank product is injected: the oracle's packed fp64 SpMM (O9) stands in for the CUDA kernel,
so shard boundaries, tail padding, the all-gather reassembly and token ranges are checked without a
GPU.  Each rank's rows / tokens are computed by the same row-local arithmetic as the single-process
reference, so the reassembled result must match it exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2410_16135_b200 import dist as vdist
from paper_2410_16135_b200 import synth, vnm


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_packed(W, V, M):
    rows, cols = W.shape
    _, values, col_idx, meta = oracle.prune_pack(W, V, M)
    g = vnm.geometry(rows, cols, V, M)
    return vnm.Packed(g, torch.from_numpy(values.view(np.int16)).view(torch.bfloat16),
                      torch.from_numpy(col_idx), torch.from_numpy(meta.view(np.int32)))


def oracle_spmm(XT, P, T=None, out=None):
    """CPU stand-in for vnm.spmm with the same signature (test only)."""
    T = XT.shape[1] if T is None else T
    x = XT[:, :T].contiguous().view(torch.int16).numpy().view(np.uint16)
    y = oracle.spmm_packed(x, P.values.view(torch.int16).numpy().view(np.uint16), P.col_idx.numpy(),
                           P.meta.numpy().view(np.uint32), P.g.rows, P.g.cols, P.g.V, P.g.M)
    out.copy_(torch.from_numpy(y).to(out.dtype))
    return out


def attach_tc(P):
    """Give P a tensor-core form of the library's sizes (contents irrelevant to the oracle stand-in), so that
    shard_packed takes its whole-128-row-tile path and slices values_tc / meta_tc."""
    nv, nm = vnm.tc_bytes(P.g)
    if nv:
        P.values_tc = torch.zeros(nv // 2, dtype=torch.bfloat16)
        P.meta_tc = torch.zeros(nm // 4, dtype=torch.int32)
    return P


def worker(rank, world, port, rows, cols, V, M, T, q, tc=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.weights(rows, cols, seed=7)
        XT = synth.activations_t(cols, T, seed=8)
        P = host_packed(W, V, M)
        if tc:
            attach_tc(P)
        Xt = torch.from_numpy(XT.view(np.int16)).view(torch.bfloat16)
        y = vdist.spmm_out_sharded(Xt, P, T=T, out_dtype=torch.float32, spmm_fn=oracle_spmm)
        yt, t0 = vdist.spmm_token_sharded(Xt, P, rank, world, out_dtype=torch.float32, spmm_fn=oracle_spmm)
        q.put((rank, y.numpy().copy(), yt.numpy().copy(), t0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,M,T,tc", [(2, 200, 90, 5, 13, False), (3, 300, 64, 8, 9, False),
                                                    (2, 64, 40, 5, 5, False), (3, 130, 33, 7, 16, False),
                                                    (4, 520, 72, 5, 11, False), (8, 1100, 48, 6, 24, False),
                                                    (4, 700, 96, 16, 9, True), (8, 1300, 40, 5, 17, True),
                                                    (2, 300, 64, 12, 8, True)])
def test_out_and_token_sharding(world, rows, cols, M, T, tc):
    """Output-feature shards (+ all-gather) and token shards reassemble the single-process product exactly,
    at world sizes 2-8, ragged row / token tails, and with a tensor-core form present (whole-128-row-tile
    shards; M = 12 / 16 take the natural 2:4 layout)."""
    V = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, rows, cols, V, M, T, q, tc)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = synth.weights(rows, cols, seed=7)
    XT = synth.activations_t(cols, T, seed=8)
    _, values, col_idx, meta = oracle.prune_pack(W, V, M)
    ref = oracle.spmm_packed(XT, values, col_idx, meta, rows, cols, V, M).astype(np.float32)
    for rank, y, yt, t0 in res:
        assert y.shape == ref.shape and np.array_equal(y, ref), f"rank {rank} out-sharded"
        assert np.array_equal(yt, ref[:, t0:t0 + yt.shape[1]]), f"rank {rank} token-sharded"
    # token ranges tile [0, T) exactly once
    covered = sorted((t0, t0 + yt.shape[1]) for _, _, yt, t0 in res)
    assert covered[0][0] == 0 and covered[-1][1] == T
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))


def test_shard_boundaries():
    """172 V-blocks (Llama up-proj at V=64) over 8 ranks: S = 22, the last rank gets 18, shapes line up."""
    rows, cols, V, M = 11008, 64, 64, 5
    g = vnm.geometry(rows, cols, V, M)
    P = vnm.Packed.empty.__func__(g, "cpu") if False else vnm.Packed(
        g, torch.zeros((g.rows_p, g.ld_val), dtype=torch.bfloat16), torch.zeros((g.rows_p // V, g.nb_pad, 4),
                                                                                dtype=torch.uint8),
        torch.zeros((g.rows_p, g.ld_meta), dtype=torch.int32))
    total = 0
    for r in range(8):
        sub, r0, pad_rows = vdist.shard_packed(P, r, 8)
        assert pad_rows == 22 * 64 and r0 == min(r * 22 * 64, rows)
        assert sub.values.shape[0] == sub.g.rows_p and sub.meta.shape[0] == sub.g.rows_p
        assert sub.col_idx.shape[0] == sub.g.rows_p // V
        total += sub.g.rows
    assert total == rows
    assert vdist.shard_rows_for_prune(rows, V, 7, 8) == (7 * 22 * 64, rows)


def tc_layout(g):
    """values_tc row length and metadata words per 128-row tile, written out from the include/vnm.h layout
    text (independently of dist.py): window form bpm = 4 blocks per MMA (8 for M = 4); the natural 2:4 form
    (M % 4 == 0, M > 8) is the M = 4 layout over cols_p / 4 channel groups; the window-16 form (other M < 16) has two
    MMAs per 4 blocks."""
    if g.M > 8 and g.M % 4 == 0:
        groups = g.cols_p // 4
        n_mma = (groups + 7) // 8 * 8 // 8
    elif g.M > 8:
        n_mma = g.nb_pad // 2
    else:
        n_mma = g.nb_pad // (8 if g.M == 4 else 4)
    n_stage = (n_mma + 3) // 4
    return 16 * n_mma, n_stage * 128 * 4


@pytest.mark.parametrize("rows,world,M,cols", [(1152, 2, 5, 384), (11008, 8, 5, 384), (384, 3, 5, 384),
                                               (200, 4, 5, 384), (512, 2, 16, 4096), (11008, 8, 16, 4096),
                                               (700, 3, 12, 200), (1000, 4, 4, 256), (640, 2, 8, 100),
                                               (11008, 8, 13, 4096), (700, 3, 9, 300), (520, 2, 11, 1000)])
def test_window_form_shards_are_whole_tiles(rows, world, M, cols):
    """With the tensor-core form present, output shards hold whole 128-row tiles and their values_tc /
    meta_tc views start at the shard's tile (include/vnm.h layouts, window and natural 2:4 forms alike);
    shards tile the rows exactly."""
    V = 64
    g = vnm.geometry(rows, cols, V, M)
    ld_tc, meta_tile = tc_layout(g)
    n_stage = meta_tile // 512
    rows_w = (g.rows_p + 127) // 128 * 128
    P = vnm.Packed(g, torch.zeros((g.rows_p, g.ld_val), dtype=torch.bfloat16),
                   torch.zeros((g.rows_p // V, g.nb_pad, 4), dtype=torch.uint8),
                   torch.zeros((g.rows_p, g.ld_meta), dtype=torch.int32),
                   torch.zeros(rows_w * ld_tc, dtype=torch.bfloat16),
                   torch.arange(rows_w // 128 * n_stage * 512, dtype=torch.int32))
    assert vnm.tc_bytes(g) == (rows_w * ld_tc * 2, rows_w // 128 * meta_tile * 4)  # the library agrees
    covered = 0
    for r in range(world):
        sub, r0, rows_shard = vdist.shard_packed(P, r, world)
        assert rows_shard % 128 == 0 and r0 % 128 == 0
        if sub.g.rows == 0:
            continue
        assert r0 == covered
        covered += sub.g.rows
        assert sub.meta_tc.numel() == (sub.g.rows_p + 127) // 128 * n_stage * 512
        assert int(sub.meta_tc[0]) == (r0 // 128) * n_stage * 512
        assert sub.values_tc.numel() == (sub.g.rows_p + 127) // 128 * 128 * ld_tc
        assert sub.values_tc.data_ptr() - P.values_tc.data_ptr() == r0 * ld_tc * 2
    assert covered == rows


def prune_worker(rank, world, port, rows, cols, V, M, align, q):
    """Row e3: each rank prunes + compresses only its own V-stripe of W (no collective on the
    data path); the stripes are gathered here only to check them."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.weights(rows, cols, seed=11, kind="outlier")
        r0, r1 = vdist.shard_rows_for_prune(rows, V, rank, world, align)
        part = oracle.prune_pack(np.ascontiguousarray(W[r0:r1]), V, M) if r1 > r0 else None
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, part))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,M,align", [(2, 200, 90, 5, 1), (4, 1100, 64, 8, 2), (8, 700, 40, 5, 2),
                                                     (3, 64, 33, 16, 1), (8, 3000, 24, 7, 1)])
def test_partitioned_prune_compress(world, rows, cols, M, align):
    """The V-stripe-partitioned mask + compression pass: the per-rank packed stripes, concatenated in rank order
    (A_n / A_i2 by rows, A_i1 by V-blocks, masks by rows), are byte-identical to the single-process pass over
    the whole weight; stripes start on V-block boundaries (whole 128-row tiles when align = 128 / V)."""
    V = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=prune_worker, args=(r, world, port, rows, cols, V, M, align, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = synth.weights(rows, cols, seed=11, kind="outlier")
    mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
    g = oracle.geometry(rows, cols, V, M)
    nb_pad = g["nb_pad"]
    got = {"mask": [], "values": [], "col_idx": [], "meta": []}
    expect_r0 = 0
    for r0, r1, part in parts:
        assert r0 == expect_r0 and (r0 == rows or r0 % (V * align) == 0)
        expect_r0 = r1
        if part is None:
            continue
        pm, pv, pc, pmeta = part
        n = r1 - r0
        n_p = -(-n // V) * V
        got["mask"].append(pm[:n_p]); got["values"].append(pv[:n_p]); got["meta"].append(pmeta[:n_p])
        got["col_idx"].append(pc.reshape(-1, nb_pad, 4)[:n_p // V])
    assert expect_r0 == rows
    assert np.array_equal(np.concatenate(got["mask"]), mask)
    assert np.array_equal(np.concatenate(got["values"]), values)
    assert np.array_equal(np.concatenate(got["meta"]), meta)
    assert np.array_equal(np.concatenate(got["col_idx"]).reshape(col_idx.shape), col_idx)
