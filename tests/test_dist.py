"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the partitioning layer.

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


def worker(rank, world, port, rows, cols, V, M, T, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.weights(rows, cols, seed=7)
        XT = synth.activations_t(cols, T, seed=8)
        P = host_packed(W, V, M)
        Xt = torch.from_numpy(XT.view(np.int16)).view(torch.bfloat16)
        y = vdist.spmm_out_sharded(Xt, P, T=T, out_dtype=torch.float32, spmm_fn=oracle_spmm)
        yt, t0 = vdist.spmm_token_sharded(Xt, P, rank, world, out_dtype=torch.float32, spmm_fn=oracle_spmm)
        q.put((rank, y.numpy().copy(), yt.numpy().copy(), t0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,M,T", [(2, 200, 90, 5, 13), (3, 300, 64, 8, 9), (2, 64, 40, 5, 5),
                                                 (3, 130, 33, 7, 16)])
def test_out_and_token_sharding(world, rows, cols, M, T):
    V = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, rows, cols, V, M, T, q)) for r in range(world)]
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


@pytest.mark.parametrize("rows,world", [(1152, 2), (11008, 8), (384, 3), (200, 4)])
def test_window_form_shards_are_whole_tiles(rows, world):
    """With the window form present, output shards hold whole 128-row tiles and their values_tc / meta_tc
    views start at the shard's tile (include/vnm.h layouts); shards tile the rows exactly."""
    V, M, cols = 64, 5, 384
    g = vnm.geometry(rows, cols, V, M)
    n_mma = g.nb_pad // 4
    ld_tc, n_stage = 16 * n_mma, (n_mma + 3) // 4
    rows_w = (g.rows_p + 127) // 128 * 128
    P = vnm.Packed(g, torch.zeros((g.rows_p, g.ld_val), dtype=torch.bfloat16),
                   torch.zeros((g.rows_p // V, g.nb_pad, 4), dtype=torch.uint8),
                   torch.zeros((g.rows_p, g.ld_meta), dtype=torch.int32),
                   torch.arange(rows_w * ld_tc, dtype=torch.int32).to(torch.float32).to(torch.bfloat16),
                   torch.arange(rows_w // 128 * n_stage * 512, dtype=torch.int32))
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
    assert covered == rows
