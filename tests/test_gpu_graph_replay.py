"""Replay stress of the decode step as bench.py times it: batched prune + compress of the Llama q / up / down
weights, then the three small-T SpMMs (T = 16, stream-K workspace), captured once in a CUDA graph and replayed
back to back (PDL between the SpMMs).  Y must stay bit-identical to the eager result on every check.

Regression: with a slot ring whose size S was not a multiple of the consumer phase count, use j + 2 of a slot
could be read by a warp that never waited on use j + 1, whose parity wait then passed while use j + 1's TMA was
in flight (a parity wait cannot tell phase j from j + 2): rare wrong data, then an illegal-instruction trap on
the producer's next arrive or a hang.  It showed within ~3000 replays at V:2:8 / 64:2:5."""
import ctypes

import pytest
import torch

from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu

SHAPES = [(4096, 4096), (11008, 4096), (4096, 11008)]


@pytest.mark.parametrize("V,M,T,batched", [(64, 5, 16, False), (64, 8, 16, False), (128, 8, 16, False),
                                           (128, 13, 32, False), (64, 5, 16, True), (128, 13, 32, True)])
def test_decode_step_graph_replays_stay_bit_identical(V, M, T, batched):
    """(128:2:13 at T = 32: only 3 ring slots fit, so 3 of the 4 consumer phases take units.)  batched: the three
    SpMMs as one vnm_spmm_batched launch (one workspace)."""
    replays, every = 2000, 250
    Ws = [to_dev_bf16(synth.weights(r, c, seed=r + c, kind="outlier")) for r, c in SHAPES]
    Xs = [to_dev_bf16(synth.activations_t(c, T, seed=c)) for r, c in SHAPES]
    Ps = vnm.prune_compress_batched(Ws, V, M)
    Ys = [torch.empty((r, T), dtype=torch.bfloat16, device="cuda") for r, _ in SHAPES]
    wss = [vnm.spmm_workspace(P.g, T, "cuda") for P in Ps]
    wsb = vnm.spmm_batched_workspace([P.g for P in Ps], T, "cuda")

    def spmms():
        if batched:
            vnm.spmm_batched(Xs, Ps, T, outs=Ys, workspace=wsb)
        else:
            for X, P, Y, ws in zip(Xs, Ps, Ys, wss):
                vnm.spmm(X, P, T=T, out=Y, workspace=ws)
    spmms()
    torch.cuda.synchronize()
    ref = [Y.clone() for Y in Ys]

    n = len(Ps)
    cps = [P.c() for P in Ps]  # the raw ABI call re-prunes into the same Packed buffers on every replay
    b_w = (ctypes.c_void_p * n)(*[W.data_ptr() for W in Ws])
    b_lw = (ctypes.c_int64 * n)(*[W.stride(0) for W in Ws])
    b_po = (ctypes.c_void_p * n)(*[ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = vnm.lib().vnm_prune_compress_batched(n, b_w, b_lw, None, None, b_po, None,
                                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == 0
        spmms()
    bad = []
    for i in range(replays):
        g.replay()
        if i % every == every - 1:
            torch.cuda.synchronize()
            bad += [(i, k) for k, (Y, R) in enumerate(zip(Ys, ref))
                    if not torch.equal(Y.view(torch.int16), R.view(torch.int16))]
    torch.cuda.synchronize()
    assert not bad, bad
