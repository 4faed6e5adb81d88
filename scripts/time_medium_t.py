"""Experiment: a T > 32 product through the small-T kernel by token tiles (vnm_spmm_batched over 32-token views of
one X^T / Y^T, up to 4 per launch) vs vnm_spmm's plan.  Usage: python scripts/time_medium_t.py rows cols V M T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
rows, cols, V, M, T = map(int, sys.argv[1:6])
P = vnm.prune_compress(to_dev_bf16(synth.weights(rows, cols, seed=1)), V, M)
X = to_dev_bf16(synth.activations_t(cols, T, seed=2))
Y = torch.empty((rows, T), dtype=torch.bfloat16, device="cuda")
Y2 = torch.empty((rows, T), dtype=torch.bfloat16, device="cuda")
tt = T // 32
Xs = [X[:, 32 * i:32 * (i + 1)] for i in range(tt)]
Ys = [Y2[:, 32 * i:32 * (i + 1)] for i in range(tt)]
ws = vnm.spmm_batched_workspace([P.g] * 4, 32, "cuda")
def tiled():
    for i in range(0, tt, 4):
        vnm.spmm_batched(Xs[i:i + 4], [P] * len(Xs[i:i + 4]), 32, outs=Ys[i:i + 4], workspace=ws)
base = lambda: vnm.spmm(X, P, T=T, out=Y)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f in [("vnm_spmm plan", base), ("small-T token tiles", tiled)]:
    for _ in range(2):
        f()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    g.replay(); torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"{rows}x{cols} {V}:2:{M} T={T} {name}: {a.elapsed_time(b) / 5 * 1e3:.1f} us", flush=True)
d = (Y.float() - Y2.float()).abs().max().item()
print("max |diff| between the two", d)
