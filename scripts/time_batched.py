"""Timing: the Llama decode trio (q / up / down) as 3 vnm_spmm launches vs one vnm_spmm_batched launch, CUDA-graph
replay after an L2 flush + write-back (cold), and back to back (warm).  Usage: python scripts/time_batched.py [T] [V] [M]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
V = int(sys.argv[2]) if len(sys.argv) > 2 else 64
M = int(sys.argv[3]) if len(sys.argv) > 3 else 5
shapes = [(4096, 4096), (11008, 4096), (4096, 11008)]
Ps = [vnm.prune_compress(to_dev_bf16(synth.weights(r, c, seed=r + c)), V, M) for r, c in shapes]
ldx = (T + 7) // 8 * 8  # leading dimensions padded to 16 bytes (the ABI's alignment rule)
Xs = [to_dev_bf16(synth.activations_t(c, T, seed=c, ld=ldx))[:, :T] for r, c in shapes]
Ys = [torch.empty((r, ldx), dtype=torch.bfloat16, device="cuda")[:, :T] for r, c in shapes]
wss = [vnm.spmm_workspace(P.g, T, "cuda") for P in Ps]
wsb = vnm.spmm_batched_workspace([P.g for P in Ps], T, "cuda")
sep = lambda: [vnm.spmm(X, P, T=T, out=Y, workspace=w) for X, P, Y, w in zip(Xs, Ps, Ys, wss)]
bat = lambda: vnm.spmm_batched(Xs, Ps, T, outs=Ys, workspace=wsb)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f in [("3 launches", sep), ("batched", bat)]:
    for _ in range(3):
        f()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        fl.zero_(); rd.sum()
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    a.record()
    for _ in range(20):
        g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"{V}:2:{M} T={T} {name}: cold median {ts[len(ts) // 2]:.2f} us (min {ts[0]:.2f})  warm {a.elapsed_time(b) / 20 * 1e3:.2f} us")
