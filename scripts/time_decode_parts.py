"""Cold CUDA-graph timing of the Llama decode layers (T = 16, 64:2:5) alone and as the 3-launch sequence, to see
whether the sequence costs more than its parts (inter-launch gaps) — python scripts/time_decode_parts.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

T, V, M = 16, 64, 5
shapes = [(4096, 4096), (11008, 4096), (4096, 11008)]
Ps = [vnm.prune_compress(to_dev_bf16(synth.weights(r, c, seed=r + c)), V, M) for r, c in shapes]
Xs = [to_dev_bf16(synth.activations_t(c, T, seed=c)) for r, c in shapes]
Ys = [torch.empty((r, T), dtype=torch.bfloat16, device="cuda") for r, c in shapes]
wss = [vnm.spmm_workspace(P.g, T, "cuda") for P in Ps]
call = lambda i: vnm.spmm(Xs[i], Ps[i], T=T, out=Ys[i], workspace=wss[i])
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, idx in [("q", [0]), ("up", [1]), ("down", [2]), ("q+up+down", [0, 1, 2]), ("up x3", [1, 1, 1])]:
    f = lambda: [call(i) for i in idx]
    for _ in range(3):
        f()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    ts = []
    for _ in range(15):
        fl.zero_(); rd.sum()
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    res[name] = ts[len(ts) // 2]
    print(f"{name:10s} cold median {res[name]:7.2f} us  (min {ts[0]:.2f})")
print(f"sum of singles {res['q'] + res['up'] + res['down']:.2f} us vs the sequence {res['q+up+down']:.2f} us")
