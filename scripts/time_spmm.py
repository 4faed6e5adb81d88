"""Quick SpMM timing: CUDA-graph replay of N back-to-back vnm_spmm calls (warm L2) and single calls after an
L2 flush (cold).  Usage: python scripts/time_spmm.py rows cols M T [tc]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16

rows, cols, M, T = map(int, sys.argv[1:5])
tc = len(sys.argv) > 5 and sys.argv[5] == "tc"
W = synth.weights(rows, cols, seed=1)
X = synth.activations_t(cols, T, seed=2)
z = os.environ.get("VNM_TS_ZERO", "")  # power probe: zero activations and / or weights
if "x" in z: X = X * 0
if "w" in z: W = W * 0
V = int(os.environ.get("VNM_TS_V", "64"))
P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=tc)
Xd = to_dev_bf16(X)
Y = torch.empty((rows, (T + 7) // 8 * 8), dtype=torch.bfloat16, device="cuda")
ws = vnm.spmm_workspace(P.g, T, "cuda")
f = lambda: vnm.spmm(Xd, P, T=T, out=Y[:, :T], workspace=ws)
for _ in range(3):
    f()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        f()
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
warm = a.elapsed_time(b) / 20 * 1e3
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    f()
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
import time
t_end = time.perf_counter() + 0.5  # clocks up under this load before measuring
while time.perf_counter() < t_end:
    g.replay()
torch.cuda.synchronize()
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
warm = a.elapsed_time(b) / 20 * 1e3
ts = []
for _ in range(10):
    fl.zero_()
    rd.sum()
    a.record(); g1.replay(); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"spmm {rows}x{cols} V={V} M={M} T={T}{' tc' if tc else ''}: warm {warm:.2f} us  cold median {ts[len(ts)//2]:.2f} us")
