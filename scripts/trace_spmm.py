"""Eager SpMM calls (L2 flushed before each) for VNM_SPMM_TRACE runs.  Usage: rows cols M T [V] [tc]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
rows, cols, M, T = map(int, sys.argv[1:5])
V = int(sys.argv[5]) if len(sys.argv) > 5 else 64
tc = len(sys.argv) > 6 and sys.argv[6] == "tc"
P = vnm.prune_compress(to_dev_bf16(synth.weights(rows, cols, seed=1)), V, M, tc=tc)
X = to_dev_bf16(synth.activations_t(cols, T, seed=2))
Y = torch.empty((rows, (T + 7) // 8 * 8), dtype=torch.bfloat16, device="cuda")
ws = vnm.spmm_workspace(P.g, T, "cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
for i in range(4):
    fl.zero_(); rd.sum(); torch.cuda.synchronize()
    print(f"--- call {i}", file=sys.stderr, flush=True)
    vnm.spmm(X, P, T=T, out=Y[:, :T], workspace=ws)
    torch.cuda.synchronize()
