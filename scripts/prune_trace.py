"""VNM_PRUNE_TRACE=1: phase times of CTA 0's first tile of the batched prune pass (Llama decode block weights)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
shapes = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]
Ws = [to_dev_bf16(synth.weights(r, c, seed=r + c + i)) for i, (r, c) in enumerate(shapes)]
for _ in range(3):
    vnm.prune_compress_batched(Ws, 64, 5)
    torch.cuda.synchronize()
