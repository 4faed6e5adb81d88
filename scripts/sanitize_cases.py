"""Small invocations of every kernel / plan for compute-sanitizer runs (memcheck, racecheck, synccheck).
Usage: python scripts/sanitize_cases.py  (plans forced through VNM_TC_PLAN in child processes is avoided here:
shapes are chosen so the default dispatch reaches each plan)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16, to_dev_f32


def check(W, XT, V, M, T, tc, out_dtype=torch.float32):
    mask = oracle.prune(W, V, M)
    Yref, Aref = oracle.gemm_ref(XT, oracle.apply_mask(W, mask, V, M))
    P = vnm.prune_compress(to_dev_bf16(W), V, M, tc=tc)
    Y = vnm.spmm(to_dev_bf16(XT), P, T=T, out_dtype=out_dtype).float().cpu().numpy().astype(np.float64)
    ok = np.all(np.abs(Y - Yref) <= oracle.tolerance(Yref, Aref, y_is_bf16=out_dtype == torch.bfloat16))
    return bool(ok)


cases = [
    # (name, rows, cols, V, M, T, tc)
    ("prune2+smallt 64:2:8 toy", 128, 64, 64, 8, 16, False),
    ("prune+smallt V=16", 96, 200, 16, 7, 9, False),
    ("smallt V=128 M=13", 256, 700, 128, 13, 5, False),
    ("gather plan 64:2:9 T=48", 192, 333, 64, 9, 48, False),
    ("window 1-CTA 64:2:5 T=300", 256, 640, 64, 5, 300, True),
    ("window pairs (tc2) 64:2:5 long K", 512, 4096, 64, 5, 512, True),
    ("tc3 resident pairs 64:2:5", 1536, 384, 64, 5, 8192, True),
    ("natural 2:4 64:2:16", 256, 640, 64, 16, 200, True),
]
allok = True
for name, rows, cols, V, M, T, tc in cases:
    W = synth.weights(rows, cols, seed=rows + cols + M, kind="outlier")
    XT = synth.activations_t(cols, T, seed=T + 1)
    ok = check(W, XT, V, M, T, tc, torch.bfloat16 if T > 64 else torch.float32)
    allok &= ok
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
# batched prune + RIA + permutation gains
Ws = [to_dev_bf16(synth.weights(r, c, seed=r + c)) for r, c in [(256, 384), (128, 200)]]
vnm.prune_compress_batched(Ws, 64, 5, tc=True)
Wd = to_dev_bf16(synth.weights(192, 256, seed=5))
act = vnm.act_norms(to_dev_bf16(synth.activations_t(256, 32, seed=6)))
sc = vnm.ria_score(Wd, act)
vnm.permute_gain(sc.contiguous(), 64, 5)
torch.cuda.synchronize()
print("batched prune / ria / permute_gain: ran", flush=True)
print("ALL OK" if allok else "SOME MISMATCH")
sys.exit(0 if allok else 1)
