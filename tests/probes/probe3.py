"""Round-1b probe (test-only): CTA-pair MMA rates.  python tests/probe3.py -> gpurun_out/probe3.json"""
import ctypes
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
P, u32 = ctypes.c_void_p, ctypes.c_uint32
L.vnm_probe_bench_mma_pair.argtypes = [P, u32, u32, u32, u32, u32, ctypes.c_int, P]
X = torch.zeros(8192 * 64, dtype=torch.int16, device="cuda")
pairs = torch.cuda.get_device_properties(0).multi_processor_count // 2
cyc = torch.zeros(pairs, dtype=torch.int64, device="cuda")
out = []
iters = 20000
for sparse, n, sbo, kb in [(1, 256, 1024, 0), (1, 256, 640, 0), (1, 256, 1024, 10), (1, 256, 1024, 12), (1, 256, 1024, 16),
                           (1, 128, 1024, 0), (0, 256, 1024, 0), (0, 256, 1024, 8), (1, 256, 1024, 6)]:
    for np_ in (1, pairs):
        st = L.vnm_probe_bench_mma_pair(X.data_ptr(), n, sparse, sbo, iters, kb, np_, cyc.data_ptr())
        c = cyc[:np_].float().mean().item() / iters
        r = dict(sparse=sparse, n=n, sbo=sbo, tma_kb_per_mma=kb, pairs=np_, status=st, cycles_per_mma=round(c, 1))
        print(r, flush=True)
        out.append(r)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "probe3.json"), "w"), indent=1)
