"""Probe (test-only): back-to-back tcgen05.mma(.sp) rate, converged-warp issue, A from shared memory (SS) vs
TMEM (TS), single CTAs (M = 128) and CTA pairs (M = 256).  python tests/probes/probe4.py"""
import ctypes
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
L.vnm_probe_bench_mma4.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                   ctypes.c_int, ctypes.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
iters = 4000
res = []
for cg in (1, 2):
    units = sms // cg
    for sparse in (1, 0):
        for ts in (0, 1):
            for n in (64, 128, 192, 224, 256):
                cyc = torch.zeros(units, dtype=torch.int64, device="cuda")
                st = L.vnm_probe_bench_mma4(cg, n, ts, sparse, iters, units, cyc.data_ptr())
                c = cyc.float() / iters
                r = dict(cg=cg, sparse=sparse, a="tmem" if ts else "smem", n=n, status=st,
                         cyc_med=round(float(c.median()), 1), cyc_max=round(float(c.max()), 1))
                res.append(r)
                print(r, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "probe4_mma.json"), "w"), indent=1)

# ---- the tc3 stage pattern (4 MMAs + commit per stage, window SBO, ring of B slots)
L.vnm_probe_bench_stage_pair.argtypes = [ctypes.c_uint32] * 6 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
pairs = sms // 2
res2 = []
for n, sbo, step, rows, ring, commit in [(224, 640, 2560, 80, 6, 4), (224, 640, 2560, 80, 6, 5)]:
    cyc = torch.zeros(pairs, dtype=torch.int64, device="cuda")
    st = L.vnm_probe_bench_stage_pair(n, sbo, step, rows, ring, 2000, commit, pairs, cyc.data_ptr())
    c = cyc.float() / (2000 * 4)
    r = dict(n=n, sbo=sbo, b_step=step, stage_rows=rows, ring=ring, commit=commit, status=st,
             cyc_per_mma_med=round(float(c.median()), 1), cyc_per_mma_max=round(float(c.max()), 1))
    res2.append(r)
    print(r, flush=True)
json.dump(res + res2, open(os.path.join(ROOT, "gpurun_out", "probe4_mma.json"), "w"), indent=1)
