"""Probe (test-only): TMA streaming of the Llama-up A_n (11008 x 1648 bf16, 36 MB) in the small-T plan's unit
order (contiguous stream-K shares), vs box shape, units in flight and an extra A_i2-like box per unit.
python tests/probes/probe_stream.py -> gpurun_out/probe_stream.json"""
import ctypes
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
i32 = ctypes.c_int32
L.vnm_probe_stream_units.argtypes = [ctypes.c_void_p, i32, i32, i32, i32, i32, i32, ctypes.c_void_p, i32, i32,
                                     i32, i32, ctypes.c_void_p]
rows, cols = 11008, 1664  # A_n of Llama up at 64:2:5 (rounded to 64-value boxes)
A = torch.ones(rows * cols, dtype=torch.int16, device="cuda")
E = torch.ones(rows * 104, dtype=torch.int32, device="cuda")
fl = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ns = ctypes.c_ulonglong(0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = []
cases = [(128, 64, 10, 0, 1, 0), (128, 64, 10, 0, 0, 0), (128, 64, 10, 0, 1, 8), (128, 64, 10, 0, 0, 8),
         (128, 64, 4, 0, 1, 0), (128, 64, 8, 4, 1, 0), (64, 64, 16, 0, 1, 0), (256, 64, 6, 0, 1, 0),
         (128, 128, 6, 0, 0, 0), (128, 256, 3, 0, 0, 0), (64, 256, 6, 0, 0, 0), (32, 256, 12, 0, 0, 0)]
for bh, bw, st, ew, swz, spin in cases:
    for gm in (1, 2):
        if gm == 2 and spin:
            continue
        best = None
        for rep in range(3):
            fl.zero_(); rd.sum(); torch.cuda.synchronize()
            st_ = L.vnm_probe_stream_units(A.data_ptr(), rows, cols, bh, bw, st, gm * sms, E.data_ptr(), 104, ew,
                                           swz, spin, ctypes.byref(ns))
            v = rows * cols * 2 / max(ns.value, 1)
            best = v if best is None or v > best else best
        r = dict(box_h=bh, box_w=bw, stages=st, extra_words=ew, sw128=swz, spin_warps=spin, ctas_per_sm=gm,
                 status=st_, gbs=round(best, 1))
        print(r, flush=True)
        out.append(r)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "probe_stream.json"), "w"), indent=1)
