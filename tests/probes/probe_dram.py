"""Probe (test-only): HBM streaming rate vs TMA box shape for the decode weight pattern.
python tests/probe_dram.py -> gpurun_out/probe_dram.json"""
import ctypes
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
i32, i64 = ctypes.c_int32, ctypes.c_int64
L.vnm_probe_stream_boxes.argtypes = [ctypes.c_void_p, i32, i32, i64, i32, i32, i32, i32, ctypes.c_void_p]
rows, cols = 11008, 1648  # A_n of Llama up at 64:2:5 (36 MB)
A = torch.ones(rows * cols, dtype=torch.int16, device="cuda")
fl = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ns = ctypes.c_ulonglong(0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = []
for bh, bw, st in [(128, 64, 4), (128, 64, 8), (64, 128, 4), (64, 256, 4), (32, 256, 4), (32, 256, 8), (16, 256, 8),
                   (8, 256, 8), (256, 64, 4), (128, 256, 3)]:
    for gm in (1, 2, 4):
        best = None
        for rep in range(3):
            fl.zero_(); rd.sum(); torch.cuda.synchronize()
            st_ = L.vnm_probe_stream_boxes(A.data_ptr(), rows, cols, cols, bh, bw, st, gm * sms, ctypes.byref(ns))
            v = rows * cols * 2 / ns.value
            best = v if best is None or v > best else best
        r = dict(box_h=bh, box_w=bw, stages=st, ctas_per_sm=gm, status=st_, gbs=round(best, 1))
        print(r, flush=True)
        out.append(r)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "probe_dram.json"), "w"), indent=1)
