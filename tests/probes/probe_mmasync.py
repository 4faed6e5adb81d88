"""Probe (test-only): rate of the legacy warp-level mma.sp m16n8k32 (bf16) on B200."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
L.vnm_probe_mma_sync_sp.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
sink = torch.zeros(1024, device="cuda")
ns = ctypes.c_ulonglong(0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
iters = 20000
for warps in (1, 4, 8, 16):
    st = L.vnm_probe_mma_sync_sp(iters, sms, warps, sink.data_ptr(), ctypes.byref(ns))
    n_mma = sms * warps * iters * 4
    flops = n_mma * 16 * 8 * 16 * 2  # effectual MACs per m16n8k32 sparse = 16 x 8 x 16
    per_sm_cycles = ns.value * 1.965 / (warps * iters * 4)
    print(f"warps/SM {warps:2d}: {ns.value / 1e3:.0f} us, {flops / ns.value / 1e3:.1f} TFLOP/s effectual, "
          f"{per_sm_cycles:.1f} SM-cycles per MMA (status {st})")
