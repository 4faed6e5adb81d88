"""TEST-ONLY probe: cycles per pair MMA of the tc3 stage pattern (probes4.cu bench_stage_pair, commit 4) for short
runs (85 stages = one DeiT-S qkv pair's work) vs long runs (2000 stages), repeated back to back."""
import ctypes, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
L.vnm_probe_bench_stage_pair_lbo.argtypes = [ctypes.c_uint32] * 6 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                                     ctypes.c_uint32]
for rep in range(2):
    for stages in (85, 200, 2000, 85):
        cyc = torch.zeros(70, dtype=torch.int64, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st = L.vnm_probe_bench_stage_pair_lbo(224, 640, 2560, 88, 5, stages, 4, 70, cyc.data_ptr(), 5 * 88 * 128)
        b.record(); torch.cuda.synchronize()
        c = cyc.float() / (stages * 4)
        print(f"stages {stages}: cycles/MMA median {float(c.median()):.1f} max {float(c.max()):.1f}; "
              f"launch {a.elapsed_time(b) * 1e3:.1f} us", flush=True)
