"""TEST-ONLY probe: the tc3 MMA stage pattern (probes4.cu bench_stage_pair) with tc3's own B-operand geometry — the
ring of S = 5 slots of 88 rows and the chunk stride (LBO) of the whole ring region (5 * 88 * 128 B) — vs the
round-2 probe's (ring 6 x 80 rows, LBO 16 KB).  Prints cycles per pair MMA (N = 224)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
L.vnm_probe_bench_stage_pair_lbo.argtypes = [ctypes.c_uint32] * 6 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                                     ctypes.c_uint32]
sms = torch.cuda.get_device_properties(0).multi_processor_count
for pairs in (74, 70):
    for n, sbo, step, rows, ring, commit, lbo in [(224, 640, 2560, 80, 6, 4, 16384), (224, 640, 2560, 88, 5, 4, 16384),
                                                  (224, 640, 2560, 88, 5, 4, 5 * 88 * 128), (224, 640, 2560, 80, 6, 4, 6 * 80 * 128),
                                                  (224, 640, 2560, 88, 5, 2, 5 * 88 * 128), (256, 640, 2560, 88, 5, 4, 5 * 88 * 128)]:
        cyc = torch.zeros(pairs, dtype=torch.int64, device="cuda")
        st = L.vnm_probe_bench_stage_pair_lbo(n, sbo, step, rows, ring, 2000, commit, pairs, cyc.data_ptr(), lbo)
        c = cyc.float() / (2000 * 4)
        print(f"pairs {pairs} n {n} rows {rows} ring {ring} commit {commit} lbo {lbo}: status {st} cycles/MMA median "
              f"{float(c.median()):.1f} max {float(c.max()):.1f}", flush=True)
