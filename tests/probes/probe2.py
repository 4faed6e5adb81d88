"""Round-2 hardware probes on a B200 (test-only):  python tests/probe2.py <mode>

modes: interleave | mma_multi | gather4 | tma_bw | tmem_cp      (one mode per process)
Results go to gpurun_out/probe2_<mode>.json and stdout."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
VALID = [0x4, 0x8, 0xC, 0x9, 0xD, 0xE]


def load():
    L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
    P, u32, i32, i64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64
    L.vnm_probe_interleave.argtypes = [P, P, P, P, u32, u32]
    L.vnm_probe_bench_mma_multi.argtypes = [u32, u32, u32, u32, u32, u32, P]
    L.vnm_probe_gather4.argtypes = [P, i64, i64, u32, P, i32, P]
    L.vnm_probe_bench_tma.argtypes = [P, i64, i64, i32, i32, i32, u32, P]
    L.vnm_probe_tmem_cp.argtypes = [u32, u32, P]
    return L


def bf16(a):
    return torch.tensor(np.asarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).cuda()


def interleave(L):
    out = []
    Bn = np.zeros((32, 64), np.float32)
    for k in range(32):
        Bn[k, k] = 1.0
    B = bf16(Bn)
    A = bf16(np.tile(np.arange(1, 129, dtype=np.float32)[:, None], (1, 16)))
    E = torch.full((128, 4), 0x44444444, dtype=torch.int64).to(torch.int32).cuda()
    cfgs = [(0, 0), (16, 0), (16, 16), (0, 16)]
    if len(sys.argv) > 2:
        cfgs = [cfgs[int(sys.argv[2])]]
    for d_lane, e_lane in cfgs:
        D = torch.zeros(128, 64, dtype=torch.float32, device="cuda")
        st = L.vnm_probe_interleave(A.data_ptr(), B.data_ptr(), E.data_ptr(), D.data_ptr(), d_lane, e_lane)
        torch.cuda.synchronize()
        Dn = D.cpu().numpy()
        lanes = {int(l): sorted(set(Dn[l][Dn[l] != 0].tolist())) for l in range(128) if np.any(Dn[l] != 0)}
        ok = all((Dn[l][:32].reshape(8, 4) != 0).tolist() == [[True, True, False, False]] * 8 for l in lanes)
        out.append({"d_lane": d_lane, "e_lane": e_lane, "status": st, "pattern_ok": ok,
                    "lanes": {str(k): v for k, v in list(lanes.items())}})
        print(d_lane, e_lane, st, ok, list(lanes.items())[:20])
    return out


def mma_multi(L):
    out = []
    nblk = torch.cuda.get_device_properties(0).multi_processor_count
    for (m, n, nacc, mode) in [(64, 256, 1, 0), (64, 128, 1, 0), (64, 128, 2, 0), (64, 128, 4, 0),
                               (64, 64, 1, 0), (64, 64, 4, 0), (128, 256, 1, 0), (128, 128, 2, 0), (128, 128, 1, 0),
                               (64, 16, 4, 0), (64, 32, 4, 0), (64, 16, 1, 0), (64, 256, 2, 0)]:
        cyc = torch.zeros(nblk, dtype=torch.int64, device="cuda")
        iters = 4096
        L.vnm_probe_bench_mma_multi(m, n, 64, nacc, mode, nblk, cyc.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = L.vnm_probe_bench_mma_multi(m, n, iters, nacc, mode, nblk, cyc.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        r = {"M": m, "N": n, "nacc": nacc, "mode": mode, "status": st,
             "cycles_per_mma": float(np.median(cyc.cpu().numpy())) / iters,
             "effectual_tflops": 2.0 * m * n * 16 * iters * nblk / ms / 1e9}
        print(json.dumps(r), flush=True)
        out.append(r)
    return out


def gather4(L):
    rows, cols = 64, 128
    X = (np.arange(rows)[:, None] * 256 + np.arange(cols)[None, :]).astype(np.uint16)
    Xd = torch.from_numpy(X.view(np.int16)).cuda()
    ridx = torch.tensor([5, 17, 2, 60, 33, 8, 41, 0], dtype=torch.int32, device="cuda")
    res = []
    for box_rows in (1, 4):
        for col in (0, 64):
            out = torch.zeros(1024, dtype=torch.uint8, device="cuda")
            st = L.vnm_probe_gather4(Xd.data_ptr(), rows, cols, box_rows, ridx.data_ptr(), col, out.data_ptr())
            torch.cuda.synchronize()
            o = out.cpu().numpy().view(np.uint16)  # 512 uint16 = 8 rows x 64
            # expected with 128B swizzle: row r (0..7) chunk c (16 B = 8 elems) at chunk c ^ r
            exp = np.zeros(512, np.uint16)
            rr = ridx.cpu().numpy()
            for r in range(8):
                for c in range(8):
                    pc = c ^ r
                    exp[r * 64 + pc * 8: r * 64 + pc * 8 + 8] = X[rr[r], col + c * 8: col + c * 8 + 8]
            plain = np.concatenate([X[rr[r], col:col + 64] for r in range(8)])
            r = {"box_rows": box_rows, "col": col, "status": st, "swizzled_match": bool(np.array_equal(o, exp)),
                 "plain_match": bool(np.array_equal(o, plain)), "first_row": o[:64].tolist()}
            print(json.dumps({k: v for k, v in r.items() if k != "first_row"}))
            res.append(r)
    return res


def tma_bw(L):
    res = []
    nblk = torch.cuda.get_device_properties(0).multi_processor_count
    for (rows, cols, label) in [(4096, 2048, "l2_16MB"), (65536, 2048, "hbm_256MB")]:
        X = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
        for gather, lanes in ((1, 1), (1, 8), (1, 32), (0, 1)):
            for ctas in (nblk, 2 * nblk):
                cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
                iters = 512
                L.vnm_probe_bench_tma(X.data_ptr(), rows, cols, 16, gather, lanes, ctas, cyc.data_ptr())
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                st = L.vnm_probe_bench_tma(X.data_ptr(), rows, cols, iters, gather, lanes, ctas, cyc.data_ptr())
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                gbs = ctas * iters * 16384 / ms / 1e6
                r = {"src": label, "gather4": gather, "lanes": lanes, "ctas": ctas, "status": st, "GBps": round(gbs, 1),
                     "bytes_per_cycle_per_sm": round(ctas * iters * 16384 / float(np.median(cyc.cpu().numpy())) / nblk, 2)}
                print(json.dumps(r), flush=True)
                res.append(r)
    return res


def tmem_cp(L):
    res = []
    for lbo, sbo in [(2048, 128), (128, 256), (16, 128), (256, 128)]:
        out = torch.zeros(128 * 4, dtype=torch.int32, device="cuda")
        st = L.vnm_probe_tmem_cp(lbo, sbo, out.data_ptr())
        torch.cuda.synchronize()
        o = out.cpu().numpy().reshape(128, 4)
        ident = np.arange(512).reshape(128, 4)
        r = {"lbo": lbo, "sbo": sbo, "status": st, "identity": bool(np.array_equal(o, ident)),
             "lane0": o[0].tolist(), "lane1": o[1].tolist(), "lane8": o[8].tolist(), "lane16": o[16].tolist(),
             "lane32": o[32].tolist(), "lane127": o[127].tolist()}
        print(json.dumps(r))
        res.append(r)
    return res


def main():
    L = load()
    mode = sys.argv[1]
    r = globals()[mode](L)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = mode + ("_" + sys.argv[2] if len(sys.argv) > 2 else "")
    json.dump(r, open(os.path.join(ROOT, "gpurun_out", f"probe2_{tag}.json"), "w"), indent=1)



def window(L):
    """Overlapping K-group windows: K-group i of the MMA reads dense rows [i*w, i*w + 8)."""
    P, u32 = ctypes.c_void_p, ctypes.c_uint32
    L.vnm_probe_window.argtypes = [P, P, P, P, u32, u32, u32, u32, u32, u32, u32]
    krows = 40
    A = bf16(np.tile(2.0 ** np.arange(16, dtype=np.float32)[None, :], (128, 1)))
    Bn = np.zeros((krows, 64), np.float32)
    for k in range(krows):
        Bn[k, k] = 1.0
    B = bf16(Bn)
    E = torch.full((128, 4), 0x44444444, dtype=torch.int64).to(torch.int32).cuda()
    res = []
    cfgs = [  # (m, layout, lbo, sbo, base_off, window_rows, start_row)
        (128, 2, 16384, 1024, 0, 8, 0), (128, 2, 16384, 640, 0, 5, 0), (128, 0, 128, krows * 16, 0, 8, 0),
        (128, 0, 80, krows * 16, 0, 5, 0), (64, 2, 16384, 640, 0, 5, 0), (64, 0, 80, krows * 16, 0, 5, 0),
        (128, 0, 96, krows * 16, 0, 6, 0), (128, 0, 112, krows * 16, 0, 7, 0), (128, 2, 16384, 768, 0, 6, 0),
        (128, 2, 16384, 640, 0, 5, 5), (128, 2, 16384, 640, 5, 5, 5), (128, 2, 16384, 640, 0, 5, 10),
        (128, 2, 16384, 640, 2, 5, 10), (128, 2, 16384, 896, 0, 7, 7), (64, 2, 16384, 640, 0, 5, 5)]
    if len(sys.argv) > 2:
        cfgs = [cfgs[int(sys.argv[2])]]
    for (m, layout, lbo, sbo, boff, w, r0) in cfgs:
        D = torch.zeros(128, 64, dtype=torch.float32, device="cuda")
        st = L.vnm_probe_window(A.data_ptr(), B.data_ptr(), E.data_ptr(), D.data_ptr(), m, krows, layout, lbo, sbo,
                                boff, r0)
        torch.cuda.synchronize()
        Dn = D.cpu().numpy()
        exp = np.zeros(64)
        for i in range(4):
            for p, j in ((0, 4 * i), (1, 4 * i + 1), (4, 4 * i + 2), (5, 4 * i + 3)):
                exp[r0 + i * w + p] += 2.0 ** j
        lane0 = Dn[0]
        r = {"m": m, "layout": layout, "lbo": lbo, "sbo": sbo, "window_rows": w, "start_row": r0, "base_off": boff,
             "status": st,
             "match_lane0": bool(np.array_equal(lane0, exp)),
             "rows_equal": bool(all(np.array_equal(Dn[l], lane0) for l in (range(128) if m == 128 else [0, 5, 32, 37]))),
             "lane0_nonzero": {int(k): float(v) for k, v in enumerate(lane0) if v != 0},
             "expected_nonzero": {int(k): float(v) for k, v in enumerate(exp) if v != 0}}
        print(json.dumps(r), flush=True)
        res.append(r)
    return res


if __name__ == "__main__":
    main()
