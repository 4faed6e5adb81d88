"""MB1/MB2 hardware probes, run on a B200:  python tests/probe_layouts.py [out.json]

MB1: discover, for tcgen05.mma.sp.cta_group::1.kind::f16 with M = 64 and M = 128, which TMEM lane /
column / nibble of the metadata steers which (row, K-group) of the MMA, and in which TMEM lane each
row of D lands.  Method: B = identity (32 x 64), so D[row][n] = the stored value the metadata routes to
logical column n.  Five trials encode (lane, column, nibble) of every metadata nibble in base 6 over
the six valid 2:4 nibbles; decoding the observed selections gives the source of each (row, group).
MB2: back-to-back MMA throughput (cycles per instruction) for sparse M=64 / M=128 and dense.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
VALID = [0x4, 0x8, 0xC, 0x9, 0xD, 0xE]


def bf16(a):
    return torch.tensor(np.asarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).cuda()


def load():
    L = ctypes.CDLL(os.path.join(ROOT, "tests", "probes", "libvnm_probe.so"))
    P, u32 = ctypes.c_void_p, ctypes.c_uint32
    L.vnm_probe_sparse_mma.argtypes = [P, P, P, P, u32, u32, u32, u32, P]
    L.vnm_probe_bench_mma.argtypes = [u32, u32, u32, u32, u32, P, P]
    return L


def run(L, A, B, E, m_mma, id2, off, sparse):
    D = torch.zeros(128, 64, dtype=torch.float32, device="cuda")
    st = L.vnm_probe_sparse_mma(A.data_ptr(), B.data_ptr(), E.data_ptr(), D.data_ptr(), m_mma, id2, off, sparse,
                                None)
    torch.cuda.synchronize()
    assert st == 0, st
    return D.cpu().numpy()


def probe_sparse(L, m_mma, id2, off):
    res = {"m_mma": m_mma, "id2": id2, "e_col_off": off}
    Bn = np.zeros((32, 64), np.float32)
    for k in range(32):
        Bn[k, k] = 1.0
    B = bf16(Bn)
    # row mapping: A[m][j] = m+1, all metadata 0x4 (positions 0,1 of every group)
    A = bf16(np.tile(np.arange(1, 129, dtype=np.float32)[:, None], (1, 16)))
    E = torch.full((128, 4), 0x44444444, dtype=torch.int64).to(torch.int32).cuda()
    D = run(L, A, B, E, m_mma, id2, off, 1)
    lane_row = {}
    for lane in range(128):
        nz = D[lane][:32]
        if np.any(nz != 0):
            vals = set(nz[nz != 0].tolist())
            lane_row[lane] = sorted(vals)
    res["lane_to_row_plus1"] = {str(k): v for k, v in lane_row.items()}
    res["row_probe_pattern_ok"] = all(
        (D[lane][:32].reshape(8, 4) != 0).tolist() == [[True, True, False, False]] * 8 for lane in lane_row)
    # metadata source decoding
    A = bf16(np.tile(np.arange(1, 17, dtype=np.float32)[None, :], (128, 1)))
    codes = {}
    anomalies = []
    for t in range(5):
        E = np.zeros((128, 4), np.uint32)
        for lane in range(128):
            for c in range(4):
                w = 0
                for q in range(8):
                    code = (lane * 4 + c) * 8 + q
                    w |= VALID[(code // 6 ** t) % 6] << (4 * q)
                E[lane, c] = w
        Et = torch.tensor(E.view(np.int32)).cuda()
        D = run(L, A, B, Et, m_mma, id2, off, 1)
        for lane in range(128):
            row = D[lane][:32]
            if not np.any(row != 0):
                continue
            for g in range(8):
                grp = row[4 * g:4 * g + 4]
                pos = [p for p in range(4) if grp[p] != 0]
                if len(pos) != 2:
                    anomalies.append((t, lane, g, grp.tolist()))
                    continue
                js = [int(grp[p]) - 1 for p in pos]
                if js != [2 * g, 2 * g + 1]:
                    anomalies.append((t, lane, g, "values", js))
                nib = pos[0] | (pos[1] << 2)
                digit = VALID.index(nib)
                codes.setdefault((lane, g), 0)
                codes[(lane, g)] += digit * 6 ** t
    mapping = {}
    for (lane, g), code in sorted(codes.items()):
        src_lane, rem = divmod(code, 32)
        src_col, src_q = divmod(rem, 8)
        mapping[f"{lane},{g}"] = [src_lane, src_col, src_q]
    res["dlane_group_to_meta_lane_col_nibble"] = mapping
    res["anomalies"] = anomalies[:20]
    res["n_anomalies"] = len(anomalies)
    return res


def probe_dense_rows(L, m_mma):
    Bn = np.zeros((32, 64), np.float32)
    for k in range(16):
        Bn[k, k] = 1.0
    A = bf16(np.tile(np.arange(1, 129, dtype=np.float32)[:, None], (1, 16)))
    E = torch.zeros(128, 4, dtype=torch.int32, device="cuda")
    D = run(L, A, bf16(Bn), E, m_mma, 0, 0, 0)
    out = {}
    for lane in range(128):
        nz = D[lane][:16]
        if np.any(nz != 0):
            out[str(lane)] = sorted(set(nz[nz != 0].tolist()))
    return {"m_mma": m_mma, "dense_lane_to_row_plus1": out}


def bench(L):
    out = []
    nblk = torch.cuda.get_device_properties(0).multi_processor_count
    for (m, n, sp) in [(64, 256, 1), (128, 256, 1), (128, 256, 0), (64, 256, 0), (64, 128, 1), (64, 64, 1),
                       (128, 128, 1), (64, 16, 1)]:
        cyc = torch.zeros(nblk, dtype=torch.int64, device="cuda")
        iters = 4096
        L.vnm_probe_bench_mma(m, n, sp, 16, nblk, cyc.data_ptr(), None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.vnm_probe_bench_mma(m, n, sp, iters, nblk, cyc.data_ptr(), None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        k_logical = 32 if sp else 16
        k_eff = 16
        flops_eff = 2.0 * m * n * k_eff * iters * nblk
        c = cyc.cpu().numpy()
        out.append({"M": m, "N": n, "sparse": sp, "cycles_per_mma": float(np.median(c)) / iters,
                    "ms": ms, "effectual_tflops": flops_eff / ms / 1e9,
                    "logical_tflops": 2.0 * m * n * k_logical * iters * nblk / ms / 1e9})
    return out


def main():
    """usage: probe_layouts.py sparse M ID2 OFF | dense | bench      (one mode per process: a fault in one
    configuration must not take the others down)"""
    L = load()
    mode = sys.argv[1]
    outdir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(outdir, exist_ok=True)
    if mode == "sparse":
        m, id2, off = map(int, sys.argv[2:5])
        r = probe_sparse(L, m, id2, off)
        name = f"probe_sparse_{m}_{id2}_{off}.json"
        print(json.dumps({k: v for k, v in r.items() if k != "dlane_group_to_meta_lane_col_nibble"})[:3000])
    elif mode == "dense":
        r = [probe_dense_rows(L, m) for m in (64, 128)]
        name = "probe_dense.json"
        print(json.dumps(r)[:3000])
    else:
        r = bench(L)
        name = "probe_bench.json"
        for b in r:
            print(json.dumps(b))
    json.dump(r, open(os.path.join(outdir, name), "w"), indent=1)


if __name__ == "__main__":
    main()
