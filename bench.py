#!/usr/bin/env python
"""Benchmark of the V:N:M sparse linear layer on B200 (BASELINE.json metric).

A step = one pass of the whole hot path over one batch of synthetic input:
for every linear layer of the workload, vnm_prune_compress(W) (importance, column L1, top-4, 2:4,
packing) then vnm_spmm(X^T, packed) -> Y^T (bf16 out, fp32 accumulate).  Default workload (N = 1):
BJ configs[1], the four DeiT-small linear layers at 64:2:5 with T = 197 x 256 tokens.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload deit_s|deit_b|llama_prefill|...]
  python bench.py --impl reference ...     # the CPU oracle on a bounded sample (reference arm)

Under torchrun (N > 1) every rank runs the same per-GPU workload on its own tokens (token sharding,
no data-path collective; scaling "weak"); timing is the max over ranks of device time.
value = useful TFLOP/s of the whole job = sum over ranks of 2*T*rows_p*K_c per step / time per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V:N:M SpMM TFLOP/s & HBM GB/s vs roofline, speedup vs dense/2:4 at 1/2/4/8 B200"

# (name, out_features = rows of W, in_features = cols of W)
WORKLOADS = {
    "toy": dict(V=64, M=8, T=16, layers=[("toy", 128, 64)], cfg=1),
    "deit_s": dict(V=64, M=5, T=197 * 256, cfg=2,
                   layers=[("qkv", 1152, 384), ("proj", 384, 384), ("fc1", 1536, 384), ("fc2", 384, 1536)]),
    "deit_b": dict(V=64, M=8, T=197 * 256, cfg=3,
                   layers=[("qkv", 2304, 768), ("proj", 768, 768), ("fc1", 3072, 768), ("fc2", 768, 3072)]),
    "llama_prefill": dict(V=64, M=5, T=2048, cfg=4,
                          layers=[("q", 4096, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]),
    "llama_decode": dict(V=64, M=5, T=16, cfg=4,
                         layers=[("q", 4096, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]),
    # every linear layer of one Llama2-7B transformer block at decode; layers whose inputs do not depend on each
    # other's outputs run as one grouped launch (vnm_spmm_batched): [q k v] [o] [gate up] [down]
    "llama_block_decode": dict(V=64, M=5, T=16, cfg=4,
                               layers=[("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
                                       ("gate", 11008, 4096), ("up", 11008, 4096), ("down", 4096, 11008)],
                               groups=[[0, 1, 2], [3], [4, 5], [6]]),
}
for _m in (4, 5, 6, 7, 8, 16):
    WORKLOADS[f"llama_mlp_m{_m}"] = dict(V=64, M=_m, T=2048, cfg=5, layers=[("up", 11008, 4096), ("down", 4096, 11008)])
# NEXT-1: the paper's V = 128 points (tab:bs-sped) on the Llama2-7B layers, decode and prefill
_LLAMA = [("q", 4096, 4096), ("up", 11008, 4096), ("down", 4096, 11008)]
for _m in (5, 8, 9, 10, 11, 13):
    WORKLOADS[f"llama_decode_v128_m{_m}"] = dict(V=128, M=_m, T=16, cfg=4, layers=_LLAMA)
    WORKLOADS[f"llama_prefill_v128_m{_m}"] = dict(V=128, M=_m, T=2048, cfg=4, layers=_LLAMA)
for _m in (4, 5, 6, 7, 8, 9, 10, 11, 13, 16):
    WORKLOADS[f"llama_mlp_v128_m{_m}"] = dict(V=128, M=_m, T=2048, cfg=5, layers=[("up", 11008, 4096), ("down", 4096, 11008)])


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def geom_numbers(rows, cols, V, M, T):
    rows_p = -(-rows // V) * V
    cols_p = -(-cols // M) * M
    nb = cols_p // M
    nb_pad = -(-nb // 8) * 8
    kc = 2 * nb
    useful = 2.0 * T * rows_p * kc
    dense = 2.0 * T * rows * cols
    packed_bytes = rows_p * 2 * nb_pad * 2 + rows_p * (nb_pad // 8) * 4 + (rows_p // V) * nb_pad * 4
    return dict(rows_p=rows_p, cols_p=cols_p, nb=nb, nb_pad=nb_pad, useful_flops=useful, dense_flops=dense,
                packed_bytes=packed_bytes, xt_bytes=cols * T * 2, yt_bytes=rows * T * 2,
                w_bytes=rows * cols * 2,
                prune_bytes=rows * cols * 2 + packed_bytes + rows_p * (-(-cols_p // 32)) * 4)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2410_16135_b200 import synth, vnm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import datetime
        # a bounded communicator timeout: a rank that dies or hangs fails the job instead of blocking it forever
        dist.init_process_group("nccl", timeout=datetime.timedelta(seconds=args.nccl_timeout),
                                device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = WORKLOADS[args.workload]
    V, M, T = wl["V"], wl["M"], wl["T"]
    cfgi = wl["cfg"]
    pk = peaks()

    # ---- synthetic inputs (host, seeded per rank), then resident copies in HBM
    layers = []
    out_mode = args.mode == "out"
    use_tc0 = T > 64 and vnm.tc_applies(V, M)
    for li, (name, rows_full, cols) in enumerate(wl["layers"]):
        # token mode: every rank its own tokens (seeded per rank) and a full weight; out mode: the same weight
        # and tokens on every rank, rank r owns a V-block-aligned row shard (whole 128-row tiles for the
        # window form) and Y^T is all-gathered
        rs = 0 if out_mode else 100 * rank
        W = synth.weights(rows_full, cols, seed=synth.seed(cfgi, 0) + 10 * li + rs, kind="outlier")
        ldx = -(-T // 8) * 8
        XT = synth.activations_t(cols, T, seed=synth.seed(cfgi, 1) + 10 * li + rs, ld=ldx)
        rows, shard_rows, r0 = rows_full, rows_full, 0
        if out_mode:
            from paper_2410_16135_b200 import dist as vdist
            al = 128 // V if use_tc0 else 1
            r0, r1 = vdist.shard_rows_for_prune(rows_full, V, rank, world, al)
            shard_rows = vdist.vblocks_per_rank(-(-rows_full // V) * V, V, world, al) * V
            W = np.ascontiguousarray(W[r0:r1]) if r1 > r0 else np.zeros((V, cols), np.uint16)
            rows = max(r1 - r0, V)
        Wh = torch.from_numpy(W.view(np.int16)).pin_memory()
        Xh = torch.from_numpy(XT.view(np.int16)).pin_memory()
        Wd = Wh.to(dev).view(torch.bfloat16)
        Xd = Xh.to(dev).view(torch.bfloat16)
        g = vnm.geometry(rows, cols, V, M)
        P = vnm.Packed.empty(g, dev)
        Yd = torch.empty((rows, ldx), dtype=torch.bfloat16, device=dev)
        Yh = torch.empty((rows, ldx), dtype=torch.int16).pin_memory()
        lay = dict(name=name, rows=rows, cols=cols, W=Wd, X=Xd, Wh=Wh, Xh=Xh, P=P, Y=Yd, Yh=Yh,
                   n=geom_numbers(rows, cols, V, M, T), n_full=geom_numbers(rows_full, cols, V, M, T))
        if out_mode:
            # the SpMM writes this rank's Y^T rows straight into its padded all-gather shard (no copy)
            lay["Ysh"] = torch.zeros((shard_rows, ldx), dtype=torch.bfloat16, device=dev)
            lay["Yall"] = torch.empty((world * shard_rows, ldx), dtype=torch.bfloat16, device=dev)
            lay["Y"] = lay["Ysh"][:rows]
        layers.append(lay)
    del W, XT
    L = vnm.lib()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    flush_rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def flush_l2():
        # write a buffer larger than L2, then read another one so the dirty lines of the write are written
        # back before the timed region (otherwise their write-back lands inside the first timed kernel)
        flush.zero_()
        flush_rd.sum()

    import ctypes

    use_tc = T > 64 and vnm.tc_applies(V, M)
    if use_tc:  # window-form buffers, written by vnm_prune_compress in the same pass (include/vnm.h)
        for l in layers:
            nv, nm = vnm.tc_bytes(l["P"].g)
            l["P"].values_tc = torch.empty(nv // 2, dtype=torch.bfloat16, device=dev)
            l["P"].meta_tc = torch.empty(nm // 4, dtype=torch.int32, device=dev)

    # every layer's mask + compression pass in ONE launch (vnm_prune_compress_batched, up to 8 weights of one
    # (V, M)); the ctypes argument arrays are built once (they hold device pointers only)
    nL = len(layers)
    cps = [l["P"].c() for l in layers]
    b_w = (ctypes.c_void_p * nL)(*[l["W"].data_ptr() for l in layers])
    b_lw = (ctypes.c_int64 * nL)(*[l["W"].stride(0) for l in layers])
    b_po = (ctypes.c_void_p * nL)(*[ctypes.cast(ctypes.pointer(cp), ctypes.c_void_p) for cp in cps])

    def prune_all():
        st = L.vnm_prune_compress_batched(nL, b_w, b_lw, None, None, b_po, None,
                                          ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        assert st == 0, vnm.status_string(st)

    for l in layers:  # split-K scratch (small T), allocated once outside the timed region
        l["ws"] = vnm.spmm_workspace(l["P"].g, T, dev)  # zero-initialised once; vnm_spmm leaves it zeroed
    # launch groups: independent layers as one vnm_spmm_batched call (workloads with "groups"; token mode)
    groups = wl.get("groups") if not out_mode else None
    groups = groups or [[i] for i in range(len(layers))]
    # every group after the first is launched with VNM_SPMM_WEIGHTS_READY: its weights were written by the prune
    # pass, which completed before the previous group's SpMM began (include/vnm.h); the small-T launches then issue
    # their first weight loads before waiting for that SpMM
    gargs = []
    for gi, gr in enumerate(groups):
        if out_mode:
            gargs.append(None)
            continue
        ls = [layers[i] for i in gr]
        wsg = vnm.spmm_batched_workspace([l["P"].g for l in ls], T, dev) if len(gr) > 1 else ls[0]["ws"]
        cpg = [l["P"].c() for l in ls]
        k = len(ls)
        flags = vnm.VNM_SPMM_WEIGHTS_READY if gi > 0 and not args.no_weights_ready else 0
        gargs.append(dict(n=k, cp=cpg, ws=wsg, flags=flags,
                          X=(ctypes.c_void_p * k)(*[l["X"].data_ptr() for l in ls]),
                          ldx=(ctypes.c_int64 * k)(*[l["X"].stride(0) for l in ls]),
                          P=(ctypes.c_void_p * k)(*[ctypes.cast(ctypes.pointer(c), ctypes.c_void_p) for c in cpg]),
                          Y=(ctypes.c_void_p * k)(*[l["Y"].data_ptr() for l in ls]),
                          ldy=(ctypes.c_int64 * k)(*[l["Y"].stride(0) for l in ls])))

    def spmm(l):
        cp = l["P"].c()
        ws = l["ws"]
        st = L.vnm_spmm(ctypes.c_void_p(l["X"].data_ptr()), l["X"].stride(0), T, ctypes.byref(cp),
                        ctypes.c_void_p(l["Y"].data_ptr()), l["Y"].stride(0), vnm.VNM_BF16,
                        ctypes.c_void_p(ws.data_ptr()) if ws is not None else None,
                        ws.numel() * 4 if ws is not None else 0,
                        ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        assert st == 0, vnm.status_string(st)

    def spmm_group(gi):
        """The layers of group gi: one vnm_spmm_batched call (independent layers; a single layer: the same plan as
        vnm_spmm, with the weights-ready flag)."""
        a = gargs[gi]
        if a is None:
            spmm(layers[groups[gi][0]])
            return
        ws = a["ws"]
        st = L.vnm_spmm_batched(a["n"], a["X"], a["ldx"], T, a["P"], a["Y"], a["ldy"], vnm.VNM_BF16, a["flags"],
                                ctypes.c_void_p(ws.data_ptr()) if ws is not None else None,
                                ws.numel() * 4 if ws is not None else 0,
                                ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        assert st == 0, vnm.status_string(st)

    def gather(l):
        # out mode: the padded shard (the SpMM wrote its rows in place) -> one NCCL all-gather (feature-major:
        # contiguous)
        if out_mode and world > 1:
            dist.all_gather_into_tensor(l["Yall"], l["Ysh"])

    def step(ev=None, ev_mid=None):
        """One step.  ev: per-launch timing events (the detail pass); ev_mid: one event between the batched
        prune pass and the SpMMs (the timed pass: the SpMM section is ev_mid -> end of step)."""
        if ev is not None:
            ev[0][0].record()
        prune_all()
        if ev_mid is not None:
            ev_mid.record()
        if ev is None:
            for gi in range(len(groups)):
                spmm_group(gi)
                for i in groups[gi]:
                    gather(layers[i])
            return
        for i, l in enumerate(layers):  # detail pass: every layer alone, an event pair around each launch
            ev[i][1].record()
            spmm(l)
            ev[i][2].record()
            gather(l)

    # e2e: host->device copies on one stream, compute on the main stream, device->host on a third, chained by
    # events per layer so the copies of layer i+1 / i-1 overlap the SpMM of layer i (PCIe is full duplex)
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def step_e2e():
        ev_w, ev_x, ev_y = torch.cuda.Event(), [torch.cuda.Event() for _ in layers], [torch.cuda.Event() for _ in layers]
        s_h2d.wait_stream(stream)
        with torch.cuda.stream(s_h2d):
            for l in layers:
                l["W"].view(torch.int16).copy_(l["Wh"], non_blocking=True)
            ev_w.record(s_h2d)
            for i, l in enumerate(layers):
                l["X"].view(torch.int16).copy_(l["Xh"], non_blocking=True)
                ev_x[i].record(s_h2d)
        stream.wait_event(ev_w)
        prune_all()
        s_d2h.wait_stream(stream)
        for gi, gr in enumerate(groups):
            for i in gr:
                stream.wait_event(ev_x[i])
            spmm_group(gi)
            for i in gr:
                l = layers[i]
                gather(l)
                ev_y[i].record(stream)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_y[i])
                    l["Yh"].copy_(l["Y"].view(torch.int16), non_blocking=True)
        stream.wait_stream(s_d2h)
        stream.wait_stream(s_h2d)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    E = lambda: torch.cuda.Event(enable_timing=True)
    # ---- the step is captured once into a CUDA graph (every launch of the step, through the C ABI, replayed
    # each timed step).  Timing events inside a graph are external-event nodes costing ~4 us each (measured:
    # 9 of them added 37 us to the DeiT-S step), so the TIMED graph holds one: between the batched prune pass
    # and the SpMMs (prune = step start -> it, SpMM section = it -> step end, both live in the timed region);
    # a second graph with an event around every launch gives the per-layer breakdown (detail, not timed).
    for _ in range(2):
        step()  # module loading / first-touch outside the capture
    torch.cuda.synchronize(dev)
    EX = lambda: torch.cuda.Event(enable_timing=True, external=True)
    ev_mid = EX()
    graph = torch.cuda.CUDAGraph()
    n_launch0 = vnm.launch_count()
    with torch.cuda.graph(graph):
        step(None, ev_mid)
    launches_per_step = vnm.launch_count() - n_launch0
    ev = [(EX(), EX(), EX()) for _ in layers]
    graph_detail = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_detail):
        step(ev)
    grouped = any(len(gr) > 1 for gr in groups)
    if grouped:  # per-group times of the grouped launches (detail)
        evg = [(EX(), EX()) for _ in groups]
        graph_groups = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_groups):
            prune_all()
            for gi in range(len(groups)):
                evg[gi][0].record()
                spmm_group(gi)
                evg[gi][1].record()
    # ---- warm-up
    for _ in range(args.warmup):
        graph.replay()
    barrier()
    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    step_ms, pc_t_ms, sp_t_ms = [], [], []
    with ClockSampler(local) as clk:
        # keep the GPU under this same load for >= 0.6 s right before the timed steps so nvidia-smi (200 ms
        # period) sees the clocks of this workload; these steps are not timed
        t_load = time.perf_counter() + 0.6
        while time.perf_counter() < t_load:
            graph.replay()
            torch.cuda.synchronize(dev)
        barrier()
        for _ in range(args.steps):
            flush_l2()
            s0, s1 = E(), E()
            s0.record(stream)
            graph.replay()
            s1.record(stream)
            torch.cuda.synchronize(dev)
            step_ms.append(s0.elapsed_time(s1))
            pc_t_ms.append(s0.elapsed_time(ev_mid))   # the batched prune pass (all layers)
            sp_t_ms.append(ev_mid.elapsed_time(s1))   # the SpMM launches of every layer, back to back
        launches = launches_per_step * args.steps
        barrier()
    # ---- per-layer breakdown (detail; same flush, not part of the timed region)
    pc_ms, sp_ms = [[] for _ in layers], [[] for _ in layers]
    for _ in range(args.steps):
        flush_l2()
        graph_detail.replay()
        torch.cuda.synchronize(dev)
        pc_ms[0].append(ev[0][0].elapsed_time(ev[0][1]))
        for i in range(len(layers)):
            sp_ms[i].append(ev[i][1].elapsed_time(ev[i][2]))
    grp_ms = [[] for _ in groups]
    if grouped:
        for _ in range(args.steps):
            flush_l2()
            graph_groups.replay()
            torch.cuda.synchronize(dev)
            for gi in range(len(groups)):
                grp_ms[gi].append(evg[gi][0].elapsed_time(evg[gi][1]))
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    # token mode: every rank does the full layers on its own tokens; out mode: the ranks share the full layers
    useful = sum(l["n_full" if out_mode else "n"]["useful_flops"] for l in layers)
    dense = sum(l["n_full" if out_mode else "n"]["dense_flops"] for l in layers)
    value = (1 if out_mode else world) * useful / (ms_per_step * 1e-3) / 1e12  # out mode: useful = full layers

    # ---- roofline of the dominant kernel (vnm_spmm), measured live above
    sp_bytes = sum(l["n"]["packed_bytes"] + l["n"]["xt_bytes"] + l["n"]["yt_bytes"] for l in layers)
    sp_t = statistics.mean(sp_t_ms) * 1e-3   # timed region: the SpMM section of the step
    pc_t = statistics.mean(pc_t_ms) * 1e-3
    hbm_t = sp_bytes / (pk["hbm_gbs"] * 1e9)
    tc_t = useful / (pk["bf16_tflops"] * 1e12)
    bound = "hbm" if hbm_t >= tc_t else "tensor"
    if bound == "hbm":
        achieved, peak, unit = sp_bytes / sp_t / 1e9, pk["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = useful / sp_t / 1e12, pk["bf16_tflops"], "TFLOP/s"
    traffic, traffic_note = None, None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            t = json.load(open(tf)).get(args.workload)
            if t:
                # dram read + write bytes of one captured launch (ncu --set full); its algorithmic bytes beside it
                li = next((i for i, l in enumerate(layers) if t["launch"].startswith(l["name"] + " ")), None)
                traffic = t["bytes_per_launch"]
                if li is not None:
                    n = layers[li]["n"]
                    traffic_note = (f"{t['launch']}: {traffic / 1e6:.1f} MB DRAM vs "
                                    f"{(n['packed_bytes'] + n['xt_bytes'] + n['yt_bytes']) / 1e6:.1f} MB algorithmic "
                                    f"({t['source']})")
        except Exception:
            traffic = None
    roofline = {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_note": traffic_note,
                "kernel": ("vnm_spmm (tcgen05.mma.sp window-form / small-T kernels, " +
                           ("independent layers grouped into vnm_spmm_batched launches" if grouped else "per-layer launches") +
                           "); time = the SpMM section of each timed step (one event after the prune pass -> step end, "
                           "inter-kernel gaps included)"),
                "peak_source": "MEASURED_PEAKS.json" if not pk.get("fallback") else "fallback",
                "spmm_share_of_step": round(sp_t / (ms_per_step * 1e-3), 4)}
    if bound == "hbm" and args.workload.startswith("deit"):
        # context, not the denominator: at these layer sizes and read:write mixes HBM itself reaches ~4.8 TB/s
        # (tests/probes/probe_mix.cu, profiles/r02f_probe_mix.txt); the 6548 GB/s peak is a 4 GB copy
        roofline["context"] = {"hbm_reachable_gbs": 4800, "frac_of_reachable": round(achieved / 4800, 4),
                               "source": "profiles/r02f_probe_mix.txt"}

    # ---- e2e through the public API with host buffers (H2D inputs, D2H Y inside the timed region)
    barrier()
    e_ms = []
    for _ in range(max(2, min(args.steps, 5))):
        flush_l2()
        a0, a1 = E(), E()
        a0.record(stream)
        step_e2e()
        a1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms.append(a0.elapsed_time(a1))
    e2e_ms = statistics.mean(e_ms)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = sum(l["Wh"].numel() * 2 + l["Xh"].numel() * 2 for l in layers)
    d2h = sum(l["Yh"].numel() * 2 for l in layers)
    e2e = {"value": round(world * useful / (e2e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)}

    # ---- baselines on the same shapes (not in the timed region): cuBLAS dense, cuSPARSELt 2:4
    base = {}
    if not args.no_baselines:
        base = baselines(layers, T, stream, flush_l2, dev, args.steps)
    sp_layer_ms = [statistics.mean(x) for x in sp_ms]
    detail = {"layers": [{"name": l["name"], "rows": l["rows"], "cols": l["cols"],
                          "spmm_us": round(1e3 * sp_layer_ms[i], 2),

                          "spmm_useful_tflops": round(l["n"]["useful_flops"] / (sp_layer_ms[i] * 1e-3) / 1e12, 2),
                          "spmm_dense_equiv_tflops": round(l["n"]["dense_flops"] / (sp_layer_ms[i] * 1e-3) / 1e12, 2),
                          "spmm_gbs": round((l["n"]["packed_bytes"] + l["n"]["xt_bytes"] + l["n"]["yt_bytes"]) /
                                            (sp_layer_ms[i] * 1e-3) / 1e9, 1),
                          **{k: v[i] for k, v in base.items() if isinstance(v, list)}}
                         for i, l in enumerate(layers)]}
    if base.get("dense_ms") is not None:
        detail["speedup_vs_dense"] = round(base["dense_ms"] / sum(sp_layer_ms), 3)
    if base.get("cslt_ms") is not None:
        detail["speedup_vs_24"] = round(base["cslt_ms"] / sum(sp_layer_ms), 3)
    detail["dense_equiv_tflops"] = round((1 if out_mode else world) * dense / (ms_per_step * 1e-3) / 1e12, 2)
    detail["prune_compress_share"] = round(pc_t / (ms_per_step * 1e-3), 4)
    detail["prune_compress_batched_us"] = round(pc_t * 1e6, 2)  # one vnm_prune_compress_batched launch, all layers
    detail["prune_gbs"] = round(sum(l["n"]["prune_bytes"] for l in layers) / pc_t / 1e9, 1)
    detail["step_ms_min"] = round(min(step_ms), 4)
    if grouped:  # the timed step's launches: groups of independent layers (one vnm_spmm_batched call each)
        detail["groups"] = []
        for gi, gr in enumerate(groups):
            t_g = statistics.mean(grp_ms[gi]) * 1e-3
            b_g = sum(layers[i]["n"]["packed_bytes"] + layers[i]["n"]["xt_bytes"] + layers[i]["n"]["yt_bytes"] for i in gr)
            detail["groups"].append({"layers": "+".join(layers[i]["name"] for i in gr), "spmm_us": round(t_g * 1e6, 2),
                                     "spmm_gbs": round(b_g / t_g / 1e9, 1),
                                     **({"dense_us": round(sum(base["dense_us"][i] for i in gr), 2)}
                                        if base.get("dense_us") else {})})
        if base.get("dense_ms") is not None:
            detail["speedup_vs_dense_grouped"] = round(base["dense_ms"] / (sum(statistics.mean(x) for x in grp_ms)), 3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_seconds)
    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
               "scaling": "strong" if out_mode else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": {"workload": f"{args.workload} V:N:M {V}:2:{M}", "tokens_per_gpu": T,
                          "layers": [f"{n} {c}->{r}" for n, r, c in wl["layers"]],
                          "parallelism": (f"output-feature sharded x{world} + NCCL all-gather of Y^T" if out_mode else
                                          f"token-sharded x{world}") if world > 1 else "single GPU",
                          "l2": "flushed between timed steps (256 MB write, then a 256 MB read so its write-back happens before the timing)",
                          "launch": "timed steps replay one CUDA graph of the step; e2e launches eagerly",
                          **({"spmm_groups": ["+".join(layers[i]["name"] for i in gr) for gr in groups]} if grouped else {})},
               "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "roofline": roofline,
               "cpu_baseline": cpu, "detail": detail}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def baselines(layers, T, stream, flush_l2, dev, steps):
    """cuBLAS dense bf16 GEMM and cuSPARSELt 2:4 on the same shapes (Y^T = W X^T), kernel time only."""
    import torch
    res = {"dense_us": [], "cslt_us": []}
    E = lambda: torch.cuda.Event(enable_timing=True)
    dense_tot, cslt_tot, cslt_ok = 0.0, 0.0, True
    for l in layers:
        W = l["W"].contiguous()
        X = l["X"][:, :T]
        Y = torch.empty((l["rows"], T), dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            torch.matmul(W, X, out=Y)
        ts = []
        for _ in range(max(3, steps)):
            flush_l2()
            a, b = E(), E()
            a.record(stream)
            torch.matmul(W, X, out=Y)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(a.elapsed_time(b))
        d = statistics.mean(ts)
        dense_tot += d
        res["dense_us"].append(round(d * 1e3, 2))
        c = None
        try:
            w24 = W.view(-1, 4).float().abs().argsort(dim=1, descending=True)[:, :2]
            m = torch.zeros_like(W.view(-1, 4), dtype=torch.bool).scatter_(1, w24, True)
            Wp = (W.view(-1, 4) * m).view_as(W)
            comp = torch._cslt_compress(Wp)
            Xc = X.contiguous()
            for _ in range(3):
                torch._cslt_sparse_mm(comp, Xc)
            ts = []
            for _ in range(max(3, steps)):
                flush_l2()
                a, b = E(), E()
                a.record(stream)
                torch._cslt_sparse_mm(comp, Xc)
                b.record(stream)
                torch.cuda.synchronize(dev)
                ts.append(a.elapsed_time(b))
            c = statistics.mean(ts)
            cslt_tot += c
        except Exception as e:  # noqa
            cslt_ok = False
            res["cslt_error"] = repr(e)[:200]
        res["cslt_us"].append(None if c is None else round(c * 1e3, 2))
    res["dense_ms"] = dense_tot
    res["cslt_ms"] = cslt_tot if cslt_ok else None
    return res


# ---------------------------------------------------------------------------------------------- CPU oracle
def cpu_baseline(wl, seconds):
    import oracle
    from paper_2410_16135_b200 import synth
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    V, M = wl["V"], wl["M"]
    inputs = []
    for li, (name, rows, cols) in enumerate(wl["layers"]):
        inputs.append((rows, cols, synth.weights(rows, cols, seed=synth.seed(wl["cfg"], 0) + 10 * li, kind="outlier")))

    def once(tokens):
        flops, el = 0.0, 0.0
        for li, (rows, cols, W) in enumerate(inputs):
            XT = synth.activations_t(cols, tokens, seed=synth.seed(wl["cfg"], 1) + 10 * li)
            t0 = time.perf_counter()
            mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
            oracle.spmm_packed(XT, values, col_idx, meta, rows, cols, V, M)
            el += time.perf_counter() - t0
            flops += geom_numbers(rows, cols, V, M, tokens)["useful_flops"]
        return flops, el

    tokens = min(wl["T"], 64)
    f, el = once(tokens)
    # grow the token sample until one pass is >= `seconds` (bounded by the workload's T)
    while el < seconds and tokens < wl["T"]:
        tokens = min(wl["T"], int(tokens * max(2.0, min(8.0, seconds / max(el, 1e-3)))))
        f, el = once(tokens)
    return {"value": round(f / el / 1e12, 6), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(inputs)} layers: prune+pack of every full weight + packed fp64 SpMM (O9) over "
                      f"{tokens} of {wl['T']} tokens; {el:.1f} s"}


def run_reference(args):
    """Reference arm: the CPU oracle as it stands, on the same workload / metric, bounded samples."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2410_16135_b200 import synth
    wl = WORKLOADS[args.workload]
    cores = len(os.sched_getaffinity(0))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    V, M = wl["V"], wl["M"]
    inputs = []
    for li, (name, rows, cols) in enumerate(wl["layers"]):
        W = synth.weights(rows, cols, seed=synth.seed(wl["cfg"], 0) + 10 * li, kind="outlier")
        inputs.append((rows, cols, W))
    tokens = min(wl["T"], args.ref_tokens)
    XTs = [synth.activations_t(c, tokens, seed=synth.seed(wl["cfg"], 1) + 10 * i) for i, (r, c, _) in enumerate(inputs)]

    def step():
        for (rows, cols, W), XT in zip(inputs, XTs):
            mask, values, col_idx, meta = oracle.prune_pack(W, V, M)
            oracle.spmm_packed(XT, values, col_idx, meta, rows, cols, V, M)

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    flops = sum(geom_numbers(r, c, V, M, tokens)["useful_flops"] for r, c, _ in inputs)
    ms = 1e3 * statistics.mean(ts)
    value = flops / (ms * 1e-3) / 1e12
    sample = (f"{len(inputs)} layers: prune+pack of every full weight + packed fp64 SpMM (O9) over {tokens} of "
              f"{wl['T']} tokens per step")
    print(json.dumps({
        "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.workload} V:N:M {V}:2:{M}", "tokens_per_gpu": wl["T"],
                   "layers": [f"{n} {c}->{r}" for n, r, c in wl["layers"]], "parallelism": "host cores"},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0}), flush=True)


def ensure_world(args):
    """--gpus N is the number of ranks: without a torchrun environment and N > 1, re-execute this command under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1); under torchrun, WORLD_SIZE must
    equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            import socket
            s = socket.socket()
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
            s.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            sys.stdout.flush()
            os.execv(sys.executable, cmd)
        return
    if int(world) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank per GPU (--gpus = nproc)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="deit_s", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="vnm", choices=["vnm", "reference"])
    ap.add_argument("--mode", default="token", choices=["token", "out"],
                    help="multi-GPU partitioning: token sharding (weak scaling, no collective) or V-block-aligned "
                         "output sharding + NCCL all-gather of Y^T (strong scaling)")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-weights-ready", action="store_true",
                    help="launch every SpMM group without VNM_SPMM_WEIGHTS_READY (comparison)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-tokens", type=int, default=1024)
    ap.add_argument("--nccl-timeout", type=int, default=600, help="seconds (torch.distributed init timeout)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ensure_world(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
