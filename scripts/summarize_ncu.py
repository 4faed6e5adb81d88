"""Summaries of ncu captures for profiles/ (run here, on the CPU box, on files gpurun brought back).

  python scripts/summarize_ncu.py launches <launches.csv> <out.txt>
      per-kernel launch count, mean/total device time and share of the listed time
  python scripts/summarize_ncu.py full <prof.ncu-rep> <out.txt> [--traffic-json profiles/ncu_traffic.json --key K]
      key metrics of a `--set full` capture (duration, DRAM bytes / throughput, L2, tensor pipe, occupancy,
      stall reasons) and optionally records dram read+write bytes per launch as the bench's `traffic`
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second", "l1tex__t_bytes.sum",
    "smsp__inst_executed.sum",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        try:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
        except (ValueError, IndexError):
            pass
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list: {path}", "# gpu__time_duration.sum (ns), --clock-control none, cold-cache serialised",
             f"{'launches':>8} {'mean_us':>10} {'total_us':>10} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / 1e3:10.1f} {sum(v) / total:7.3f}  {k[:110]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out, traffic_json=None, key=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {path}"]
    per_launch = []
    for data in rows[2:]:
        d = dict(zip(h, data))
        lines.append(f"## {d.get('Kernel Name', '')[:120]}")
        for k in KEYS:
            if k in d:
                lines.append(f"{k:70s} {d[k]} {u[h.index(k)]}")
        stalls = [(n, d[n]) for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")]
        stalls = sorted(((n, float(v.replace(',', '') or 0)) for n, v in stalls), key=lambda x: -x[1])[:8]
        lines.append("top stall reasons (pc samples): " + ", ".join(f"{n.split('stalled_')[1]}={int(v)}" for n, v in stalls))
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * (1e6 if "Mbyte" in u[h.index("dram__bytes_read.sum")] else 1e3 if "Kbyte" in u[h.index("dram__bytes_read.sum")] else 1e9 if "Gbyte" in u[h.index("dram__bytes_read.sum")] else 1)
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * (1e6 if "Mbyte" in u[h.index("dram__bytes_write.sum")] else 1e3 if "Kbyte" in u[h.index("dram__bytes_write.sum")] else 1e9 if "Gbyte" in u[h.index("dram__bytes_write.sum")] else 1)
            per_launch.append(rd + wr)
        except (KeyError, ValueError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json and key and per_launch:
        try:
            t = json.load(open(traffic_json))
        except FileNotFoundError:
            t = {}
        t[key] = per_launch[0]
        json.dump(t, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj, key)
