"""One line per bench JSON: value, roofline, per-layer SpMM numbers (for quick reading of gpurun output)."""
import json
import sys

for fn in sys.argv[1:]:
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
    except Exception as e:  # noqa
        print(fn, "unreadable", e)
        continue
    r = d.get("roofline", {})
    det = d.get("detail", {})
    print(fn, d["config"]["workload"], "value", d["value"], d["unit"], "ms", d["ms_per_step"],
          "roof", r.get("bound"), r.get("achieved"), r.get("unit"), r.get("frac"),
          "e2e", d.get("e2e", {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"),
          "vs_dense", det.get("speedup_vs_dense"), "vs_24", det.get("speedup_vs_24"),
          "prune_batched_us", det.get("prune_compress_batched_us"), det.get("prune_gbs"), "GB/s")
    for l in det.get("layers", []):
        print("   ", l["name"], f"spmm {l['spmm_us']}us {l['spmm_useful_tflops']}TF {l['spmm_gbs']}GB/s",
              "dense", l.get("dense_us"), "cslt", l.get("cslt_us"))
