"""SASS listing of an ncu report with per-instruction execution counts (source page), for reading here."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
ie = h.index("Instructions Executed")
rows = [x for x in r[2:] if len(x) > ie and x[ie].replace(".", "").isdigit()]
tot = sum(float(x[ie]) for x in rows)
print("total warp instructions", tot)
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
for x in rows:
    f = float(x[ie]) / tot
    if f >= lo:
        print(f"{100 * f:5.2f}%  {x[0][-5:]}  {x[1][:110]}")
