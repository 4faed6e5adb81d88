"""Top SASS lines by warp-stall samples of an ncu report (source page), for reading profiles here."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
i = h.index("Warp Stall Sampling (All Samples)")
j = h.index("Warp Stall Sampling (Not-issued Samples)")
rows = [x for x in r[2:] if len(x) > i and x[i].isdigit()]
tot = sum(int(x[i]) for x in rows)
print("total samples", tot)
for x in sorted(rows, key=lambda x: -int(x[i]))[:n]:
    print(f"{x[i]:>6} {x[j]:>6}  {x[0][-5:]}  {x[1][:100]}")
