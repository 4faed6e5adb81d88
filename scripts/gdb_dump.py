# cuda-gdb helper (source after the exception / interrupt): maps every warp's PC of the focused block to a source
# line and dumps the small-T kernel's barrier words.  Env: DUMP_BAR_OFF = byte offset of full[] in dynamic smem.
import os, re
import gdb
out = gdb.execute("info cuda warps", to_string=True)
print(out)
for pc in sorted(set(re.findall(r"0x[0-9a-f]{12,}", out))):
    try:
        print(pc, gdb.execute("info line *" + pc, to_string=True).strip()[:300])
    except gdb.error as e:
        print(pc, "?", e)
off = int(os.environ.get("DUMP_BAR_OFF", "0"))
for base in (off, off + 1024):
    try:
        print("smem @", base, gdb.execute("x/24xg (@shared unsigned long long*)%d" % base, to_string=True))
    except gdb.error as e:
        print("smem read failed", base, e)
