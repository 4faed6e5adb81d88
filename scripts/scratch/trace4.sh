mkdir -p gpurun_out
bash scripts/trace3.sh > /dev/null 2>&1
for m in 1; do timeout 60 python /tmp/tr.py 16 $m flush > gpurun_out/trace_m$m.log 2>&1; echo "== mode $m"; grep "trace q" gpurun_out/trace_m$m.log | sed -n "14,22p"; done
