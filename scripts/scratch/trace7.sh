bash scripts/trace3.sh > /dev/null 2>&1
sed -i 's/fl.zero_()/fl.zero_(); torch.cuda.synchronize()/' /tmp/tr.py
for m in 1 7 9 10; do timeout 60 python /tmp/tr.py 16 $m flush > gpurun_out/trace_m$m.log 2>&1; echo "== mode $m $(grep 'cta span' gpurun_out/trace_m$m.log | cut -c1-30)"; done
