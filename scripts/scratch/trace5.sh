bash scripts/trace3.sh > /dev/null 2>&1
sed -i 's/fl.zero_()/fl.zero_(); torch.cuda.synchronize()/' /tmp/tr.py
timeout 60 python /tmp/tr.py 16 1 flush > gpurun_out/trace_m1.log 2>&1; grep "cta span" gpurun_out/trace_m1.log
timeout 60 python /tmp/tr.py 16 1 > gpurun_out/trace_w.log 2>&1; grep "cta span" gpurun_out/trace_w.log
