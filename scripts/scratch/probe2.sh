mkdir -p gpurun_out
for m in interleave mma_multi gather4 tma_bw tmem_cp; do
  timeout 120 python tests/probe2.py $m > gpurun_out/probe2_$m.log 2>&1; echo "$m exit $?"; tail -14 gpurun_out/probe2_$m.log
done
