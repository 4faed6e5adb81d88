mkdir -p gpurun_out
for s in "11008 4096 5 16" "4096 4096 5 16"; do
  VNM_SPMM_TRACE=1 timeout 120 python scripts/time_spmm.py $s > gpurun_out/r02c_trace_$(echo $s | tr ' ' _).txt 2>&1
  tail -3 gpurun_out/r02c_trace_$(echo $s | tr ' ' _).txt
  timeout 120 python scripts/time_spmm.py $s
  VNM_SMALLT=0 timeout 120 python scripts/time_spmm.py $s
done
C="python scripts/time_spmm.py 11008 4096 5 16"
timeout 120 $C > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_smallt -s 25 -c 1 -o gpurun_out/r02c_prof_smallt_up $C > gpurun_out/r02c_ncu.log 2>&1; echo "ncu exit $?"
