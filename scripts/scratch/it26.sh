S="python scripts/time_spmm.py"
VNM_TC_PLAN=3 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it26_t3.log 2>&1; echo "tc3 tests exit $?"; tail -2 gpurun_out/it26_t3.log
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "pair_resident or deit" > gpurun_out/it26_f.log 2>&1; echo "forced+deit tests exit $?"; tail -2 gpurun_out/it26_f.log
for shape in "1536 384 5" "1152 384 5"; do set -- $shape
  for s in 5 6 7; do VNM_TC3_S=$s VNM_TC_PLAN=3 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 S<=$s /"; done
done
VNM_TC_PLAN=3 VNM_SPMM_TRACE=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | grep -A2 "tc3 NT" | head -3
