S="python scripts/time_spmm.py"
VNM_TC_PLAN=3 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it9_tests.log 2>&1; echo "tc3 tests exit $?"; tail -2 gpurun_out/it9_tests.log
for shape in "1536 384 5" "1152 384 5" "384 384 5" "2304 768 8" "3072 768 8" "768 768 8"; do set -- $shape
  VNM_TC_PLAN=1 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc  /"
  for nt in 192 224; do for epi in 0 1; do
    VNM_TC3_EPI=$epi VNM_TC_PLAN=3 VNM_TC3_NT=$nt timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 $nt epi=$epi /"
  done; done
done
VNM_TC_PLAN=3 VNM_TC3_NT=224 VNM_SPMM_TRACE=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | grep -A4 "tc3 NT" | head -6
