S="python scripts/time_spmm.py"
VNM_TC_PLAN=3 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it17_t3.log 2>&1; echo "tc3 tests exit $?"; tail -2 gpurun_out/it17_t3.log
VNM_TC_PLAN=4 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled or llama_prefill" > gpurun_out/it17_t4.log 2>&1; echo "tc4 tests exit $?"; tail -2 gpurun_out/it17_t4.log
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "pair_resident" > gpurun_out/it17_f.log 2>&1; echo "forced test exit $?"; tail -2 gpurun_out/it17_f.log
for shape in "1536 384 5 50432" "1152 384 5 50432" "11008 4096 5 2048" "4096 11008 5 2048" "4096 4096 5 2048" "11008 4096 8 2048" "11008 4096 4 2048"; do set -- $shape
  timeout 60 $S $1 $2 $3 $4 tc 2>&1 | tail -1 | sed "s/^/  default /"
  VNM_TC_PLAN=3 timeout 60 $S $1 $2 $3 $4 tc 2>&1 | tail -1 | sed "s/^/  tc3 /"
  VNM_TC_PLAN=4 timeout 60 $S $1 $2 $3 $4 tc 2>&1 | tail -1 | sed "s/^/  tc3-stream /"
done
VNM_TC_PLAN=4 VNM_SPMM_TRACE=1 timeout 60 $S 11008 4096 5 2048 tc 2>&1 | grep -A3 "tc3 NT" | head -4
