VNM_TC_PLAN=3 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled or natural" > gpurun_out/it35.log 2>&1; echo "tc3 tests $?"; tail -1 gpurun_out/it35.log
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "pair_resident" > gpurun_out/it35b.log 2>&1; echo "forced $?"; tail -1 gpurun_out/it35b.log
S="python scripts/time_spmm.py"
for shape in "1536 384 5" "1152 384 5"; do set -- $shape; for i in 1 2; do timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1; done; done
