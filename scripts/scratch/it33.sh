VNM_TC_PLAN=1 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled or prefill" > gpurun_out/it33.log 2>&1; echo "tc forced $?"; tail -1 gpurun_out/it33.log
VNM_TC_PLAN=1 VNM_TC_CFG=256,1 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it33b.log 2>&1; echo "tc 256 forced $?"; tail -1 gpurun_out/it33b.log
S="python scripts/time_spmm.py"
for shape in "384 1536 5" "384 384 5" "1536 384 5" "768 3072 8" "2304 768 8"; do set -- $shape
  for cfg in "192,1" "256,1"; do VNM_TC_PLAN=1 VNM_TC_CFG=$cfg timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  $cfg /"; done
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it33_deit_s.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it33_deit_s.json
