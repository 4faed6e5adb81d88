S="python scripts/time_spmm.py"
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 > gpurun_out/it10_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/it10_tests.log
for shape in "1152 384 5" "384 384 5" "1536 384 5" "384 1536 5" "2304 768 8" "768 768 8" "3072 768 8" "768 3072 8"; do set -- $shape
  for cfg in "192,1" "256,1" "128,2" "192,2"; do
    VNM_TC_PLAN=1 VNM_TC_CFG=$cfg timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc $cfg /"
  done
  VNM_TC_PLAN=2 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 /"
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it10_deit_s.json 2>gpurun_out/it10_deit_s.err; echo "bench exit $?"
timeout 300 python bench.py --workload deit_b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it10_deit_b.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it10_*.json
