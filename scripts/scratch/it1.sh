S="python scripts/time_spmm.py"
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 > gpurun_out/it1_tests.log 2>&1; echo "spmm tests exit $?"; tail -2 gpurun_out/it1_tests.log
for shape in "1536 384 5" "1536 1536 5" "384 1536 5" "1152 384 5"; do set -- $shape
  for abl in 15 0; do
    for cfg in "192,1" "256,1"; do
      VNM_ABL=$abl VNM_TC_PLAN=1 VNM_TC_CFG=$cfg timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc $cfg abl=$abl /"
    done
    for nt in 192 256; do
      VNM_ABL=$abl VNM_TC_PLAN=2 VNM_TC2_NT=$nt timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 $nt abl=$abl /"
    done
  done
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it1_deit_s.json 2>gpurun_out/it1_deit_s.err; echo "bench exit $?"
timeout 300 python bench.py --workload llama_prefill --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it1_llama_prefill.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it1_*.json
