mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 > gpurun_out/t4_tests.log 2>&1; echo "tests $?"; tail -25 gpurun_out/t4_tests.log
for w in deit_s llama_prefill llama_decode deit_b; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t4_$w.json 2> gpurun_out/t4_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t4_$w.err; continue; }
done
python scripts/bench_summary.py gpurun_out/t4_*.json
