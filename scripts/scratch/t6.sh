mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py -m gpu -q -x --timeout 200 > gpurun_out/t6_tests.log 2>&1; echo "prune tests $?"; tail -4 gpurun_out/t6_tests.log
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window or any_v or deit or prefill or toy" > gpurun_out/t6_tests2.log 2>&1; echo "spmm tests $?"; tail -3 gpurun_out/t6_tests2.log
bash scripts/trace_prune.sh
for w in deit_s llama_decode llama_prefill; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t6_$w.json 2> gpurun_out/t6_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t6_$w.err; continue; }
done
python scripts/bench_summary.py gpurun_out/t6_*.json
