mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/t15_tests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/t15_tests.log
for w in deit_s llama_prefill llama_decode llama_mlp_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t15_$w.json 2> gpurun_out/t15_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t15_$w.err; }
done
python scripts/bench_summary.py gpurun_out/t15_*.json
