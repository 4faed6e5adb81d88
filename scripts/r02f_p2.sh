# prune2 for 8 < M <= 16: parity, regressions, then the V = 128 M > 8 workloads
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_gpu_prune.py tests/test_gpu_window16.py 2>&1 | tail -4
for w in llama_prefill_v128_m13 llama_prefill_v128_m9 llama_decode_v128_m13 llama_mlp_m16 llama_decode; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_p2_$w.json 2>/dev/null
done
python scripts/bench_summary.py gpurun_out/r02f_p2_*.json | grep -v "^    "
