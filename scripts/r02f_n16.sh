# natural 2:4 form at M = 16 written by prune2: parity + the M = 16 workloads
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_gpu_prune.py tests/test_gpu_window16.py tests/test_gpu_spmm.py -k "natural or m16 or window16 or prune2 or batched or m9" 2>&1 | tail -3
for w in llama_mlp_m16 llama_mlp_v128_m16 llama_mlp_m5; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_n16_$w.json 2>/dev/null
done
python scripts/bench_summary.py gpurun_out/r02f_n16_*.json | grep -v "^    "
