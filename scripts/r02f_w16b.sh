# window-16 form: parity, then the V = 128 MLP M-sweep (T = 2048) and prefill workloads
mkdir -p gpurun_out
timeout 1200 python -m pytest -q tests/test_gpu_window16.py 2>&1 | tail -3
for m in 4 5 8 9 10 11 13 16; do
  timeout 300 python bench.py --workload llama_mlp_v128_m$m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_llama_mlp_v128_m$m.json 2>/dev/null
done
for m in 9 10 11 13; do
  timeout 300 python bench.py --workload llama_prefill_v128_m$m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_llama_prefill_v128_m$m.json 2>/dev/null
done
python scripts/bench_summary.py gpurun_out/r02f_bench_llama_*v128*.json
