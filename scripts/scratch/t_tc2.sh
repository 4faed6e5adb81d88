mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x -k "window or prefill or deit or tails or shapes or bf16 or identity or integer or m4" --timeout 120 > gpurun_out/t2_tests.log 2>&1; echo "tests $?"; tail -15 gpurun_out/t2_tests.log
for w in deit_s llama_prefill deit_b llama_mlp_m4 llama_mlp_m8; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t2_$w.json 2> gpurun_out/t2_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t2_$w.err; continue; }
done
python scripts/bench_summary.py gpurun_out/t2_*.json
