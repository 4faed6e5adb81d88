mkdir -p gpurun_out
timeout 120 python tests/probe3.py > gpurun_out/probe3.log 2>&1; echo "probe3 $?"; cat gpurun_out/probe3.log | tail -20
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x -k "window or prefill or deit or tails or shapes or bf16 or identity or integer or m4" --timeout 120 > gpurun_out/t3_tests.log 2>&1; echo "tests $?"; tail -15 gpurun_out/t3_tests.log
for w in deit_s deit_b llama_prefill; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t3_$w.json 2> gpurun_out/t3_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t3_$w.err; continue; }
done
VNM_TC2_ARES=0 timeout 200 python bench.py --workload deit_s --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t3_deit_s_nores.json 2> /dev/null
python scripts/bench_summary.py gpurun_out/t3_*.json
