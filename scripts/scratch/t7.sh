mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window or any_v or deit or prefill or toy or bf16 or identity or integer" > gpurun_out/t7_tests.log 2>&1; echo "spmm tests $?"; tail -3 gpurun_out/t7_tests.log
VNM_TC2_NT=256 timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window or any_v or deit" > gpurun_out/t7_tests2.log 2>&1; echo "spmm tests NT=256 $?"; tail -3 gpurun_out/t7_tests2.log
bash scripts/trace_tc2.sh 2>&1 | grep -v "tiles 0 "
for w in deit_s deit_b llama_prefill; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t7_$w.json 2> gpurun_out/t7_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t7_$w.err; continue; }
done
VNM_TC2_NT=192 timeout 200 python bench.py --workload llama_prefill --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t7_llama_prefill_192.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/t7_*.json
