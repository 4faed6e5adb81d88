mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py -m gpu -q -x --timeout 200 > gpurun_out/t5_tests.log 2>&1; echo "prune tests $?"; tail -25 gpurun_out/t5_tests.log
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window or any_v or deit or prefill" > gpurun_out/t5_tests2.log 2>&1; echo "spmm tests $?"; tail -5 gpurun_out/t5_tests2.log
for w in deit_s llama_decode; do
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t5_$w.json 2> gpurun_out/t5_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t5_$w.err; continue; }
done
python scripts/bench_summary.py gpurun_out/t5_*.json
C="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune2 -s 7 -c 1 -o gpurun_out/pp3_llama $C > gpurun_out/pp3.log 2>&1; echo "ncu $?"
