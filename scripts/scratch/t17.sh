mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_ria.py -m gpu -q -x --timeout 300 > gpurun_out/t17_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/t17_tests.log
timeout 200 python bench.py --workload deit_s --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t17_deit_s.json 2>/dev/null
timeout 200 python bench.py --workload deit_b --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t17_deit_b.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/t17_*.json
bash scripts/trace_prune.sh
