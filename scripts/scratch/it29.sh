timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_prune.py -m gpu -q -x --timeout 300 -k "natural or m16 or pair_resident" > gpurun_out/it29.log 2>&1; echo "tests $?"; tail -2 gpurun_out/it29.log
timeout 300 python bench.py --workload llama_mlp_m16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it29_m16.json 2>/dev/null; echo "bench $?"
python scripts/bench_summary.py gpurun_out/it29_m16.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/it29_launches.csv python bench.py --workload llama_mlp_m16 --steps 2 --warmup 3 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
