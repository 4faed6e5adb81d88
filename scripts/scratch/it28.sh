timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_prune.py -m gpu -q -x --timeout 300 -k "natural or m16 or pair_resident or batched or window" > gpurun_out/it28.log 2>&1; echo "tests $?"; tail -3 gpurun_out/it28.log
timeout 300 python bench.py --workload llama_mlp_m16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it28_m16.json 2>gpurun_out/it28_m16.err; echo "bench $?"; tail -2 gpurun_out/it28_m16.err
python scripts/bench_summary.py gpurun_out/it28_m16.json
