timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "decode or slab or token_tails or config1 or determinism" > gpurun_out/it40.log 2>&1; echo "tests $?"; tail -1 gpurun_out/it40.log
S="python scripts/time_spmm.py"
for shape in "11008 4096" "4096 4096" "4096 11008"; do set -- $shape; timeout 60 $S $1 $2 5 16 2>&1 | tail -1; done
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it40_dec.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it40_dec.json
