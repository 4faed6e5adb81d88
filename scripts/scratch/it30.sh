timeout 900 python -m pytest tests/test_gpu_prune.py -m gpu -q -x --timeout 300 > gpurun_out/it30.log 2>&1; echo "prune tests $?"; tail -2 gpurun_out/it30.log
for w in llama_decode deit_s llama_prefill; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it30_$w.json 2>/dev/null; done
python scripts/bench_summary.py gpurun_out/it30_*.json | grep -v "^    "
