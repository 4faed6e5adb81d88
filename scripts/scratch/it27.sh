timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_prune.py -m gpu -q -x --timeout 300 > gpurun_out/it27.log 2>&1; echo "tests $?"; tail -2 gpurun_out/it27.log
for pdl in 0 1; do
  VNM_PDL=$pdl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it27_deit_s_$pdl.json 2>/dev/null
  VNM_PDL=$pdl timeout 300 python bench.py --workload llama_prefill --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it27_llama_$pdl.json 2>/dev/null
  VNM_PDL=$pdl timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it27_dec_$pdl.json 2>/dev/null
done
python scripts/bench_summary.py gpurun_out/it27_*.json | grep -v "^    "
