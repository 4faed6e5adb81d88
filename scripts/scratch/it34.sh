timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 > gpurun_out/it34.log 2>&1; echo "spmm tests $?"; tail -1 gpurun_out/it34.log
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it34_deit_s_$i.json 2>/dev/null; done
VNM_TC_CFG=192,1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it34_deit_s_old.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it34_*.json
