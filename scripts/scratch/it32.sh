timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 > gpurun_out/it32.log 2>&1; echo "spmm tests $?"; tail -2 gpurun_out/it32.log
VNM_TC_PLAN=2 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it32b.log 2>&1; echo "tc2 forced $?"; tail -1 gpurun_out/it32b.log
VNM_TC_PLAN=1 timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -k "window_plan or deit_sampled" > gpurun_out/it32c.log 2>&1; echo "tc forced $?"; tail -1 gpurun_out/it32c.log
for w in deit_b llama_mlp_m8; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it32_$w.json 2>/dev/null; done
S="python scripts/time_spmm.py"
for shape in "2304 768" "3072 768" "768 768" "768 3072"; do set -- $shape; timeout 60 $S $1 $2 8 50432 tc 2>&1 | tail -1; done
python scripts/bench_summary.py gpurun_out/it32_*.json | grep -v "^    "
