mkdir -p gpurun_out
VNM_TC2_STG=1 timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window or any_v or deit or bf16" > gpurun_out/t8_tests.log 2>&1; echo "spmm tests stg $?"; tail -3 gpurun_out/t8_tests.log
for stg in 0 1; do for w in deit_s deit_b; do
  VNM_TC2_STG=$stg timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t8_${w}_stg$stg.json 2> gpurun_out/t8_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/t8_$w.err; continue; }
done; done
VNM_TC_PLAN=1 timeout 200 python bench.py --workload deit_s --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t8_deit_s_1cta.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/t8_*.json
