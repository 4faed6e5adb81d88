mkdir -p gpurun_out
for cfg in "1 x 0" "2 192 0" "2 256 0" "2 192 1"; do set -- $cfg
  for w in deit_s deit_b; do
    VNM_TC_PLAN=$1 VNM_TC2_NT=$2 VNM_TC2_ARES=$3 timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t12_${w}_$1_$2_$3.json 2>/dev/null || echo "$w $cfg FAIL"
  done
done
python scripts/bench_summary.py gpurun_out/t12_*.json
