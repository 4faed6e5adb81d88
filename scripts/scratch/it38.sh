S="python scripts/time_spmm.py"
for shape in "768 3072 8" "384 1536 5"; do set -- $shape
  for pf in 0 2 3 4; do VNM_TC_PLAN=2 VNM_TC_PF=$pf timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 pf=$pf /"; done
done
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "deit or window or prefill" > gpurun_out/it38.log 2>&1; echo "tests $?"; tail -1 gpurun_out/it38.log
for w in deit_b deit_s; do for pf in 0 3; do VNM_TC_PF=$pf timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it38_${w}_$pf.json 2>/dev/null; done; done
python scripts/bench_summary.py gpurun_out/it38_*.json | grep -v "^    "
