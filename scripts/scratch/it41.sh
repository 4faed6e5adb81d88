S="python scripts/time_spmm.py"
for pf in 0 4 8 12; do
  for shape in "11008 4096" "4096 4096"; do set -- $shape; VNM_PAIR_PF=$pf timeout 60 $S $1 $2 5 16 2>&1 | tail -1 | sed "s/^/  pf=$pf /"; done
  VNM_PAIR_PF=$pf timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it41_dec_$pf.json 2>/dev/null
done
python scripts/bench_summary.py gpurun_out/it41_*.json | grep -v "^    "
