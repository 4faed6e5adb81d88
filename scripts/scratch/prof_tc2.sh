mkdir -p gpurun_out
for w in llama_prefill deit_s; do
  C="python bench.py --workload $w --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
  timeout 300 $C > gpurun_out/p2_$w.json 2> gpurun_out/p2_$w.err || { echo "$w plain FAIL"; tail -5 gpurun_out/p2_$w.err; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 7 -c 1 -o gpurun_out/p2_spmm_$w $C > gpurun_out/p2_ncu_$w.log 2>&1; echo "$w spmm full $?"
done
