# ncu --set full of the decode SpMM (Llama up, T=16), the prefill window SpMM (Llama up, T=2048) and the
# prune/compress pass (Llama up weight), each after a plain run exits 0.
mkdir -p gpurun_out
for w in llama_decode llama_prefill; do
  C="python bench.py --workload $w --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
  timeout 300 $C > gpurun_out/pb_$w.json 2> gpurun_out/pb_$w.err || { echo "$w plain FAIL"; tail -5 gpurun_out/pb_$w.err; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/pb_launches_$w.csv $C > /dev/null 2>&1; echo "$w launches $?"
  # second layer (up) of the captured step: skip the warm-up launches (2 eager steps of 3 layers)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 7 -c 1 -o gpurun_out/pb_spmm_$w $C > gpurun_out/pb_ncu_$w.log 2>&1; echo "$w spmm full $?"
done
C="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_pack -s 7 -c 1 -o gpurun_out/pb_prune_llama $C > gpurun_out/pb_ncu_prune.log 2>&1; echo "prune full $?"
C="python bench.py --workload deit_s --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_pack -s 8 -c 1 -o gpurun_out/pb_prune_deit $C > gpurun_out/pb_ncu_prune2.log 2>&1; echo "prune deit full $?"
