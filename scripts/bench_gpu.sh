mkdir -p gpurun_out
B="python bench.py"
timeout 600 $B --steps 10 --warmup 3 > gpurun_out/bench_deit_s.json 2> gpurun_out/bench_deit_s.err; echo "deit_s exit $?"
tail -c 3000 gpurun_out/bench_deit_s.json; tail -3 gpurun_out/bench_deit_s.err
for w in llama_prefill llama_decode deit_b; do
  timeout 300 $B --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w exit $?"
  tail -c 1500 gpurun_out/bench_$w.json; tail -2 gpurun_out/bench_$w.err
done
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_deit_s.csv $C > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 12 -c 1 -o gpurun_out/prof_spmm_deit_s $C > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_pack -s 12 -c 1 -o gpurun_out/prof_prune_deit_s $C > gpurun_out/ncu_full_prune.log 2>&1; echo "ncu full prune exit $?"
