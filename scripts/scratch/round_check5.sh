# Full GPU check (round 1d): tests, smoke, bench on every workload, launch lists and ncu captures.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/rc5_tests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/rc5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc5_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/rc5_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/rc5_bench_deit_s.json 2> gpurun_out/rc5_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_mlp_m4 llama_mlp_m5 llama_mlp_m6 llama_mlp_m7 llama_mlp_m8 llama_mlp_m16 toy; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rc5_bench_$w.json 2> gpurun_out/rc5_bench_$w.err; echo "$w exit $?"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rc5_ref.json 2> gpurun_out/rc5_ref.err; echo "ref exit $?"
python scripts/bench_summary.py gpurun_out/rc5_bench_*.json
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rc5_launches_deit_s.csv $C > /dev/null 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc3 -s 5 -c 1 -o gpurun_out/rc5_prof_spmm_deit_s $C > /dev/null 2>&1; echo "ncu full spmm exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune2 -s 3 -c 1 -o gpurun_out/rc5_prof_prune_deit_s $C > /dev/null 2>&1; echo "ncu full prune exit $?"
C="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/rc5_launches_llama_prefill.csv $C > /dev/null 2>&1; echo "ncu launches llama exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 7 -c 1 -o gpurun_out/rc5_prof_spmm_llama_up $C > /dev/null 2>&1; echo "ncu full llama exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune2 -s 7 -c 1 -o gpurun_out/rc5_prof_prune_llama_up $C > /dev/null 2>&1; echo "ncu full prune llama exit $?"
