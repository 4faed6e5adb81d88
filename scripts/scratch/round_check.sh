# Full GPU check: gpu tests, smoke, bench on every workload, launch list and ncu captures (DeiT-S default).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/rc_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/rc_tests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/rc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/rc_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/rc_bench_deit_s.json 2> gpurun_out/rc_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_mlp_m4 llama_mlp_m8 llama_mlp_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rc_bench_$w.json 2> gpurun_out/rc_bench_$w.err; echo "$w exit $?"
done
python scripts/bench_summary.py gpurun_out/rc_bench_*.json
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rc_launches_deit_s.csv $C > gpurun_out/rc_ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 8 -c 1 -o gpurun_out/rc_prof_spmm_deit_s $C > gpurun_out/rc_ncu_full.log 2>&1; echo "ncu full exit $?"
