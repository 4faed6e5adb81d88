# Round-1c check of HEAD: GPU tests, smoke, bench on the main workloads.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rc3_build.log 2>&1; echo "build exit $?"
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/rc3_tests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/rc3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc3_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/rc3_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/rc3_bench_deit_s.json 2> gpurun_out/rc3_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rc3_bench_$w.json 2> gpurun_out/rc3_bench_$w.err; echo "$w exit $?"
done
python scripts/bench_summary.py gpurun_out/rc3_bench_*.json
