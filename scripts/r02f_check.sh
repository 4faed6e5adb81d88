# Round 2 (re-entry): HEAD check — GPU tests, smoke, default bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/r02f_gputests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/r02f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/r02f_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02f_bench_deit_s.json 2> gpurun_out/r02f_bench_deit_s.err; echo "deit_s exit $?"
python scripts/bench_summary.py gpurun_out/r02f_bench_*.json
