# Round 2 (re-entry, HEAD after prune2 LEAN = 2): GPU suite, smoke, the default bench and a few workloads
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02k_gputests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/r02k_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/r02k_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02k_bench_deit_s.json 2> gpurun_out/r02k_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_prefill_v128_m13 llama_mlp_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench_$w.json 2> gpurun_out/r02k_bench_$w.err; echo "$w exit $?"
done
python scripts/bench_summary.py gpurun_out/r02k_bench_*.json > gpurun_out/r02k_bench_summary.txt 2>&1; grep -v "^    " gpurun_out/r02k_bench_summary.txt
