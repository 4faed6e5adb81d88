# Round 2 (re-entry, final pass A): GPU tests + smoke, every bench workload, the reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02f_gputests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/r02f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/r02f_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02f_bench_deit_s.json 2> gpurun_out/r02f_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_block_decode llama_mlp_m4 llama_mlp_m5 llama_mlp_m6 llama_mlp_m7 llama_mlp_m8 llama_mlp_m16 toy llama_decode_v128_m5 llama_decode_v128_m8 llama_decode_v128_m9 llama_decode_v128_m10 llama_decode_v128_m11 llama_decode_v128_m13 llama_prefill_v128_m5 llama_prefill_v128_m8 llama_prefill_v128_m9 llama_prefill_v128_m10 llama_prefill_v128_m11 llama_prefill_v128_m13 llama_mlp_v128_m4 llama_mlp_v128_m5 llama_mlp_v128_m8 llama_mlp_v128_m9 llama_mlp_v128_m10 llama_mlp_v128_m11 llama_mlp_v128_m13 llama_mlp_v128_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_$w.json 2> gpurun_out/r02f_bench_$w.err; echo "$w exit $?"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02f_bench_reference_deit_s.json 2> gpurun_out/r02f_ref.err; echo "ref exit $?"
python scripts/bench_summary.py gpurun_out/r02f_bench_*.json > gpurun_out/r02f_bench_summary.txt 2>&1
