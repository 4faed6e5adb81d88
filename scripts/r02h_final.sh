# Round 2 (re-entry, final): GPU suite, smoke, every bench workload after the MMA-loop change
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02h_gputests.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/r02h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/r02h_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02h_bench_deit_s.json 2> gpurun_out/r02h_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_block_decode llama_mlp_m4 llama_mlp_m5 llama_mlp_m6 llama_mlp_m7 llama_mlp_m8 llama_mlp_m16 toy llama_decode_v128_m5 llama_decode_v128_m8 llama_decode_v128_m9 llama_decode_v128_m10 llama_decode_v128_m11 llama_decode_v128_m13 llama_prefill_v128_m5 llama_prefill_v128_m8 llama_prefill_v128_m9 llama_prefill_v128_m10 llama_prefill_v128_m11 llama_prefill_v128_m13 llama_mlp_v128_m4 llama_mlp_v128_m5 llama_mlp_v128_m8 llama_mlp_v128_m9 llama_mlp_v128_m10 llama_mlp_v128_m11 llama_mlp_v128_m13 llama_mlp_v128_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_$w.json 2> gpurun_out/r02h_bench_$w.err; echo "$w exit $?"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02h_bench_reference_deit_s.json 2> gpurun_out/r02h_ref.err; echo "ref exit $?"
python scripts/bench_summary.py gpurun_out/r02h_bench_*.json > gpurun_out/r02h_bench_summary.txt 2>&1
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02h_plain1.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches_deit_s.csv $C > /dev/null 2>&1; echo "launches deit_s exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc3 -s 13 -c 1 -o gpurun_out/r02h_prof_tc3_deit_s $C > /dev/null 2>&1; echo "full tc3 exit $?"
