# Round 2: every bench workload (builder-run), launch lists and ncu captures of the top kernels
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench_deit_s.json 2> gpurun_out/r02b_bench_deit_s.err; echo "deit_s exit $?"
for w in deit_b llama_prefill llama_decode llama_mlp_m4 llama_mlp_m5 llama_mlp_m6 llama_mlp_m7 llama_mlp_m8 llama_mlp_m16 toy llama_decode_v128_m5 llama_decode_v128_m8 llama_decode_v128_m13 llama_prefill_v128_m5 llama_prefill_v128_m8 llama_prefill_v128_m13 llama_mlp_v128_m4 llama_mlp_v128_m5 llama_mlp_v128_m8 llama_mlp_v128_m16; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_$w.json 2> gpurun_out/r02b_bench_$w.err; echo "$w exit $?"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b_bench_reference_deit_s.json 2> gpurun_out/r02b_ref.err; echo "ref exit $?"
python scripts/bench_summary.py gpurun_out/r02b_bench_*.json > gpurun_out/r02b_bench_summary.txt 2>&1
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02b_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_deit_s.csv $C > /dev/null 2>&1; echo "ncu launches deit exit $?"
C="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02b_plain2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_llama_decode.csv $C > /dev/null 2>&1; echo "ncu launches decode exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_smallt -s 9 -c 1 -o gpurun_out/r02b_prof_smallt_llama_up $C > /dev/null 2>&1; echo "ncu full smallt exit $?"
C="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02b_plain3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02b_launches_llama_prefill.csv $C > /dev/null 2>&1; echo "ncu launches prefill exit $?"
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc3 -s 12 -c 1 -o gpurun_out/r02b_prof_tc3_deit_s $C > /dev/null 2>&1; echo "ncu full tc3 exit $?"
