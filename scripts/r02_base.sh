# Round 2 baseline: decode bench, ncu of the small-T (pair) decode kernel on Llama up T=16.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt 2>&1
C="python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02a_bench_llama_decode.json 2> gpurun_out/r02a_bench_llama_decode.err; echo "decode bench exit $?"
for s in "11008 4096 5 16" "4096 11008 5 16" "4096 4096 5 16" "11008 4096 5 1" "11008 4096 5 8"; do
  timeout 120 python scripts/time_spmm.py $s >> gpurun_out/r02a_time.txt 2>&1
done
cat gpurun_out/r02a_time.txt
C="python scripts/time_spmm.py 11008 4096 5 16"
timeout 120 $C > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_pair -s 25 -c 1 -o gpurun_out/r02a_prof_pair_up $C > gpurun_out/r02a_ncu.log 2>&1; echo "ncu exit $?"
