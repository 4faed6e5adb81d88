mkdir -p gpurun_out
C3="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C3 > gpurun_out/p_plain3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"vnm_spmm_kernel" -s 10 -c 1 -o gpurun_out/prof_dec_up $C3 > gpurun_out/p_ncu3.log 2>&1; echo "ncu3 $?"
C1="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C1 > gpurun_out/p_plain1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prune_pack" -s 10 -c 1 -o gpurun_out/prof_prune_tc_up $C1 > gpurun_out/p_ncu1.log 2>&1; echo "ncu1 $?"
