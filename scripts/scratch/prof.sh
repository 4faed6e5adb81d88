mkdir -p gpurun_out
C1="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
C2="python bench.py --workload deit_s --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
C3="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C1 > gpurun_out/p_plain1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 10 -c 1 -o gpurun_out/prof_v2_llama_up $C1 > gpurun_out/p_ncu1.log 2>&1; echo "ncu1 $?"
timeout 300 $C2 > gpurun_out/p_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm -s 12 -c 1 -o gpurun_out/prof_v2_deit_qkv $C2 > gpurun_out/p_ncu2.log 2>&1; echo "ncu2 $?"
timeout 300 $C3 > gpurun_out/p_plain3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"vnm_spmm|prune_pack" -s 20 -c 2 -o gpurun_out/prof_v2_decode $C3 > gpurun_out/p_ncu3.log 2>&1; echo "ncu3 $?"
