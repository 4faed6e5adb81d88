mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prune.py -m gpu -q --timeout 200 -k "window" > gpurun_out/it_tcp.log 2>&1; echo "tc prune tests exit $?"; tail -3 gpurun_out/it_tcp.log
C1="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
export VNM_TC_CFG=256,1
timeout 300 $C1 > gpurun_out/p_plain1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"vnm_spmm_tc" -s 4 -c 1 -o gpurun_out/prof_tc256_llama_up $C1 > gpurun_out/p_ncu1.log 2>&1; echo "ncu1 $?"
export VNM_TC_CFG=192,1
C2="python bench.py --workload deit_s --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C2 > gpurun_out/p_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prune_pack" -s 12 -c 1 -o gpurun_out/prof_prune_deit $C2 > gpurun_out/p_ncu2.log 2>&1; echo "ncu2 $?"
C3="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C3 > gpurun_out/p_plain3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prune_pack" -s 10 -c 1 -o gpurun_out/prof_prune_llama_up $C3 > gpurun_out/p_ncu3.log 2>&1; echo "ncu3 $?"
