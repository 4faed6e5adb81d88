mkdir -p gpurun_out
C="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune2 -s 7 -c 1 -o gpurun_out/pp2_llama $C > gpurun_out/pp2.log 2>&1; echo "ncu $?"
