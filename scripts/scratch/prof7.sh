mkdir -p gpurun_out
C="python bench.py --workload deit_s --steps 2 --warmup 3 --no-cpu-baseline --no-baselines"
timeout 300 $C > gpurun_out/p7_plain.json 2> gpurun_out/p7_plain.err && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vnm_spmm_tc" -s 4 -c 1 -o gpurun_out/prof_tc_deit $C > gpurun_out/p7_ncu.log 2>&1; echo "ncu $?"
