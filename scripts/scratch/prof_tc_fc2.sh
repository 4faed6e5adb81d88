C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc_kernel -s 5 -c 1 -o gpurun_out/rc9_prof_tc_fc2 $C > /dev/null 2>&1; echo "ncu $?"
