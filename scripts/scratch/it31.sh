S="python scripts/time_spmm.py"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_pair -s 3 -c 1 -o gpurun_out/prof_pair_up $S 11008 4096 5 16 > /dev/null 2>&1; echo "ncu $?"
