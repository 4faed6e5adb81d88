mkdir -p gpurun_out
C="python scripts/time_spmm.py 11008 4096 5 16"
timeout 120 $C && timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_smallt -s 25 -c 1 -o gpurun_out/r02j_prof_smallt_up $C > gpurun_out/r02j_ncu.log 2>&1; echo "ncu exit $?"
