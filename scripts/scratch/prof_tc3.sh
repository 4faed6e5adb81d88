S="python scripts/time_spmm.py"
VNM_TC_PLAN=3 VNM_TC3_NT=224 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc3 -s 3 -c 1 -o gpurun_out/prof_tc3_fc1 $S 1536 384 5 50432 tc > gpurun_out/prof_tc3.log 2>&1; echo "ncu tc3 $?"
VNM_TC_PLAN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc_ -s 3 -c 1 -o gpurun_out/prof_tc_fc1 $S 1536 384 5 50432 tc > gpurun_out/prof_tc.log 2>&1; echo "ncu tc $?"
