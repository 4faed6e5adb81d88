S="python scripts/time_spmm.py"
VNM_TC_PLAN=3 VNM_TC3_NT=224 VNM_SPMM_TRACE=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | grep -A4 "tc3 NT" | head -6
VNM_ABL=4 VNM_TC_PLAN=3 VNM_TC3_NT=224 VNM_SPMM_TRACE=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | grep -A4 "tc3 NT" | head -6
