S="python scripts/time_spmm.py"
timeout 60 $S 11008 4096 5 2048 tc 2>&1 | tail -1
VNM_SPMM_TRACE=1 timeout 60 $S 11008 4096 5 2048 tc 2>&1 | grep -A8 "tc2 NT" | head -9
for abl in 1 4 5 15; do VNM_ABL=$abl timeout 60 $S 11008 4096 5 2048 tc 2>&1 | tail -1 | sed "s/^/  abl=$abl /"; done
VNM_TC2_NT=192 timeout 60 $S 11008 4096 5 2048 tc 2>&1 | tail -1 | sed "s/^/  nt192 /"
