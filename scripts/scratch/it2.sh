S="python scripts/time_spmm.py"
for abl in 0 1 2 4 8; do
  VNM_ABL=$abl VNM_TC_PLAN=1 VNM_TC_CFG=192,1 timeout 120 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc 192 abl=$abl /"
  VNM_ABL=$abl VNM_TC_PLAN=2 VNM_TC2_NT=192 timeout 120 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 192 abl=$abl /"
  VNM_ABL=$abl VNM_TC_PLAN=2 VNM_TC2_NT=256 timeout 120 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 256 abl=$abl /"
done
for nt in 192 256; do
VNM_TC_PLAN=2 VNM_TC2_NT=$nt VNM_SPMM_TRACE=1 timeout 120 $S 1536 384 5 50432 tc 2>&1 | grep -A6 "tc2 NT" | head -8
done
