S="python scripts/time_spmm.py"
for shape in "1536 384 5" "1152 384 5"; do set -- $shape
  for pf in 0 1 2 3; do
    VNM_TC3_PF=$pf VNM_TC_PLAN=3 timeout 60 $S $1 $2 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 pf=$pf /"
  done
done
VNM_TC3_PF=1 VNM_TC_PLAN=3 VNM_SPMM_TRACE=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | grep -A3 "tc3 NT" | head -4
