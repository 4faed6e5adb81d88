S="python scripts/time_spmm.py"
for shape in "1536 384 5" "1536 1536 5"; do set -- $shape
  for abl in 15 0; do
    for cfg in "128,1" "192,1" "256,1"; do
      VNM_ABL=$abl VNM_TC_PLAN=1 VNM_TC_CFG=$cfg timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc $cfg abl=$abl /"
    done
    for nt in 192 256; do
      VNM_ABL=$abl VNM_TC_PLAN=2 VNM_TC2_NT=$nt timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 $nt abl=$abl /"
    done
  done
done
