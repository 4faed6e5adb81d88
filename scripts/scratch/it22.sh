S="python scripts/time_spmm.py"
for shape in "384 384 5" "384 1536 5" "768 768 8"; do set -- $shape
  for cfg in "128,1" "192,1" "256,1"; do
    VNM_TC_PLAN=1 VNM_TC_CFG=$cfg timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc $cfg /"
  done
done
