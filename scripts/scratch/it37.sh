S="python scripts/time_spmm.py"
for shape in "384 1536 5" "384 384 5" "768 3072 8" "2304 768 8"; do set -- $shape
  for pf in 0 2 3 4 6; do VNM_TC_PLAN=1 VNM_TC_PF=$pf timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  pf=$pf /"; done
done
