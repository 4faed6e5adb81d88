S="python scripts/time_spmm.py"
for shape in "1536 384 5" "1152 384 5"; do set -- $shape
  for nt in 192 224; do for i in 1 2; do VNM_TC3_NT=$nt timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  nt=$nt /"; done; done
done
