S="python scripts/time_spmm.py"
for shape in "384 1536 5" "384 384 5" "768 3072 8" "768 768 8" "2304 768 8" "3072 768 8"; do set -- $shape
  timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  default /"
  for nt in 224 256; do
    VNM_TC3_NT=$nt VNM_TC_PLAN=4 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  stream $nt /"
    VNM_TC3_NT=$nt VNM_TC_PLAN=3 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  res-if-fits $nt /"
  done
done
