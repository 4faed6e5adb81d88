S="python scripts/time_spmm.py"
for shape in "11008 4096" "4096 4096" "4096 11008"; do set -- $shape
  timeout 60 $S $1 $2 5 16 2>&1 | tail -1
  VNM_DEC=1 timeout 60 $S $1 $2 5 16 2>&1 | tail -1 | sed 's/^/  dec /'
done
VNM_SPMM_TRACE=1 timeout 60 $S 11008 4096 5 16 2>&1 | grep -A25 "pair plan" | head -26
