S="python scripts/time_spmm.py"
for shape in "2304 768 8" "3072 768 8" "768 768 8"; do set -- $shape
  timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  default /"
  VNM_TC_PLAN=3 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 ms2 /"
  VNM_TC_PLAN=3 VNM_TC3_MS=4 timeout 60 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 ms4 /"
done
