for s in "1536 384 5 50432" "1152 384 5 50432"; do
  echo "NT=224"; timeout 120 python scripts/time_spmm.py $s tc
  echo "NT=192"; VNM_TC3_NT=192 timeout 120 python scripts/time_spmm.py $s tc
  echo "NT=224 MS=2"; VNM_TC3_MS=2 timeout 120 python scripts/time_spmm.py $s tc
  echo "NT=192 MS=2"; VNM_TC3_MS=2 VNM_TC3_NT=192 timeout 120 python scripts/time_spmm.py $s tc
done
