for sh in "11008 4096 5 16" "4096 11008 5 16" "4096 4096 5 16" "11008 4096 5 1" "11008 4096 5 32" "11008 4096 5 64"; do
  timeout 60 python scripts/time_spmm.py $sh
done
