bash scripts/trace4.sh | tail -8
for sh in "11008 4096 5 16" "4096 11008 5 16"; do
  timeout 60 python scripts/time_spmm.py $sh
done
