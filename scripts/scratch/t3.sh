bash scripts/trace4.sh 2>&1 | head -10
timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x -k "slab or decode or toy or tails" --timeout 100 2>&1 | tail -2
for sh in "11008 4096 5 16" "4096 11008 5 16" "11008 4096 5 1" "11008 4096 5 32"; do
  timeout 60 python scripts/time_spmm.py $sh
done
