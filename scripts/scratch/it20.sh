S="python scripts/time_spmm.py"
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 > gpurun_out/it20.log 2>&1; echo "spmm tests $?"; tail -2 gpurun_out/it20.log
for shape in "11008 4096" "4096 4096" "4096 11008"; do set -- $shape
  VNM_SPMM_MEMSET=1 timeout 60 $S $1 $2 5 16 2>&1 | tail -1 | sed 's/^/  memset /'
  timeout 60 $S $1 $2 5 16 2>&1 | tail -1 | sed 's/^/  nomemset /'
done
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it20_dec.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it20_dec.json
