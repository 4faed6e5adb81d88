# Round 2: new small-T plan (spmm_smallt.cu): parity + timing vs the previous plan
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -x -q --timeout 600 -k "smallt or slab or decode or workspace or pdl or chained or binding or previous or toy or token_tails" > gpurun_out/r02b_tests.log 2>&1; echo "tests exit $?"; tail -15 gpurun_out/r02b_tests.log
for s in "11008 4096 5 16" "4096 11008 5 16" "4096 4096 5 16" "11008 4096 5 1" "11008 4096 5 8" "11008 4096 5 32"; do
  timeout 120 python scripts/time_spmm.py $s >> gpurun_out/r02b_time.txt 2>&1
  VNM_SMALLT=0 timeout 120 python scripts/time_spmm.py $s >> gpurun_out/r02b_time_old.txt 2>&1
done
for s in "11008 4096 8 16" "11008 4096 13 16"; do VNM_TS_V=128 timeout 120 python scripts/time_spmm.py $s >> gpurun_out/r02b_time.txt 2>&1; done
echo NEW; cat gpurun_out/r02b_time.txt; echo OLD; cat gpurun_out/r02b_time_old.txt
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_llama_decode.json 2> gpurun_out/r02b_bench_llama_decode.err; echo "decode bench exit $?"
python -c "import json;d=json.load(open('gpurun_out/r02b_bench_llama_decode.json'));print(d['ms_per_step'],d['roofline'],d['detail']['layers'])"
