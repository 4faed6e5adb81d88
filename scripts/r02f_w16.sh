# window-16 form: parity (new tests + window-form regressions), then timing
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_gpu_window16.py 2>&1 | tail -15
timeout 1200 python -m pytest -q -x tests/test_gpu_spmm.py tests/test_gpu_prune.py tests/test_gpu_timed_path.py 2>&1 | tail -3
for sh in "11008 4096" "4096 11008"; do for m in 9 11 13 15; do
  VNM_TS_V=128 timeout 120 python scripts/time_spmm.py $sh $m 2048 tc 2>&1
done; done
for w in llama_prefill_v128_m13 llama_prefill; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_w16_$w.json 2> gpurun_out/r02f_w16_$w.err; python scripts/bench_summary.py gpurun_out/r02f_w16_$w.json
done
