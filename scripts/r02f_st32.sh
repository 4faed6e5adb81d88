# tc3 epilogue: 256-bit direct stores (VNM_TC3_ST32=1, default) vs the transpose-slot path
mkdir -p gpurun_out
for st in 0 1; do for sh in "1152 384" "1536 384"; do
  VNM_TC3_ST32=$st timeout 120 python scripts/time_spmm.py $sh 5 50432 tc 2>&1 | sed "s/^/st32=$st /"
done; done
for st in 0 1; do VNM_TC3_ST32=$st timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/r02f_st32_$st.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r02f_st32_$st.json; done
timeout 900 python -m pytest -q -x tests/test_gpu_timed_path.py tests/test_gpu_spmm.py -k "deit or pair_resident or window or timed or bench_step" 2>&1 | tail -3
