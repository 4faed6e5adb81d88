# tc3 with the specialised MMA loop: skeleton (ablation build), production timing, parity
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 5 261 0; do VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc | sed "s/^/abl=$abl /"; done
unset VNM_LIB
for sh in "1152 384" "1536 384"; do timeout 120 python scripts/time_spmm.py $sh 5 50432 tc | sed "s/^/prod /"; done
timeout 900 python -m pytest -q -x tests/test_gpu_tc3_ts.py tests/test_gpu_timed_path.py tests/test_gpu_spmm.py -k "deit or pair_resident or window or timed or tc3 or bench_step" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_deit_s.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r02h_bench_deit_s.json
