mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -x -q --timeout 600 -k "smallt or slab or decode or workspace or pdl or chained or toy or token_tails" > gpurun_out/r02h_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/r02h_tests.log
VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 11008 4096 5 16 2>&1 | grep smallt
for s in "11008 4096 5 16" "4096 11008 5 16" "4096 4096 5 16" "11008 4096 5 1" "11008 4096 5 32"; do
  timeout 120 python scripts/time_spmm.py $s
done
for abl in 1 15; do
  echo "abl=$abl"; VNM_LIB=paper_2410_16135_b200/libvnm_abl.so VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 11008 4096 5 16
done
