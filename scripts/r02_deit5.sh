L=paper_2410_16135_b200/libvnm_abl.so
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_timed_path.py -m gpu -x -q --timeout 600 -k "pair_resident or deit or window_plan or bounds" 2>&1 | tail -2
for ovh in 1 0; do
 for s in "1536 384 5 50432" "1152 384 5 50432"; do echo "ovh=$ovh"; VNM_TC3_OVH=$ovh timeout 120 python scripts/time_spmm.py $s tc; done
 echo "abl 5 ovh=$ovh"; VNM_TC3_OVH=$ovh VNM_LIB=$L VNM_ABL=5 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A2 "call 3" | tail -1
 echo "abl 0 ovh=$ovh"; VNM_TC3_OVH=$ovh VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A2 "call 3" | tail -1
done
