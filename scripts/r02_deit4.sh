L=paper_2410_16135_b200/libvnm_abl.so
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -x -q --timeout 600 -k "v128 or v32" 2>&1 | tail -2
for abl in 5 0; do
echo "abl $abl"; VNM_LIB=$L VNM_ABL=$abl VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A3 "call 3" | tail -2
done
timeout 300 python tests/probes/probe4.py 2>&1 | tail -2
