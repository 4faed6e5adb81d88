L=paper_2410_16135_b200/libvnm_abl.so
for S in 3 4 5; do
echo "abl 5 S=$S"; VNM_TC3_S=$S VNM_LIB=$L VNM_ABL=5 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A3 "call 3" | tail -2
done
echo "abl 5 M=8 (no peek)"; VNM_TC_PLAN=3 VNM_LIB=$L VNM_ABL=5 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 8 50432 64 tc 2>&1 | grep -A3 "call 3" | tail -2
echo "abl 5 M=4"; VNM_TC_PLAN=3 VNM_LIB=$L VNM_ABL=5 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 4 50432 64 tc 2>&1 | grep -A3 "call 3" | tail -2
