L=paper_2410_16135_b200/libvnm_abl.so
for abl in 5 1 0; do
echo "abl $abl"; VNM_LIB=$L VNM_ABL=$abl VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A8 "call 3" | head -8
done
