mkdir -p gpurun_out
for abl in 0 15 11 4; do
  VNM_LIB=paper_2410_16135_b200/libvnm_abl.so VNM_ABL=$abl VNM_SPMM_TRACE=2 timeout 120 python scripts/trace_spmm.py 11008 4096 5 16 > gpurun_out/r02i_trace_abl$abl.txt 2>&1
  echo "abl $abl"; grep -A6 "call 3" gpurun_out/r02i_trace_abl$abl.txt | cut -c1-420
done
