mkdir -p gpurun_out
L=paper_2410_16135_b200/libvnm_abl.so
for s in "1536 384 5 50432" "1152 384 5 50432"; do
  for abl in 0 1 2 4 5 32; do
    echo "abl=$abl $s"; VNM_LIB=$L VNM_ABL=$abl timeout 120 python scripts/time_spmm.py $s tc
  done
  echo "NT=256"; VNM_TC3_NT=256 timeout 120 python scripts/time_spmm.py $s tc
done
for s in "384 1536 5 50432" "384 384 5 50432"; do timeout 120 python scripts/time_spmm.py $s tc; done
VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A20 "call 3" | head -20
