for s in "1536 384 5 50432" "1152 384 5 50432"; do
  echo "E=8"; timeout 120 python scripts/time_spmm.py $s tc
  echo "E=12"; VNM_LIB=paper_2410_16135_b200/libvnm_var_e12.so timeout 120 python scripts/time_spmm.py $s tc
  echo "E=16"; VNM_LIB=paper_2410_16135_b200/libvnm_var_e16.so timeout 120 python scripts/time_spmm.py $s tc
done
VNM_LIB=paper_2410_16135_b200/libvnm_var_e16.so VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1536 384 5 50432 64 tc 2>&1 | grep -A2 "call 3" | tail -1
