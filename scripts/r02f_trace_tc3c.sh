# tc3 MMA-only skeleton: production MMA loop (VNM_ABL=5) vs the probe's minimal loop (VNM_ABL=261)
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 5 261; do
  echo "=== abl=$abl"
  VNM_ABL=$abl VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | grep -A3 "^tc3" | tail -4
  VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc
done
