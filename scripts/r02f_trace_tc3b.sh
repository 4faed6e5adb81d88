# tc3 MMA-only skeleton (VNM_ABL=5) per-CTA counters under different configurations
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for cfg in "" "VNM_TC3_NT=256" "VNM_TC3_NT=192" "VNM_TC3_S=3" "VNM_TC3_MS=2" "VNM_TC3_OVH=0"; do
  echo "=== $cfg"
  env $cfg VNM_ABL=5 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | grep -A3 "^tc3" | tail -4
done
