# tc3 per-CTA counters (VNM_SPMM_TRACE=1) for DeiT-S qkv: full kernel and the MMA-only skeleton (ablation build)
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 0 5; do
  echo "=== abl=$abl"
  VNM_ABL=$abl VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | tail -18
done
