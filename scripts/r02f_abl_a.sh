# tc3: does reading A at 32-byte offsets inside the SW128 atom slow the MMAs?  (ablation build; cold medians)
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 0 128 64 5 133 69; do for sh in "1152 384" "1536 384"; do
  VNM_ABL=$abl timeout 120 python scripts/time_spmm.py $sh 5 50432 tc 2>&1 | sed "s/^/abl=$abl /"
done; done
