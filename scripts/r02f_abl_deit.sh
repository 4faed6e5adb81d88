# DeiT-S window-form kernels, ablations (cold medians): 0 full, 1 no epilogue, 2 no Y stores, 4 no loads, 32 no X^T loads (tc3)
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 0 1 2 4 32; do for sh in "1152 384" "1536 384" "384 1536" "384 384"; do
  VNM_ABL=$abl timeout 120 python scripts/time_spmm.py $sh 5 50432 tc 2>&1 | sed "s/^/abl=$abl /"
done; done
