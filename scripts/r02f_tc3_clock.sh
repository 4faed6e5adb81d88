# tc3 with the MMA loop's clock reads only under tracing: skeleton (ablation build) and the production kernel
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 5 261 0; do VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc | sed "s/^/abl=$abl /"; done
unset VNM_LIB
for sh in "1152 384" "1536 384"; do timeout 120 python scripts/time_spmm.py $sh 5 50432 tc | sed "s/^/prod /"; done
