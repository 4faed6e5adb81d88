# tc3 ablations with the specialised MMA loop (cold / warm): 0 full, 1 no epilogue, 2 no Y stores, 4 no loads, 5 neither
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 0 1 2 4 5; do for sh in "1152 384" "1536 384"; do VNM_ABL=$abl timeout 120 python scripts/time_spmm.py $sh 5 50432 tc | sed "s/^/abl=$abl /"; done; done
VNM_ABL=0 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | grep -A3 "^tc3" | tail -4
