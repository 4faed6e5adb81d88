export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 5 261 1029; do VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc | sed "s/^/abl=$abl /"; done
