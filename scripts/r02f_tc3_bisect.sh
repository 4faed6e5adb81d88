# bisecting the tc3 MMA loop: the probe-like loop (abl 261) plus one production feature at a time
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 261 773 1285 2309 3845 5; do VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc | sed "s/^/abl=$abl /"; done
