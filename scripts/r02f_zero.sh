# tc3 MMA-only skeleton (VNM_ABL=5) with real vs zero weights (zero W: A values 0, uniform metadata) and the full kernel
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 5 0; do for z in "" w x xw; do
  VNM_TS_ZERO=$z VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 1152 384 5 50432 tc 2>&1 | sed "s/^/abl=$abl zero=$z /"
done; done
