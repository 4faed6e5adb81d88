# tc2 ablations on Llama up / down prefill (T = 2048, 64:2:5): full / no A loads / no Y stores / no loads
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_abl.so
for abl in 0 16 2 18 4; do for sh in "11008 4096" "4096 11008"; do
  VNM_ABL=$abl timeout 120 python scripts/time_spmm.py $sh 5 2048 tc 2>&1 | sed "s/^/abl=$abl /"
done; done
