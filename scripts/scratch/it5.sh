S="python scripts/time_spmm.py"
for T in 8192 50432; do for abl in 0 1; do
  VNM_ABL=$abl VNM_TC_PLAN=3 VNM_TC3_NT=224 timeout 60 $S 1536 384 5 $T tc 2>&1 | tail -1 | sed "s/^/  tc3 abl=$abl /"
  VNM_ABL=$abl VNM_TC_PLAN=1 timeout 60 $S 1536 384 5 $T tc 2>&1 | tail -1 | sed "s/^/  tc  abl=$abl /"
done; done
for s in 3 4; do VNM_TC3_S=$s VNM_TC_PLAN=3 VNM_TC3_NT=224 timeout 60 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 S=$s /"; done
