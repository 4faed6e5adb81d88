S="python scripts/time_spmm.py"
for abl in 0 1 4 16 32 17 33; do VNM_ABL=$abl VNM_TC_PLAN=4 timeout 60 $S 11008 4096 5 2048 tc 2>&1 | tail -1 | sed "s/^/  stream abl=$abl /"; done
