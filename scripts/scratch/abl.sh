mkdir -p gpurun_out
python scripts/hbm_write_probe.py
S="python scripts/time_spmm.py"
for shape in "1536 384 5" "384 1536 5"; do set -- $shape
  for abl in 0 1 2 4 8 5 6 7 15; do
    VNM_ABL=$abl VNM_TC_PLAN=1 timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc abl=$abl /"
    VNM_ABL=$abl VNM_TC_PLAN=2 VNM_TC2_NT=192 timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2-192 abl=$abl /"
  done
done
