S="python scripts/time_spmm.py"
for shape in "1536 384 5" "1536 1536 5"; do set -- $shape
  for z in "" x w xw; do
    VNM_TS_ZERO=$z VNM_ABL=0 VNM_TC_PLAN=1 VNM_TC_CFG=256,1 timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc 256 zero=$z abl=0 /"
    VNM_TS_ZERO=$z VNM_ABL=15 VNM_TC_PLAN=1 VNM_TC_CFG=256,1 timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc 256 zero=$z abl=15 /"
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_throttle_reasons.active --format=csv
