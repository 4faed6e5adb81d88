S="python scripts/time_spmm.py"
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 50 > gpurun_out/it4_clk.csv 2>&1 &) 
for nt in 224 192; do for abl in 0 1 2 4 5 15; do
  VNM_ABL=$abl VNM_TC_PLAN=3 VNM_TC3_NT=$nt timeout 60 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc3 $nt abl=$abl /"
done; done
for abl in 0 1 4 5; do VNM_ABL=$abl VNM_TC_PLAN=1 timeout 60 $S 1536 384 5 50432 tc 2>&1 | tail -1 | sed "s/^/  tc abl=$abl /"; done
sleep 1; sort gpurun_out/it4_clk.csv | uniq -c | sort -rn | head -12
