# DeiT-B (64:2:8) layers through each window-form kernel (cold medians): 1 tc, 2 tc2, 3 tc3 resident, 4 tc3 streamed
for plan in 1 2 3 4; do for sh in "2304 768" "3072 768" "768 3072" "768 768"; do
  VNM_TC_PLAN=$plan timeout 120 python scripts/time_spmm.py $sh 8 50432 tc 2>&1 | sed "s/^/plan=$plan /"
done; done
