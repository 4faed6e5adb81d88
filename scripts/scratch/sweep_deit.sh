# DeiT-shape SpMM plan comparison: 1-CTA window kernel vs CTA-pair kernel (A resident or streamed), NT.
mkdir -p gpurun_out
S="python scripts/time_spmm.py"
for shape in "1152 384 5" "1536 384 5" "384 1536 5" "384 384 5" "3072 768 8" "768 3072 8"; do
  set -- $shape
  echo "== $1x$2 M=$3"
  VNM_TC_PLAN=1 timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed 's/^/  tc   /'
  for nt in 192 256; do for ares in 0 1; do
    VNM_TC_PLAN=2 VNM_TC2_NT=$nt VNM_TC2_ARES=$ares timeout 120 $S $1 $2 $3 50432 tc 2>&1 | tail -1 | sed "s/^/  tc2 nt=$nt ares=$ares /"
  done; done
done
echo "== traces (1536x384 M=5)"
VNM_TC_PLAN=2 VNM_TC2_NT=192 VNM_SPMM_TRACE=1 timeout 120 $S 1536 384 5 50432 tc 2>&1 | grep -A4 "tc2 NT" | head -6
VNM_TC_PLAN=2 VNM_TC2_NT=256 VNM_SPMM_TRACE=1 timeout 120 $S 1536 384 5 50432 tc 2>&1 | grep -A4 "tc2 NT" | head -6
