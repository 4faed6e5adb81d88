mkdir -p gpurun_out
C="python scripts/time_spmm.py 11008 4096 5 16"
timeout 120 $C > gpurun_out/p6_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"vnm_spmm_slab" -s 3 -c 1 -o gpurun_out/prof_slab $C > gpurun_out/p6_ncu.log 2>&1; echo "ncu $?"
