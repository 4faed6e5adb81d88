# Round 2 (final pass B): launch lists + ncu --set full of the top kernels (each after its plain run exits 0)
mkdir -p gpurun_out
C="python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02c_plain1.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_deit_s.csv $C > /dev/null 2>&1; echo "launches deit_s exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_tc3 -s 13 -c 1 -o gpurun_out/r02c_prof_tc3_deit_s $C > /dev/null 2>&1; echo "full tc3 exit $?"
C="python bench.py --workload llama_decode --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02c_plain2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_llama_decode.csv $C > /dev/null 2>&1; echo "launches decode exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vnm_spmm_smallt -s 10 -c 1 -o gpurun_out/r02c_prof_smallt_llama_up $C > /dev/null 2>&1; echo "full smallt exit $?"
C="python bench.py --workload llama_prefill --steps 2 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $C > gpurun_out/r02c_plain3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02c_launches_llama_prefill.csv $C > /dev/null 2>&1; echo "launches prefill exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune2 -s 3 -c 1 -o gpurun_out/r02c_prof_prune_llama $C > /dev/null 2>&1; echo "full prune exit $?"
