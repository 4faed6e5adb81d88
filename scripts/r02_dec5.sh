mkdir -p gpurun_out
timeout 300 python tests/probes/probe_stream.py > gpurun_out/r02f_probe_stream.txt 2>&1; echo "probe $?"; cat gpurun_out/r02f_probe_stream.txt
for abl in 0 1 9 11 15 2 4 8; do
  echo "abl=$abl"; VNM_LIB=paper_2410_16135_b200/libvnm_abl.so VNM_ABL=$abl timeout 120 python scripts/time_spmm.py 11008 4096 5 16
done
