# producer / epilogue counters of tc3 with the specialised MMA loop (experiment build), DeiT-S qkv
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_tf.so
VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | grep -A4 "^tc3" | tail -5
