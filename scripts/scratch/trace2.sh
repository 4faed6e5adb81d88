bash scripts/trace.sh > /dev/null 2>&1
for d in 0 1 2 3; do echo "dbg $d"; VNM_SPMM_DBG=$d python /tmp/tr.py 16 2>&1 | sed -n 10,14p; done
