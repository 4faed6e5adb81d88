timeout 300 python tests/probes/probe4.py 2>&1 | tail -8
