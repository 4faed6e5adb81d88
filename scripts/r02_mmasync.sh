timeout 300 python tests/probes/probe_mmasync.py
