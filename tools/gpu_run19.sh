timeout 120 python tools/tc_sparse_probe.py 2>&1 | tail -5
