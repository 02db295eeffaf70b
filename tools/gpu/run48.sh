timeout 300 python tools/gpu/bwd_check.py 2>&1 | tail -20
