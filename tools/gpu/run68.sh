timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "cross_tile or many_work" 2>&1 | tail -2
