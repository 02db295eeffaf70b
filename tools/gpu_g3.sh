timeout 900 python -m pytest tests/test_gpu_fa.py -x -q 2>&1 | tail -15
timeout 300 python tools/gpu/observed_errors.py 2>&1 | tail -5
timeout 120 ./tools/calib/ubench_handoff 2>&1 | tail -8
