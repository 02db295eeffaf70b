timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/calibrate.py > gpurun_out/calibration.json 2>gpurun_out/calibration.err; tail -3 gpurun_out/calibration.err; cat gpurun_out/calibration.json
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd 2>&1 | tail -20
