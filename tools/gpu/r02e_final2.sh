# final state: full GPU suite (incl. the shape fuzz), smoke, default bench line, reference arm, launch list
mkdir -p gpurun_out/r02e
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r02e/pytest_gpu.txt; cat gpurun_out/r02e/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e/smoke.txt 2>&1; tail -2 gpurun_out/r02e/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e/bench_c5.json 2> gpurun_out/r02e/bench_c5.err; tail -c 300 gpurun_out/r02e/bench_c5.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e/reference_arm.json 2>&1; tail -c 300 gpurun_out/r02e/reference_arm.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_fwd|gemm" -c 10 --csv --log-file gpurun_out/r02e/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-legs > gpurun_out/r02e/ncu_launch.log 2>&1; tail -3 gpurun_out/r02e/launches_c5.csv
