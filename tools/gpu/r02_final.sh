# round 2 final evidence: tests, smoke, default bench line, reference arm, launch list, ncu, sanitizer
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 400 gpurun_out/bench_c5.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_arm.json 2>&1; tail -c 300 gpurun_out/reference_arm.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_fwd|gemm" -c 10 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-legs > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_final python tools/prof_run.py fa 2 > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log
timeout 900 ncu --set full --clock-control none -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c5_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline --skip-legs > gpurun_out/ncu_c5.log 2>&1; tail -1 gpurun_out/ncu_c5.log
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.txt 2>&1; tail -3 gpurun_out/sanitizer_memcheck.txt
