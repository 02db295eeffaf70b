timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_bwd_kernel -c 1 -f -o gpurun_out/bwd_c3_full python tools/prof_run.py bwd 2 > gpurun_out/ncu_bwd.log 2>&1; tail -2 gpurun_out/ncu_bwd.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_bwd.csv python tools/prof_run.py bwd 3 > /dev/null 2>&1
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_c4.json
