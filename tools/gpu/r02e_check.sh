# end-of-round re-check of the committed state (after the C4 leg and the tiny-length test), plus backward traces
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r02e/pytest_gpu.txt; cat gpurun_out/r02e/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e/smoke.txt 2>&1; tail -2 gpurun_out/r02e/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e/bench_c5.json 2> gpurun_out/r02e/bench_c5.err; tail -c 600 gpurun_out/r02e/bench_c5.json
timeout 300 python tools/bwd_trace_stats.py fa_bwd > gpurun_out/r02e/bwd_trace_fa_bwd.txt 2>&1; head -40 gpurun_out/r02e/bwd_trace_fa_bwd.txt
