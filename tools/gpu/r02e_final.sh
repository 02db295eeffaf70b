# re-check after the backward MMA-warp changes: full GPU suite, smoke, default bench line, backward timing
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r02e/pytest_gpu.txt; cat gpurun_out/r02e/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e/smoke.txt 2>&1; tail -2 gpurun_out/r02e/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02e/bench_c5.json 2> gpurun_out/r02e/bench_c5.err; tail -c 1500 gpurun_out/r02e/bench_c5.json
timeout 300 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
