set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -c 3000 gpurun_out/g1_bench.json
timeout 300 python tools/trace_stats.py 4 32 8192 > gpurun_out/g1_trace_stats.txt 2>&1; head -40 gpurun_out/g1_trace_stats.txt
