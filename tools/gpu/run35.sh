timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_stats.py 2 32 16384 fa_fwd 1 > gpurun_out/trace_c4.txt 2>&1
