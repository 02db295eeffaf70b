timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd_cal >> gpurun_out/trace_c3.txt 2>&1
