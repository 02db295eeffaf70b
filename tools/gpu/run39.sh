timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace39.txt 2>&1
tail -5 gpurun_out/trace39.txt
