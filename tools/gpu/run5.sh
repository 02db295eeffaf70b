export TWFA_LIB=paper_2512_18134_b200/variants/poly1000.so
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_fa2.txt 2>&1
