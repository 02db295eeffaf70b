# backward MMA warp: memoized waits (default) vs every wait (memo0) vs + loads on warp 14
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_trace.py -x -q 2>&1 | tail -2
TWFA_LIB=$V/bwdld14.so timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/memo0.so $V/bwdld14.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/memo0.so $V/bwdld14.so
timeout 300 python tools/bwd_trace_stats.py fa_bwd 2>&1 | head -40
