# backward: streamed loads on their own warp (TWFA_BWD_LOAD_WARP=14) vs loads on the MMA warp
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants/bwdld14.so
TWFA_LIB=$V timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V
TWFA_LIB=$V timeout 300 python tools/bwd_trace_stats.py fa_bwd 2>&1 | head -40
