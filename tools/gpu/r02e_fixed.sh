# backward: TMA / MMA program unrolled with compile-time op kinds (TWFA_BWD_FIXED=1, default) vs the loop (fixed0)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/fixed0.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/fixed0.so
timeout 300 python tools/bwd_trace_stats.py fa_bwd 2>&1 | head -14
