# backward: TMA / MMA warp program on one elected lane (TWFA_BWD_SOLO=1, default now) vs the whole warp (solo0)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_trace.py -x -q 2>&1 | tail -2
TWFA_LIB=$V/rdld14.so timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/solo0.so $V/rdld14.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/solo0.so $V/rdld14.so
timeout 300 python tools/bwd_trace_stats.py fa_bwd 2>&1 | head -40
