V=paper_2512_18134_b200/variants
REPS=3 timeout 600 python tools/variants.py $V/base.so $V/probe.so paper_2512_18134_b200/libtwfa.so 2>&1
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 600 python tools/variants.py $V/base.so paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 2>&1 | head -34
