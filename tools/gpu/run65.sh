V=paper_2512_18134_b200/variants
timeout 300 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/noxtile.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/noxtile.so 2>&1
