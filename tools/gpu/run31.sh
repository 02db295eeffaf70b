REPS=3 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/snake.so 2>&1
