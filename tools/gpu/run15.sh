REPS=3 SCHEDS=fa_fwd_tcvl,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/defer.so 2>&1
