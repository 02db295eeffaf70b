REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/solo.so 2>&1
