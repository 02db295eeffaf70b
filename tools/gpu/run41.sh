V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/whatif1.so $V/whatif2.so $V/whatif3.so 2>&1
