V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly2.so $V/poly4.so $V/poly8.so 2>&1
REPS=2 SCHEDS=fa_fwd_fixedtc:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly4.so 2>&1
