V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly16.so $V/poly8.so $V/poly4.so $V/parts2.so $V/parts8.so 2>&1
