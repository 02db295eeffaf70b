V=paper_2512_18134_b200/variants
SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/poly8.so $V/poly4.so $V/poly2.so 2>&1
