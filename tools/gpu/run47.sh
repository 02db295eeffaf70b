V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/parts4.so $V/parts8.so 2>&1
REPS=1 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/parts4.so $V/parts8.so 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
