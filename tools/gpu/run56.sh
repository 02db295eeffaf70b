V=paper_2512_18134_b200/variants
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/nospec.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/nospec.so 2>&1
