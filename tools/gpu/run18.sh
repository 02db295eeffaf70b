timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
REPS=2 SCHEDS=fa_fwd,fa_fwd_fixedtc,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
