timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
V=paper_2512_18134_b200/variants
SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py $V/poly1000.so $V/poly8.so $V/poly4.so $V/poly2.so 2>&1
