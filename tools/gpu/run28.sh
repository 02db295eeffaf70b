V=paper_2512_18134_b200/variants
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/poly1000.so $V/poly8.so $V/poly4.so 2>&1
