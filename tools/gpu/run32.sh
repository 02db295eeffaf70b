V=paper_2512_18134_b200/variants
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/notok.so $V/tok.so 2>&1
