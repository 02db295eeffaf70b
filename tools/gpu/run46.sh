V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd,fa_fwd_split timeout 900 python tools/variants.py $V/lean_split.so 2>&1
