V=paper_2512_18134_b200/variants
REPS=2 SCHEDS=fa_fwd,fa_fwd_ring2 timeout 900 python tools/variants.py $V/lean_r2.so 2>&1
