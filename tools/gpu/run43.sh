V=paper_2512_18134_b200/variants
timeout 60 tools/calib/ubench_mmaq
REPS=2 SCHEDS=fa_fwd timeout 900 python tools/variants.py $V/lean.so $V/whatif4.so 2>&1
