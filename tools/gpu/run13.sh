SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
