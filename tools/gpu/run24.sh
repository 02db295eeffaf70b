REPS=3 SCHEDS=fa_fwd,fa_fwd_vlcal timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
