# forward knob re-check on the final kernel (C3 sustained, per clock)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
REPS=2 timeout 900 python tools/sustained.py $L $V/TWFA_PROBE_PARTS_0.so $V/TWFA_MEMO_WAITS_0.so $V/TWFA_XTILE_0.so $V/TWFA_PAIR_P_PARTS_4.so
