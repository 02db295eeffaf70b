V=paper_2512_18134_b200/variants
TWFA_LIB=$V/eager.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "noncausal or causal_matches or many_work" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/eager.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/eager.so 2>&1
