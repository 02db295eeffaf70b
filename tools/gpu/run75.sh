V=paper_2512_18134_b200/variants
TWFA_LIB=$V/pred.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "noncausal or causal_matches or ragged or many_work" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/pred.so 2>&1
