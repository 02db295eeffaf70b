V=paper_2512_18134_b200/variants
TWFA_LIB=$V/shalves.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "not split and not double and not interpreter and not pybind and not host_tool" 2>&1 | tail -1
REPS=3 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/shalves.so 2>&1
REPS=2 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so $V/shalves.so 2>&1
