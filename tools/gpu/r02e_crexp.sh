# correction warps compute the last 32-key chunk of P (TWFA_CR_EXP=1) vs default
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants/crexp.so
TWFA_LIB=$V timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "oracle and not random" 2>&1 | tail -3
TWFA_LIB=$V timeout 600 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -3
REPS=3 timeout 600 python tools/sustained.py $L $V
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V
TWFA_PAIR=0 REPS=2 timeout 400 python tools/sustained.py $L $V | sed "s/^/pair=0 /"
