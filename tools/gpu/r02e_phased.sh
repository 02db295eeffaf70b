# phased chunk (all FFMA2 arguments before the MUFU ops) vs default, C3 sustained, interleaved
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
TWFA_LIB=$V/phased.so timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "oracle" 2>&1 | tail -2
REPS=3 timeout 600 python tools/sustained.py $L $V/phased.so
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V/phased.so
