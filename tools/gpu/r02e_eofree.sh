# forward: the epilogue releases O_k for the next tile's PV_k(0) right after reading it (TWFA_EARLY_OFREE=1) vs after CR(0)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 900 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
timeout 300 python tools/gpu/tile_boundary_cost.py
TWFA_LIB=$V/eof0.so timeout 300 python tools/gpu/tile_boundary_cost.py | sed "s/^/eof0 /"
REPS=2 timeout 600 python tools/sustained.py $L $V/eof0.so
SHAPE=16,64,1024 REPS=2 timeout 400 python tools/sustained.py $L $V/eof0.so | sed "s/^/S=1K /"
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V/eof0.so | sed "s/^/C4 /"
