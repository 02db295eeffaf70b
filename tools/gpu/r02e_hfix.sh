# forward: softmax warps run [MX_k, EX_k] with compile-time kinds (TWFA_HEAVY_FIXED=1, default) vs the loop
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
REPS=3 timeout 600 python tools/sustained.py $L $V/hfix0.so
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V/hfix0.so
