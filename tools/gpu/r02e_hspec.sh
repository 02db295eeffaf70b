# forward spec kernels: softmax warps run [MX_k, EX_k] with compile-time kinds and no generic loop (TWFA_HEAVY_SPEC=1)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 900 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -q > gpurun_out/hs_tests.txt 2>&1; tail -1 gpurun_out/hs_tests.txt
REPS=3 timeout 600 python tools/sustained.py $L $V/hs0.so
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V/hs0.so | sed "s/^/C4 /"
TWFA_PAIR=0 REPS=2 timeout 400 python tools/sustained.py $L $V/hs0.so | sed "s/^/pair0 /"
