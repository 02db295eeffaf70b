# backward: the fixed production program in its own kernel instantiation (fa_bwd_kernel<true>) vs the generic kernel
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_trace.py -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/nofix.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/nofix.so
for s in fa_bwd_split fa_bwd_cal; do BSCHED=$s timeout 300 python tools/gpu/bwd_time.py $L | sed "s/^/$s /"; done
