timeout 300 python -m pytest tests/test_gpu_fa.py tests/test_gpu_bwd.py -x -q -k "causal or ragged or many_work or cross_tile or tail or split" 2>&1 | tail -1
for i in 1 2; do
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
TWFA_WORK_LISTS=0 CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed 's/^/nolist /'
done
CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
