timeout 300 python -m pytest tests/test_gpu_fa.py -x -q -k "causal or ragged or many_work or cross_tile or cudnn" 2>&1 | tail -1
for i in 1 2; do
CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
TWFA_WORK_LISTS=0 CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed 's/^/nolist /'
done
