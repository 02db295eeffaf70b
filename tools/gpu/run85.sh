for MB in 16 32 48 96; do
TWFA_WL_GROUP_MB=$MB CAUSAL=1 SHAPE=2,32,16384 SCHEDS=fa_fwd timeout 300 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed "s/^/fwd MB=$MB /"
TWFA_WL_GROUP_MB=$MB CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/bwd MB=$MB /"
done
