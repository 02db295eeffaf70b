# backward: streamed loads deferred to just before DP (15) / DK (19) / DQ (20) on the MMA warp
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
for x in ldk ldq; do TWFA_LIB=$V/$x.so timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/ldp.so $V/ldk.so $V/ldq.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/ldk.so $V/ldq.so
