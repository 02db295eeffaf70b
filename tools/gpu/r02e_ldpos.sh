# backward fixed program: streamed loads after ST (0, plan order), first (1), before DK (2), last (3)
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
for x in 1 2 3; do TWFA_LIB=$V/ldpos$x.so timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/ldpos1.so $V/ldpos2.so $V/ldpos3.so; done
SHAPE=2,32,16384 CAUSAL=1 timeout 300 python tools/gpu/bwd_time.py $L $V/ldpos1.so $V/ldpos2.so $V/ldpos3.so
