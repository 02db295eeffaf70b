timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so; done
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so
CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwd_eager.so
