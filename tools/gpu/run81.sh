timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
for B in fa_bwd fa_bwd_qstage fa_bwd_split; do BSCHED=$B timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/$B /"; done
for B in fa_bwd fa_bwd_qstage; do BSCHED=$B CAUSAL=1 SHAPE=2,32,16384 timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so | sed "s/^/$B /"; done
