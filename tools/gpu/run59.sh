timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so
