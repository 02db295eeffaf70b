V=paper_2512_18134_b200/variants
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdred.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdred.so
TWFA_LIB=$V/bwdred.so timeout 120 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
