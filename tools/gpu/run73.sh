V=paper_2512_18134_b200/variants
timeout 200 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/rd_old.so paper_2512_18134_b200/libtwfa.so $V/rd_old.so
BSCHED=fa_bwd_split timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/rd_old.so
