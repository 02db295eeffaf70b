V=paper_2512_18134_b200/variants
timeout 600 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so $V/bwdw1.so $V/bwdw2.so
