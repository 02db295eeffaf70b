timeout 120 python tools/gpu/bwd_time.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwdw2.so paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/bwdw2.so
