# CTA-pair forward vs single-CTA forward: parity tests, then interleaved timing (C3, C4)
timeout 600 python -m pytest tests/test_gpu_fa.py -x -q 2>&1 | tail -5
for P in 1 0 1 0; do TWFA_PAIR=$P timeout 120 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed "s/^/pair=$P /"; done
for P in 1 0; do TWFA_PAIR=$P SHAPE=2,32,16384 CAUSAL=1 timeout 120 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1 | sed "s/^/C4 pair=$P /"; done
