cp /tmp/old_order.so paper_2512_18134_b200/variants/old_order.so 2>/dev/null
REPS=3 SCHEDS=fa_fwd timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/poly1000.so 2>&1
timeout 600 python -m pytest tests/test_gpu_trace.py -q 2>&1 | tail -1
