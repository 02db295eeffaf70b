timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
REPS=3 SCHEDS=fa_fwd,fa_fwd_vl,fa_fwd_cal timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/realized_gantt.py fa_fwd gpurun_out/realized_fa_fwd 2>&1 | tail -3
