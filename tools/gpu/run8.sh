timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
TWFA_KERNEL=interpreter SCHEDS=fa_fwd,fa_fwd:experiments/E1_fa4 timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd:experiments/E1_fa4 > gpurun_out/trace_e1.txt 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd > gpurun_out/trace_fa.txt 2>&1
