REPS=2 SCHEDS=fa_fwd_ring2:experiments/R2_pertile,fa_fwd:experiments/E2_pertile timeout 900 python tools/variants.py paper_2512_18134_b200/libtwfa.so 2>&1
timeout 300 python tools/trace_stats.py 4 32 8192 fa_fwd_ring2:experiments/R2_pertile > gpurun_out/trace_r2p.txt 2>&1
