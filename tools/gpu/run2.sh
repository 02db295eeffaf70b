cd $GRAFT_REPO_ROOT
SCHEDS=fa_fwd,fa_fwd_cal,fa_fwd_tcvl,fa_fwd:experiments/E1_fa4,fa_fwd:experiments/E2_pertile,fa_fwd:experiments/E3_sep timeout 600 python tools/variants.py paper_2512_18134_b200/libtwfa.so > gpurun_out/variants.txt 2>&1
cat gpurun_out/variants.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_full python tools/prof_run.py fa 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
