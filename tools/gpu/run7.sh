SCHED=fa_fwd:experiments/E1_fa4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/e1_full python tools/prof_run.py fa 2 > gpurun_out/ncu_e1.log 2>&1
tail -2 gpurun_out/ncu_e1.log
