SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/spec_ex_full python tools/prof_run.py fa 2 > gpurun_out/ncu_specex.log 2>&1
tail -1 gpurun_out/ncu_specex.log
