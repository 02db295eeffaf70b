export TWFA_LIB=paper_2512_18134_b200/variants/lean.so
SCHED=fa_fwd timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/lean_full python tools/prof_run.py fa 2 > gpurun_out/ncu_lean.log 2>&1
tail -3 gpurun_out/ncu_lean.log
