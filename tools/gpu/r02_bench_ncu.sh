# round 2: default bench line (C5 S=8K, N=1), reference arm, ncu captures of the forward (pair and single) and GEMM
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 3000 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; tail -c 1500 gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fa_fwd -c 10 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-legs > gpurun_out/ncu_launch.log 2>&1
for P in 1 0; do TWFA_PAIR=$P timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -c 1 -f -o gpurun_out/fa_c3_pair$P python tools/prof_run.py fa 2 > gpurun_out/ncu_full_$P.log 2>&1; tail -2 gpurun_out/ncu_full_$P.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -f -o gpurun_out/gemm_full python tools/prof_run.py gemm 2 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
