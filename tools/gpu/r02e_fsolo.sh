# forward + backward: TMA / MMA warp on one elected lane (TWFA_SOLO / TWFA_BWD_SOLO = 1, default now) vs solo0
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 900 python -m pytest tests/test_gpu_fa.py tests/test_gpu_trace.py -x -q 2>&1 | tail -2
REPS=3 timeout 600 python tools/sustained.py $L $V/solo0.so
SHAPE=2,32,16384 CAUSAL=1 REPS=2 timeout 400 python tools/sustained.py $L $V/solo0.so
for P in 0; do TWFA_PAIR=$P REPS=2 timeout 400 python tools/sustained.py $L $V/solo0.so | sed "s/^/pair=$P /"; done
timeout 300 python tools/gpu/bwd_time.py $L $V/solo0.so $V/rdld14.so
