# backward, non-production schedules: light ops dispatched by kind to compile-time specializations (default) vs the loop
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_trace.py -x -q 2>&1 | tail -1
for s in fa_bwd_split fa_bwd_qstage fa_bwd_cal fa_bwd; do BSCHED=$s timeout 300 python tools/gpu/bwd_time.py $L $V/sw0.so | sed "s/^/$s /"; done
