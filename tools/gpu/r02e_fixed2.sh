# backward with the fixed program: + one-lane issue, + memoized waits, - whole-row dQ readout
L=paper_2512_18134_b200/libtwfa.so; V=paper_2512_18134_b200/variants
TWFA_LIB=$V/fsolo.so timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/gpu/bwd_time.py $L $V/fsolo.so $V/fmemo.so $V/frd0.so; done
