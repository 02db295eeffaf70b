timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
sed -n '1,17p' tools/gpu/run37.sh > /tmp/g.sh
bash /tmp/g.sh
for L in paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_old.so paper_2512_18134_b200/libtwfa.so paper_2512_18134_b200/variants/gemm_old.so; do TWFA_LIB=$L timeout 120 python /tmp/g.py; done
