# GEMM 8192^3: DRAM bytes per launch for more raster groups (A/B evict_last), and cuBLAS for reference
for G in 4 6 8 10 12; do echo "group $G"; TWFA_GEMM_GROUP=$G timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -c 1 python tools/prof_run.py gemm 2 2>&1 | grep -E "dram__|gpu__time" ; done
cat > /tmp/cublas_one.py <<'PY'
import torch
a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16); b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
for _ in range(3): c = a @ b.t()
torch.cuda.synchronize()
PY
echo cublas; timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gemm|nvjet|sm100|cutlass" -c 1 python /tmp/cublas_one.py 2>&1 | grep -E "dram__|gpu__time|==PROF== Profiling|  [a-z_0-9]+.*\(" | head -8
timeout 300 python tools/gemm_time.py 4 6 8 10 12
