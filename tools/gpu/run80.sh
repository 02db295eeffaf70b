timeout 600 ncu --set full --clock-control none -k regex:gemm -c 1 -f -o gpurun_out/gemm_full python tools/prof_run.py gemm 2 > /dev/null 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page details 2>/dev/null | grep -E "Duration|SM Frequency|L2 Hit Rate|DRAM Throughput|Memory Throughput|L1/TEX Hit|Compute \(SM\) Throughput" | head -10
