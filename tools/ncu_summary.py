"""Summarise an `ncu --set full` capture into profiles/ncu_summary.json.
usage: python tools/ncu_summary.py <report.ncu-rep> <workload> [flops_per_launch]"""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, workload = sys.argv[1], sys.argv[2]
flops = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
m = dict(zip(h, v))
def f(k):
    return float(m[k].replace(",", ""))
def mb(k):  # ncu reports Mbyte / Gbyte / Kbyte
    unit = u[h.index(k)].split("/")[0]
    return f(k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
dur_s = f("gpu__time_duration.sum") * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}[u[h.index("gpu__time_duration.sum")]]
e = {
    "kernel": m.get("Kernel Name", ""),
    "duration_ms": dur_s * 1e3,
    "sm_ghz": f("sm__cycles_elapsed.avg.per_second") * {"Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}.get(u[h.index("sm__cycles_elapsed.avg.per_second")], float("nan")) if "sm__cycles_elapsed.avg.per_second" in m else None,
    "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
    "dram_read_bytes": mb("dram__bytes_read.sum"),
    "dram_write_bytes": mb("dram__bytes_write.sum"),
    "tensor_pipe_active_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "tc_pipe_active_pct": f("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
    "xu_pipe_inst_pct": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_active_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_active_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active") if "sm__inst_issued.avg.pct_of_peak_sustained_active" in m else None,
    "registers_per_thread": f("launch__registers_per_thread"),
    "smem_per_block_bytes": mb("launch__shared_mem_per_block") if u[h.index("launch__shared_mem_per_block")] != "" else None,
    "grid": int(f("launch__grid_size")), "block": int(f("launch__block_size")),
}
if flops:
    e["flops_per_launch"] = flops
    e["tflops_under_ncu"] = flops / dur_s / 1e12
p = os.path.join(ROOT, "profiles", "ncu_summary.json")
allj = json.load(open(p)) if os.path.exists(p) else {}
allj[workload] = e
json.dump(allj, open(p, "w"), indent=1, sort_keys=True)
print(json.dumps(e, indent=1))
