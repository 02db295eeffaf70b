"""Solve analysis-only loop problems (not realized by the kernels) with the
unmodified reference solver into paper_2512_18134_b200/schedules/analysis/:
fa_fwd_exsplit -- the production forward model with EX_k split into its MUFU
part (EXM_k, 4 units) and its FMA part (EXF_k), to show which bound holds the
initiation interval."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_problems as mp
raw = mp.fa_forward_problem(tc_variable_latency=True, calibrated=True, ex_split=True)  # reads calibration.json
mp.OUT = os.path.join(mp.OUT, "analysis")
os.makedirs(mp.OUT, exist_ok=True)
meta = mp.solve("fa_fwd_exsplit", raw, 9, 2, sys.argv[1] if len(sys.argv) > 1 else "z3 -in")
print({k: meta.get(k) for k in ("status", "I", "L", "joint_s")})
