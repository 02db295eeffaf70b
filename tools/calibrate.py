#!/usr/bin/env python3
"""B200 cost-model calibration for the FA-forward loop graph.

The reference takes raw op costs in cycles and normalizes them itself
(costnorm.cpp:140-242). The paper takes them from documentation or from
direct measurement. This tool measures them on the GPU,
with the realized kernel of the current production schedule. It runs one
traced C3 launch (tools/trace_stats.py's trace: per-op issue / ready / done
clocks on CTA 0 of a full grid) and writes
paper_2512_18134_b200/schedules/calibration.json.

That file holds the raw cycles and the costs in units of T = 256 clk.
`tools/make_problems.py` builds the calibrated problems (`fa_fwd`,
`fa_fwd_cal`) from it.

Per op:
* MX_k, EX_k, CR_k: median of (done - ready) over steady trips. That is the
  op's execution after its inputs arrived; waiting on the producer is
  excluded.
* S_k, PV_k: the tensor-core time of a 128x128x128 bf16 tcgen05 GEMM,
  max(M, 128) * N / 256 * K / 16 = 512 clk. Issue is asynchronous; the
  issuing thread's time measures queueing, not the op.
* spill: the cross-warp handoff latency, half the measured mbarrier
  ping-pong round trip (tools/calib/ubench_bar.cu, 423 clk; one way ~212).
* spill_row: the cross-warp cost of MX_k's value. That value is the S row
  held in registers (regs = 128) plus the row max. A consumer on another warp
  re-reads the row from tensor memory (the MX load time) and waits for the
  handoff.

usage (on a GPU box): python tools/calibrate.py [--schedule fa_fwd] [--write]
"""
import argparse
import datetime
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "paper_2512_18134_b200", "schedules", "calibration.json")
T = 256
HANDOFF_ROUND_TRIP = 423  # tools/calib/ubench_bar.cu on B200


def measure(schedule, B=4, H=32, S=8192):
    import numpy as np
    import torch
    import paper_2512_18134_b200 as twfa
    prob, sol = twfa.load_schedule(schedule)
    plan = twfa.Plan(prob, sol)
    ids = [n["id"] for n in json.loads(prob)["graph"]["nodes"]]
    nw, cap = plan.describe()["num_warps"], 8192
    tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device="cuda")
    q, k, v = (torch.randn(B, H, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
    twfa.fa_fwd(plan, q, k, v)
    twfa.fa_fwd(plan, q, k, v, trace=tr, trace_cap=cap)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
    work = {}
    for w in range(nw):
        for i in range(int(t[w, 0, 0])):
            node, it, trip, t_issue, t_ready, t_done = (int(x) for x in t[w, 1 + i, :6])
            if t_ready == 0:
                continue  # ops that never waited (e.g. CR without a rescale)
            kind = ids[node].rstrip("0123456789")
            work.setdefault(kind, []).append((t_done - t_ready) % (1 << 32))
    return {k: float(np.median(v)) for k, v in work.items()}, torch.cuda.get_device_name(0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schedule", default="fa_fwd")
    ap.add_argument("--write", action="store_true")
    args = ap.parse_args()
    med, gpu = measure(args.schedule)
    gemm = 128 * 128 // 256 * 128 // 16  # 512 clk, tcgen05 floor
    raw = {"S": gemm, "PV": gemm, "MX": med.get("MX"), "EX": med.get("EX"), "CR": med.get("CR", T),
           "spill": HANDOFF_ROUND_TRIP / 2}
    if raw["MX"] is not None:
        raw["spill_row"] = raw["MX"] + raw["spill"]
    units = {k: max(1, int(round(v / T))) for k, v in raw.items() if v is not None}
    rec = {"T": T, "raw_clk": raw, "units": units, "gpu": gpu, "schedule_traced": args.schedule,
           "when": datetime.datetime.utcnow().isoformat(timespec="seconds") + "Z",
           "how": __doc__.split("\n\n")[1].strip()}
    print(json.dumps(rec, indent=1))
    if args.write:
        with open(OUT, "w") as f:
            json.dump(rec, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
