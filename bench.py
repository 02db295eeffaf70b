#!/usr/bin/env python3
"""Benchmark of the Twill-scheduled FA-forward executor on B200.

Metric (BASELINE.json): FA-fwd TFLOPS/GPU (bf16, d=128) & tensor-pipe
utilisation at 1/2/4/8 B200. One step = one FA-forward pass (one kernel
launch per GPU) over the rank's shard of synthetic bf16 Q/K/V resident in HBM.

Workload (default, BASELINE config 5 at S = 8192): non-causal, d = 128, a
FIXED job of B = 16, H = 64 (1024 independent (b, h) pairs). With N GPUs the
flattened pairs are split into N contiguous ranges (shard.pair_range), one
process per GPU, no collective on the data path: strong scaling, value =
job FLOPs / max-over-ranks time. `--scaling weak` instead gives every rank
the whole config (B per GPU fixed). FLOPs per step = 4 B H S^2 d (two GEMMs;
causal counts the unmasked triangle, 2 B H S^2 d). Inputs (>= 3 x 256 MiB per
rank at N = 8) exceed the 126 MB L2, so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c4|c5] [--seq S] [--scaling strong|weak]

`--gpus N` with N > 1 outside torchrun re-launches itself under
torch.distributed.run (one process per GPU, NCCL, NCCL_DEBUG=INFO so the
communicator's rank count is in the log); under torchrun (the driver's launch)
each process is one rank. `--share-gpu` maps several ranks onto the visible
GPUs with gloo collectives (functional check of the N > 1 path on a one-GPU
box; its timings are not scaling numbers).

--impl reference times the reference's CPU path on the host cores of this
box: the unmodified weftsched solver (oracle/_ref) on the committed FA problem
plus the fp32 host attention restatement (oracle/) on a bounded sample of the
same workload, and BASELINE config 1 (B=1 H=2 S=512 d=64) on all cores and on
one core.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FA-fwd TFLOPS/GPU (bf16, d=128) & tensor-pipe util at 1/2/4/8 B200"
UNIT = "TFLOPS"
D = 128
CONFIGS = {
    # name: (B, H, S, causal, seed, description) -- B x H is the job (strong
    # scaling) or the per-GPU slice (weak scaling)
    "c3": (4, 32, 8192, False, 2026, "BASELINE config 3: FA fwd bf16 non-causal d=128 B=4 H=32 S=8192"),
    "c4": (2, 32, 16384, True, 2027, "BASELINE config 4: FA fwd bf16 causal d=128 B=2 H=32 S=16384"),
    "c5": (16, 64, 8192, False, 3000, "BASELINE config 5: FA fwd bf16 non-causal d=128 B=16 H=64, S sweep point"),
}
SM_FLOP_PER_CLK = 8192  # dense bf16 tcgen05 per SM per clock (B200_PROFILING.md)


def fa_flops(pairs, S, causal):
    f = 4.0 * pairs * S * S * D
    return f / 2 if causal else f


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("bf16_tflops", 1590.0), j.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 6650.0, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed
    region, on the NVML device of the given CUDA device (PCI bus id)."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.power = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _handle(self, pynvml):
        import torch
        try:
            pr = torch.cuda.get_device_properties(self.device)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.device.index or 0)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = self._handle(pynvml)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "sw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "hw_thermal_slowdown": getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_power_cap": getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
                "hw_power_brake": getattr(pynvml, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        self.power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for n, bit in names.items():
                            if r & bit:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(0.005)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: record why
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        pw = sorted(self.power)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s), "power_w": round(pw[len(pw) // 2], 1) if pw else None}


# ---------------------------------------------------------------- ranks
class Ranks:
    """Process-group plumbing: NCCL, one process per GPU (torchrun env), or
    gloo with several ranks per GPU (--share-gpu). Collectives are only used
    outside the timed regions."""

    def __init__(self, share_gpu=False, device=None):
        import torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = None
        self.dist = None
        if device == "cpu":  # host-side tests of the rank plumbing (gloo)
            self.device = torch.device("cpu")
            share_gpu = True
        else:
            n_dev = max(1, torch.cuda.device_count())
            if self.world > 1 and not share_gpu and n_dev < int(os.environ.get("LOCAL_WORLD_SIZE", self.world)):
                raise SystemExit(f"bench.py: {os.environ.get('LOCAL_WORLD_SIZE', self.world)} ranks on this node "
                                 f"but only {n_dev} visible GPU(s); use --share-gpu for a functional run")
            self.device = torch.device("cuda", self.local % n_dev)
            torch.cuda.set_device(self.device)
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            self.backend = "gloo" if share_gpu else "nccl"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.device)
            else:
                dist.init_process_group("gloo")

    def _t(self, x, dtype):
        import torch
        dev = self.device if self.backend == "nccl" else "cpu"
        return torch.tensor(x, dtype=dtype, device=dev)

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.device.index])
            else:
                self.dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        import torch
        t = self._t([x], torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_objects(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def gather_checksums(self, local, shard):
        from paper_2512_18134_b200.shard import gather_pair_checksums
        if self.world == 1:
            return local.cpu()
        x = local if self.backend == "nccl" else local.cpu()
        return gather_pair_checksums(x, shard, self.dist)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: one process per GPU under
    torch.distributed.run, the same arguments; rank 0 prints the line."""
    if not args.share_gpu:
        import torch
        if torch.cuda.device_count() < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but {torch.cuda.device_count()} GPU(s) visible", file=sys.stderr)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- reference arm
def cpu_attention_sample(target_s=10.0, threads=0):
    """fp32 host attention (oracle restatement) on a bounded sample of the
    workload: the first `rows` query rows of H heads against S = 8192 keys.
    Returns (tflops, seconds, sample description, threads)."""
    import numpy as np
    from tests import oracle_lib
    S = 8192
    threads = threads or os.cpu_count()
    rng = np.random.default_rng(7)

    def run(H, rows):
        q = oracle_lib.round_bf16(rng.standard_normal((1, H, rows, D), dtype=np.float32))
        k = oracle_lib.round_bf16(rng.standard_normal((1, H, S, D), dtype=np.float32))
        v = oracle_lib.round_bf16(rng.standard_normal((1, H, S, D), dtype=np.float32))
        t0 = time.perf_counter()
        oracle_lib.attention(q, k, v, online=True, tile=128, threads=threads)
        return time.perf_counter() - t0

    probe = run(1, 64)
    flops_probe = 4.0 * 64 * S * D
    rate = flops_probe / max(probe, 1e-6)
    rows = 256
    H = max(1, min(1024, int(round(target_s * rate / (4.0 * rows * S * D)))))
    secs = run(H, rows)
    flops = 4.0 * H * rows * S * D
    return flops / secs / 1e12, secs, f"fp32 online-softmax host attention, H={H} heads x {rows} query rows x S={S} keys, d={D}", threads


def solver_time():
    """The reference's own CPU path: weftsched joint_search on the committed
    FA-forward problem with the pinned backend (z3 -in), via oracle/_ref."""
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        import _weftsched
    except ImportError as e:
        return {"unavailable": f"oracle/_ref not built: {e}"}
    import paper_2512_18134_b200 as twfa
    prob, _ = twfa.load_schedule("fa_fwd")
    meta = json.load(open(os.path.join(twfa.schedule_dir(), "fa_fwd.meta.json")))
    backend = meta["backend"]
    z3 = os.path.join(os.path.dirname(sys.executable), "z3")
    cmd = backend if backend == "internal" else backend.replace("z3", z3 if os.path.exists(z3) else "z3", 1)
    version = None
    if backend != "internal":
        try:
            version = subprocess.run([cmd.split()[0], "--version"], capture_output=True, text=True,
                                     timeout=30).stdout.strip()
        except OSError:
            version = "unavailable"
    t0 = time.perf_counter()
    r = _weftsched.joint(prob, 0, meta["stream_depth"], "" if backend == "internal" else cmd)
    secs = time.perf_counter() - t0
    sol = json.loads(twfa.load_schedule("fa_fwd")[1])
    same = r.get("status") == "sat" and r["M"] == sol["M"] and r["A"] == sol["A"] and r["I"] == sol["I"]
    return {"seconds": round(secs, 3), "backend": backend, "backend_version": version,
            "pinned_version": meta.get("backend_version"), "max_decisions": meta.get("max_decisions", 28),
            "cores": 1, "I": r.get("I"), "matches_committed_schedule": bool(same)}


def c1_reference():
    """BASELINE config 1 as stated: fp32 host attention B=1 H=2 S=512 d=64
    (loop semantics proj/tests/testutil.hpp:13-15) on all host cores and on
    one core, seed 7; best of 5 runs each."""
    import numpy as np
    from tests import oracle_lib
    B, H, S, d = 1, 2, 512, 64
    rng = np.random.default_rng(7)
    q, k, v = (rng.standard_normal((B, H, S, d), dtype=np.float32) for _ in range(3))
    flops = 4.0 * B * H * S * S * d
    out = {"shape": {"B": B, "H": H, "S": S, "d": d}, "flops": flops}
    for name, threads in (("all_cores", os.cpu_count()), ("one_core", 1)):
        best = None
        for _ in range(5):
            t0 = time.perf_counter()
            oracle_lib.attention(q, k, v, online=True, tile=128, threads=threads)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        out[name] = {"threads": threads, "ms": round(best * 1e3, 3), "gflops": round(flops / best / 1e9, 2)}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B, H, S, causal, _, desc = CONFIGS[args.config]
    S = args.seq or S
    import numpy as np
    from tests import oracle_lib
    threads = os.cpu_count()
    # one step: 1024 query rows of two (b, h) pairs against all S keys
    # (~8.6 GFLOP at S = 8192: a bounded, representative sample)
    rows, Hs, Sk = 1024, 2, S
    rng = np.random.default_rng(11)
    q = oracle_lib.round_bf16(rng.standard_normal((1, Hs, rows, D), dtype=np.float32))
    k = oracle_lib.round_bf16(rng.standard_normal((1, Hs, Sk, D), dtype=np.float32))
    v = oracle_lib.round_bf16(rng.standard_normal((1, Hs, Sk, D), dtype=np.float32))
    flops = 4.0 * Hs * rows * Sk * D / (2 if causal else 1)
    for _ in range(args.warmup):
        oracle_lib.attention(q, k, v, causal=causal, online=True, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_lib.attention(q, k, v, causal=causal, online=True, threads=threads)
    secs = time.perf_counter() - t0
    tflops = flops * args.steps / secs / 1e12
    solver = solver_time()
    sample = (f"per step: fp32 online-softmax host attention (oracle restatement; the reference has no "
              f"attention numerics) for {rows} query rows x {Sk} keys x d={D} of {Hs} (b,h) pairs")
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) rounded to bf16",
        "config": {"workload": desc, "B": B, "H": H, "S": S, "d": D, "causal": causal},
        "cpu_baseline": {"value": tflops, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "solver": solver,
        "c1": c1_reference(),
        "e2e": {"value": tflops, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def realized_schedule(twfa, plan, q, k, v, causal):
    """Steady-state cycles per trip of the realized schedule (one traced launch
    of the same workload, outside the timed region) against the solver's
    prediction I x (raw clk per normalized unit, schedules/fa_fwd.meta.json).
    Measured = median clock64 distance between consecutive issues of S1 on
    its warp in CTA 0 (one trip = 256 query rows x one K/V tile)."""
    import numpy as np
    import torch
    desc = plan.describe()
    meta = json.load(open(os.path.join(twfa.schedule_dir(), "fa_fwd.meta.json")))
    unit = min(int(raw) // norm for raw, norm in meta["cost_map"].items())
    nw, cap = desc["num_warps"], 8192
    tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device=q.device)
    twfa.fa_fwd(plan, q, k, v, causal=causal, trace=tr, trace_cap=cap)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().view(np.uint32).reshape(nw, cap, 8).astype(np.int64)
    prob = json.loads(twfa.load_schedule("fa_fwd")[0])
    s1 = [n["id"] for n in prob["graph"]["nodes"]].index("S1")
    w = desc["nodes"]["S1"]["warp_start"]
    n = int(t[w, 0, 0])
    recs = t[w, 1:1 + n]
    clk = recs[recs[:, 0] == s1][:, 3]
    trips = recs[recs[:, 0] == s1][:, 2]
    d = np.diff(clk) % (1 << 32)
    d = d[np.diff(trips) == 1]  # consecutive trips of one work tile
    return {"I": desc["I"], "unit_clk": unit, "predicted_clk_per_trip": desc["I"] * unit,
            "measured_clk_per_trip": float(np.median(d)) if len(d) else None,
            "trip": f"256 query rows x {desc.get('kv_tile', 128)} keys", "kernel": desc.get("kernel"),
            "how": "traced launch, CTA 0, median S1 issue-to-issue; tracing adds ~10%"}


def in_kernel_clock(twfa, plan, q, k, v, causal):
    """The SM clock the forward actually ran at: one traced launch of the same
    workload right after the timed region (same power state); the kernel
    stamps clock64 and %globaltimer in CTA 0 after its setup and at its
    teardown (words 1-4 of the trace). NVML samples (averaged over
    milliseconds) overstate the clock of a short burst: the board's power
    limit pulls the clock down within milliseconds of the kernel starting."""
    import numpy as np
    import torch
    nw, cap = plan.describe()["num_warps"], 64
    tr = torch.zeros(nw * cap * 8, dtype=torch.int32, device=q.device)
    twfa.fa_fwd(plan, q, k, v, causal=causal, trace=tr, trace_cap=cap)
    torch.cuda.synchronize()
    w = tr[:5].cpu().numpy().view(np.uint32).astype(np.int64)
    clk = (w[3] - w[1]) % (1 << 32)
    ns = (w[4] - w[2]) % (1 << 32)
    return {"sm_mhz": round(clk / ns * 1e3) if ns else None, "cta0_ms": round(ns / 1e6, 3),
            "how": "CTA 0's clock64 / %globaltimer span (setup to teardown) in one traced launch after the "
                   "timed region"}


def ncu_reference(workload):
    """Static ncu evidence for the kernel (profiles/ncu_summary.json): the
    DRAM traffic per launch and the ncu tensor-pipe figure, tagged with the SM
    clock of that capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    e = json.load(open(p)).get(workload)
    return e


def timed(step, steps, ranks, stream, clock_device):
    """W already done; barrier + sync, K steps between CUDA events on the
    launching stream, sync + barrier; returns (local ms, max ms, clocks)."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(clock_device) as clocks:
        torch.cuda.synchronize()
        ranks.barrier()
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ranks.barrier()
    ms_local = e0.elapsed_time(e1)
    return ms_local, ranks.max(ms_local), clocks.summary()


def run_ours(args, ranks):
    import torch
    import paper_2512_18134_b200 as twfa
    from paper_2512_18134_b200.shard import PairShard, job_digest
    from __graft_entry__ import build_lib
    build_lib()
    dev = ranks.device
    world, rank = ranks.world, ranks.rank
    B, H, S, causal, seed, desc = CONFIGS[args.config]
    S = args.seq or S
    if args.config == "c5":
        seed = 3000 + S // 1024
    pairs_cfg = B * H
    job_pairs = pairs_cfg * (world if args.scaling == "weak" else 1)
    shard = PairShard(job_pairs, world, rank)
    plan = twfa.Plan(*twfa.load_schedule("fa_fwd"))
    q, k, v = shard.make_inputs(S, D, seed, dev, torch.bfloat16)
    o = torch.empty_like(q)
    n_local = shard.count
    flops_local = fa_flops(n_local, S, causal)
    flops_job = fa_flops(job_pairs, S, causal)
    stream = torch.cuda.current_stream(dev)

    def step():
        if n_local:
            twfa.fa_fwd(plan, q, k, v, causal=causal, out=o)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    ms_local, ms, clocks = timed(step, args.steps, ranks, stream, dev)
    ms_per_step = ms / args.steps
    value = flops_job * args.steps / (ms * 1e-3) / 1e12
    per_launch_ms = ms_local / args.steps
    achieved = flops_local / (per_launch_ms * 1e-3) / 1e12 if n_local else 0.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965
    # tensor pipe busy fraction implied by the run itself: the algorithmic
    # dense-bf16 flops of one launch over what the tensor pipes of all SMs
    # could do at the sampled SM clock in the launch's time
    tensor_pipe_run = achieved * 1e12 / (sms * SM_FLOP_PER_CLK * sm_mhz * 1e6) if n_local else None

    # whole-job output check: exact per-pair checksums, gathered to rank 0
    cks = ranks.gather_checksums(shard.checksums(o), shard)
    digest = job_digest(cks.numpy())
    per_rank = ranks.gather_objects({"rank": rank, "device": str(dev), "pairs": [shard.start, shard.stop],
                                     "ms_per_step": ms_local / args.steps, "clocks": clocks,
                                     "tflops": achieved})

    # FA backward of the same shard (the paper's second loop; reported
    # beside the headline, not part of it): 5 GEMMs = 10 B H S^2 d flops
    bwd = None
    if n_local and not args.skip_legs:
        bplan = twfa.Plan(*twfa.load_schedule("fa_bwd"))
        o_f, lse = twfa.fa_fwd(plan, q, k, v, causal=causal, return_lse=True)
        dout = torch.randn_like(q)
        ws = torch.empty(n_local * S * 129 * 4, device=dev, dtype=torch.uint8)
        bwd_steps = max(1, min(args.steps, 10))
        for _ in range(3):
            twfa.fa_bwd(bplan, q, k, v, o_f, dout, lse, causal=causal, workspace=ws)
        torch.cuda.synchronize()
        bl, bm, _ = timed(lambda: twfa.fa_bwd(bplan, q, k, v, o_f, dout, lse, causal=causal, workspace=ws),
                          bwd_steps, ranks, stream, dev)
        bwd = {"value": 2.5 * flops_job * bwd_steps / (bm * 1e-3) / 1e12, "unit": UNIT,
               "ms_per_step": bm / bwd_steps, "steps": bwd_steps,
               "schedule": "fa_bwd.solution.json (I=%d)" % bplan.describe()["I"],
               "note": "backward of the same job; 4 launches per step (D pre-pass, dQ accumulator memset, main "
                       "kernel, dQ post-pass); not the headline metric"}
        del o_f, lse, dout, ws
        torch.cuda.empty_cache()

    # end to end through the reference-facing C ABI with HOST buffers:
    # twfa_fa_fwd_host (the call the reference's C++ host / CLI / ctypes
    # binding makes) on page-locked host Q, K, V, O; every step copies the
    # inputs host -> device and O device -> host inside the call, pipelined
    # over (b, h) chunks and three CUDA streams. Synchronous call: timed by
    # the host clock between barriers, max over ranks.
    e2e = None
    if n_local and not args.skip_legs:
        import numpy as np
        pin = [x.cpu().pin_memory() for x in (q, k, v)]
        ho = torch.empty_like(pin[0]).pin_memory()
        hq, hk, hv, hon = (t.view(torch.int16).numpy().view(np.uint16) for t in (*pin, ho))

        def e2e_step():
            twfa.fa_fwd_host(plan, hq, hk, hv, causal=causal, out=hon)

        e2e_steps = max(1, min(args.steps, 10))
        for _ in range(2):
            e2e_step()
        ranks.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        t1 = time.perf_counter()
        ranks.barrier()
        e2e_s = ranks.max(t1 - t0)
        same = torch.equal(ho.to(dev), o)  # the host call computed the device call's O
        e2e = {"value": flops_job * e2e_steps / e2e_s / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": 3 * q.numel() * q.element_size() * world,
               "d2h_bytes_per_step": o.numel() * o.element_size() * world, "steps": e2e_steps,
               "ms_per_step": e2e_s / e2e_steps * 1e3, "o_bit_identical_to_device_call": bool(same),
               "path": "twfa_fa_fwd_host (C ABI, include/twfa.h) on page-locked host buffers: chunked H2D / kernel "
                       "/ D2H pipeline over three CUDA streams inside the call; host clock around the synchronous "
                       "call, max over ranks"}
        del pin, ho, hq, hk, hv, hon

    ranks.barrier()
    if rank != 0:
        return
    peak, _, peak_kind = measured_peaks()
    meta = json.load(open(os.path.join(twfa.schedule_dir(), "fa_fwd.meta.json")))
    workload = f"fa_fwd_{args.config}" + (f"_S{S}" if args.seq else "")
    desc_plan = plan.describe()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic N(0,1) bf16 Q/K/V generated on device, one generator per (b,h) pair (seed {seed})",
        "config": {"workload": desc, "B": B, "H": H, "S": S, "d": D, "causal": causal, "job_pairs": job_pairs,
                   "pairs_per_rank": [r["pairs"] for r in per_rank],
                   "parallelism": f"bh-shard x{world} ({args.scaling} scaling), no collective on the data path"
                                  + (f", {ranks.backend} for barriers/timing" if world > 1 else ""),
                   "schedule": "fa_fwd.solution.json (%s, I=%d)" % (meta["backend"], desc_plan["I"]),
                   "l2": "inputs 3x%d MiB per rank > 126 MB L2; no flush" % (q.numel() * 2 >> 20)},
        "per_gpu_tflops": value / world,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "peak_kind": f"{peak_kind} bf16 burst (MEASURED_PEAKS.json)",
                     "kernel": "twfa::fa_fwd_spec (" + desc_plan.get("kernel", "?") + ", "
                               + ("CTA pairs, cta_group::2" if desc_plan.get("cta_pair") else "one CTA per tile")
                               + ")",
                     "flops_per_launch": flops_local, "launch_ms": per_launch_ms,
                     "spec_peak_at_sampled_clock": sms * SM_FLOP_PER_CLK * sm_mhz * 1e6 / 1e12},
        "tensor_pipe": {"busy_frac_from_run": tensor_pipe_run, "sm_mhz": sm_mhz,
                        "how": "algorithmic flops per launch / (SMs x 8192 flop/clk x sampled SM clock x launch "
                               "time), this run (NVML median SM clock during the timed region)",
                        "power_w": clocks.get("power_w"),
                        "note": "under sustained load the 1000 W board limit (sw_power_cap) sets the SM clock; "
                                "this per-clock fraction is the clock-independent figure (DESIGN.md 10)"},
        "clocks": clocks,
        "per_rank": per_rank,
        "job_checksum": {"digest": digest, "pairs": int(cks.numel()),
                         "how": "sha256 over the per-pair int64 sums of O's bf16 bit patterns, in pair order; "
                                "independent of N"},
        "gpu_launches": args.steps,
    }
    if e2e:
        line["e2e"] = e2e
    if bwd:
        line["fa_bwd"] = bwd
    # ncu evidence: DRAM traffic of this exact launch (one GPU) and the ncu
    # tensor-pipe figure, tagged with the workload and the clock it ran at
    ncu = ncu_reference(workload)
    if ncu and world == 1:
        line["roofline"]["traffic"] = ncu.get("dram_bytes_per_launch")
    key = workload if ncu else "fa_fwd_c3"
    ncu = ncu or ncu_reference(key)
    if ncu:
        line["tensor_pipe"]["ncu"] = {"workload": key, "tensor_pipe_active_pct": ncu.get("tensor_pipe_active_pct"),
                                      "xu_pipe_inst_pct": ncu.get("xu_pipe_inst_pct"), "sm_ghz": ncu.get("sm_ghz"),
                                      "source": "profiles/ncu_summary.json (ncu --set full --clock-control none, "
                                                "one launch)"}
    if world == 1 and n_local:
        # the clock the kernel ran at (NVML's median can miss the power cap's
        # pull-down in a short timed region); tensor-pipe fraction per clock
        # from it
        ik = in_kernel_clock(twfa, plan, q, k, v, causal)
        line["tensor_pipe"]["in_kernel_clock"] = ik
        if ik.get("sm_mhz"):
            line["tensor_pipe"]["busy_frac_at_kernel_clock"] = \
                achieved * 1e12 / (sms * SM_FLOP_PER_CLK * ik["sm_mhz"] * 1e6)
    if not args.skip_legs:
        line["schedule_realized"] = realized_schedule(twfa, plan, q, k, v, causal)
        # whole work tile, untraced: the modulo schedule's makespan for N
        # iterations, (N - 1) I + L units (the reference's simulate_pipeline,
        # sim.cpp:371-466; tests/test_lowering.py checks the formula against
        # it), against the timed launches at the sampled SM clock
        sr = line["schedule_realized"]
        n_iter = -(-S // 128)
        tiles = n_local * (-(-S // 256))
        grid = min(tiles, sms)
        if not causal and sr.get("unit_clk"):
            sr["predicted_tile_clk"] = ((n_iter - 1) * sr["I"] + desc_plan["L"]) * sr["unit_clk"]
            sr["measured_tile_clk"] = per_launch_ms * 1e-3 * sm_mhz * 1e6 / (tiles / grid)
            sr["measured_clk_per_trip_untraced"] = sr["measured_tile_clk"] / n_iter
            sr["tile"] = f"256 query rows x {n_iter} K/V iterations; {tiles / grid:.1f} tiles per CTA"
        line["legs"] = side_legs(twfa, plan, dev, stream)
    if world == 1 and not args.no_cpu_baseline:
        tfl, secs, sample, threads = cpu_attention_sample()
        line["cpu_baseline"] = {"value": tfl, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": sample, "seconds": round(secs, 2),
                                "solver": solver_time()}
    print(json.dumps(line), flush=True)


def side_legs(twfa, plan, dev, stream):
    """Rank 0, after the timed region: C3 (the round-1 headline shape, short
    burst), C4 (causal) and the C2 GEMM mainloop 8192^3 with its own
    roofline."""
    import torch
    peak, _, _ = measured_peaks()
    out = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.Generator(device=dev).manual_seed(2026)
    q, k, v = (torch.randn(4, 32, 8192, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    for _ in range(3):
        twfa.fa_fwd(plan, q, k, v, out=o)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(20):
        twfa.fa_fwd(plan, q, k, v, out=o)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    f = fa_flops(128, 8192, False)
    out["c3"] = {"tflops": f / (ms * 1e-3) / 1e12, "ms": ms, "launches": 20,
                 "workload": "C3 B=4 H=32 S=8192 non-causal, 20 launches back to back"}
    del q, k, v, o
    # C4: causal, B=2 H=32 S=16384 (flops of the unmasked triangle)
    g.manual_seed(2027)
    q, k, v = (torch.randn(2, 32, 16384, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    for _ in range(3):
        twfa.fa_fwd(plan, q, k, v, causal=True, out=o)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(20):
        twfa.fa_fwd(plan, q, k, v, causal=True, out=o)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    out["c4"] = {"tflops": fa_flops(64, 16384, True) / (ms * 1e-3) / 1e12, "ms": ms, "launches": 20,
                 "workload": "C4 B=2 H=32 S=16384 causal (flops of the unmasked triangle), 20 launches"}
    del q, k, v, o
    gp = twfa.Plan(*twfa.load_schedule("gemm_mainloop"))
    M = N = K = 8192
    g.manual_seed(1234)
    a = (torch.randn(M, K, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    b = (torch.randn(N, K, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        twfa.gemm(gp, a, b, out=c)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(20):
        twfa.gemm(gp, a, b, out=c)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
    out["gemm_c2"] = {"tflops": tf, "ms": ms, "launches": 20,
                      "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "frac": tf / peak,
                                   "algorithmic_bytes": (M * K + N * K + M * N) * 2,
                                   # dram__bytes_read.sum + dram__bytes_write.sum of one launch
                                   # (ncu, profiles/r02b_gemm_policy.txt, default L2 policy)
                                   "traffic": 0.994e9 + 0.127e9},
                      "kernel": "twfa::gemm_kernel (CTA pair, cta_group::2, 256x256 tiles, TMA-store epilogue)",
                      "workload": "BASELINE config 2: GEMM mainloop bf16 8192^3 (C = A B^T), 20 launches"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--seq", type=int, default=0, help="override S (C5 sweep points)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--share-gpu", action="store_true", help="several ranks per GPU, gloo (functional runs)")
    ap.add_argument("--skip-legs", action="store_true", help="headline only (no backward / e2e / side legs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    ranks = Ranks(share_gpu=args.share_gpu)
    try:
        run_ours(args, ranks)
    finally:
        ranks.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
