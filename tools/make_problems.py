#!/usr/bin/env python3
"""Author the Blackwell (sm_100a) loop problems in the reference's problem
format (`/root/reference/proj/src/ir.cpp:93-229`: machine + graph, strict keys)
and, with --solve, run them through the reference scheduler (oracle/_ref, the
unmodified weftsched built in place) to produce the golden schedules the
B200 executor consumes.

Outputs (paper_2512_18134_b200/schedules/):
  <name>.raw.json        raw B200 cycle costs
  <name>.json            normalized problem (reference `normalize`, U given)
  <name>.solution.json   reference `joint` output (pinned backend)
  <name>.listing.txt     reference `codegen` listing of that solution
  <name>.meta.json       cost map, F, backend, solve seconds

Raw costs (B200, one 128-key KV tile, one 128-row Q sub-tile, d = 128):
  QK^T / PV GEMM  128x128x128 bf16 = 2.1 MMAC / 4096 MAC/clk/SM  = 512 clk (TC)
  EX  16384 exp2 at 16/clk/SM (MUFU)                              = 1024 clk
  MX  tcgen05.ld of S + 16384 FMNMX at 64/clk                      = 256 clk
  CR  tcgen05.ld/st of O (64 KiB round trip) + 16384 FMUL          = 256 clk
  spill (row statistics through shared memory + mbarrier)         = 256 clk
  TMA tile load (32 KiB)                                           = 512 clk
Everything is a power-of-two multiple of 256, so normalization at U >= 7 is
exact (F = 0) with one unit = 256 SM cycles.
"""
import argparse
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "paper_2512_18134_b200", "schedules")


def node(id_, unit, cycles, **kw):
    n = {"id": id_, "rrt": {unit: [1] * cycles} if unit else {}, "cycles": cycles}
    n.update(kw)
    return n


def edge(src, dst, d, delta=0, blocking=False):
    e = {"src": src, "dst": dst, "d": d}
    if delta:
        e["delta"] = delta
    if blocking:
        e["blocking"] = True
    return e


def fa_forward_problem(tc_variable_latency=False, calibrated=False, s_ring=1, split_s=False, ex_split=False):
    """FA-forward loop body on sm_100a: two 128-row Q sub-tiles (k = 0, 1)
    share one 128-key K/V tile per iteration.

    Warps: 16 (4 aligned warpgroup slots); warp 15 is the variable-latency
    (TMA) warp, so warpgroup ops can use slots 0, 4, 8 only. Per-warp register
    budget 224 models a softmax warpgroup after setmaxnreg: one tile's S row
    (MX, 128 regs) and packed P / row sum (EX, 64) fit, a second tile or a
    correction working set (CR, 64) does not.
    Tensor memory: 512 columns; S/P and O of each sub-tile take 128 each.
    The causal variant runs the same loop body (masking only changes the
    per-tile trip count and applies the mask inside MX on diagonal tiles), so
    it shares this problem and its schedule.
    Blocking edges are the mbarrier waits of the realized kernel: TMA landed
    (LD -> GEMM), MMA committed (S -> MX, PV -> CR), P stored (EX -> PV),
    O rescaled (CR -> PV).

    s_ring = 2 double-buffers S in tensor memory instead: the S/P columns of
    each sub-tile (128) hold two 64-key S tiles, so the K/V tile is 64 keys,
    every per-iteration cost halves, and S_k(i+1) no longer waits for
    PV_k(i): the edge PV_k -> S_k carries delta = 2 (S_k(i+2) overwrites the
    P_k(i) that PV_k(i) reads). The executor derives the ring depth (and the
    64-key tile) from that delta.

    split_s issues each S_k as two N = 64 GEMMs. SA_k computes keys 0-63
    into S columns 0-63; it only waits for MX_k(i-1) to hold its row in
    registers (edge MX_k -> SA_k, delta 1). SB_k computes keys 64-127 into
    columns 64-127, where P_k (bf16) is aliased; it follows PV_k(i-1)
    (edge PV_k -> SB_k, delta 1). Half of the next S then overlaps EX_k.
    """
    T = 256  # raw clk per unit (see module docstring)
    # per-op durations in units of T: datasheet throughput (default) or the
    # values measured on B200 by the in-kernel trace (tools/timeline.py):
    # MX ~500 clk (TMEM load of the S row + max + handoff), EX ~1500 clk
    # (MUFU-bound exp of a 128x128 tile + bf16 pack + TMEM store)
    cost = dict(S=2, PV=2, MX=1, EX=4, CR=1)
    spill = 1
    if calibrated:
        # measured on B200 (tools/calibrate.py -> schedules/calibration.json),
        # rounded to units of T = 256 clk (the normalizer then maps them
        # exactly, F = 0; the reference's ILP on the unrounded cycles, with
        # five distinct costs, distorts ratios by F >= 512 at U <= 16)
        cal = json.load(open(os.path.join(OUT, "calibration.json")))
        assert cal["T"] == T
        cost = {k: v for k, v in cal["units"].items() if k != "spill"}
        spill = cal["units"]["spill_row"]  # MX's value is the S row: re-read + handoff
    if s_ring == 2:  # 64-key iterations: GEMMs 256 clk, 8192 exp2 = 512 clk
        cost = dict(S=1, PV=1, MX=1, EX=2, CR=1)
    machine = {
        "units": [{"name": "TC", "capacity": 1}, {"name": "TMA", "capacity": 1},
                  {"name": "MUFU", "capacity": 1}, {"name": "ALU", "capacity": 1},
                  {"name": "FMA", "capacity": 1}],
        "memories": [{"name": "tmem", "capacity": 512}],
        "num_warps": 16,
        "reg_limit": 224,
        "vl_warp": 15,
    }
    kv = 128 // s_ring  # keys per K/V tile
    ld = 2 // s_ring  # streamed: zero cycles after the rewrite
    nodes = [
        node("LDK", "TMA", ld, variable_latency=True),
        node("LDV", "TMA", ld, variable_latency=True),
    ]
    edges = []
    for k in (0, 1):
        if split_s:
            half = max(1, cost["S"] // 2)
            nodes += [node(f"SA{k}", "TC", half, footprint={"tmem": kv // 2}),
                      node(f"SB{k}", "TC", half, footprint={"tmem": kv // 2})]
            edges += [edge("LDK", f"SA{k}", 0, blocking=True), edge("LDK", f"SB{k}", 0, blocking=True),
                      edge(f"SA{k}", f"MX{k}", half, blocking=True), edge(f"SB{k}", f"MX{k}", half, blocking=True),
                      edge(f"MX{k}", f"SA{k}", cost["MX"], delta=1),
                      edge(f"PV{k}", f"SB{k}", 0, delta=1)]
        else:
            nodes += [node(f"S{k}", "TC", cost["S"], footprint={"tmem": kv})]
            edges += [edge("LDK", f"S{k}", 0, blocking=True), edge(f"S{k}", f"MX{k}", cost["S"], blocking=True),
                      # S_k(i+1) overwrites the TMEM columns P_k(i) is read from: the
                      # calibrated model waits for PV_k's completion (cross-warp commit)
                      edge(f"PV{k}", f"S{k}", cost["PV"] if calibrated else 0, delta=s_ring)]
        if ex_split:
            # EX_k as its MUFU part (EXM_k: 16384 exp2 at 16/clk = 4 units)
            # and its FMA part (EXF_k: scale-subtract, bf16 pack, row sum and
            # the P stores, the rest of the calibrated EX); analysis only
            # (the kernel realizes EX as one op)
            exm = 4
            exf = max(1, cost["EX"] - exm)
            nodes += [node(f"MX{k}", "ALU", cost["MX"], regs=kv, spill_cost=spill, warps_required=4),
                      # the exponentials' values stay in the warpgroup's registers
                      # until EXF packs and stores them: a whole EX as spill cost
                      node(f"EXM{k}", "MUFU", exm, regs=kv // 2, spill_cost=cost["EX"], warps_required=4),
                      node(f"EXF{k}", "FMA", exf, regs=kv // 2, warps_required=4),
                      node(f"CR{k}", "FMA", cost["CR"], regs=64, warps_required=4),
                      node(f"PV{k}", "TC", cost["PV"], footprint={"tmem": 128})]
            edges += [edge(f"MX{k}", f"EXM{k}", cost["MX"]), edge(f"EXM{k}", f"EXF{k}", exm),
                      edge(f"MX{k}", f"MX{k}", cost["MX"], delta=1), edge(f"EXM{k}", f"EXM{k}", exm, delta=1),
                      edge(f"EXF{k}", f"EXF{k}", exf, delta=1), edge(f"MX{k}", f"CR{k}", cost["MX"]),
                      edge(f"EXF{k}", f"PV{k}", exf, blocking=True), edge("LDV", f"PV{k}", 0, blocking=True),
                      edge(f"CR{k}", f"PV{k}", cost["CR"], blocking=True),
                      edge(f"PV{k}", f"CR{k}", cost["PV"], delta=1, blocking=True),
                      edge(f"PV{k}", f"PV{k}", cost["PV"], delta=1)]
            continue
        nodes += [
            # split S: SA_k(i+1) overwrites S columns right after MX_k(i) read them,
            # so the S row (MX_k's value) cannot be re-read by a consumer on another
            # warp: a spill cost of a whole EX (reusing an existing cost, so the
            # normalization is unchanged) keeps EX_k with MX_k
            node(f"MX{k}", "ALU", cost["MX"], regs=kv, spill_cost=cost["EX"] if split_s else spill,
                 warps_required=4),
            node(f"EX{k}", "MUFU", cost["EX"], regs=kv // 2, warps_required=4),
            node(f"CR{k}", "FMA", cost["CR"], regs=64, warps_required=4),
            node(f"PV{k}", "TC", cost["PV"], footprint={"tmem": 128}),
        ]
        edges += [
            edge(f"MX{k}", f"EX{k}", cost["MX"]),
            edge(f"MX{k}", f"MX{k}", cost["MX"], delta=1),
            edge(f"EX{k}", f"EX{k}", cost["EX"], delta=1),
            edge(f"MX{k}", f"CR{k}", cost["MX"]),
            edge(f"EX{k}", f"PV{k}", cost["EX"], blocking=True),
            edge("LDV", f"PV{k}", 0, blocking=True),
            edge(f"CR{k}", f"PV{k}", cost["CR"], blocking=True),
            edge(f"PV{k}", f"CR{k}", cost["PV"], delta=1, blocking=True),
            edge(f"PV{k}", f"PV{k}", cost["PV"], delta=1),
        ]
    if tc_variable_latency:
        # tcgen05.mma is asynchronous: its completion is only observed through
        # an mbarrier (tcgen05.commit) and its latency depends on what else
        # occupies the tensor pipe. Marked variable-latency, the GEMMs share the
        # reserved warp with the TMA loads (they are not streamed: they have
        # predecessors, so they keep their cycles and TC reservations).
        for n in nodes:
            if n["id"][0] in "SP":
                n["variable_latency"] = True
    # scale to raw cycles
    for n in nodes:
        n["cycles"] *= T
        n["rrt"] = {u: [1] * n["cycles"] for u in n["rrt"]}
        if n.get("spill_cost"):
            n["spill_cost"] *= T
    for e in edges:
        e["d"] *= T
    return {"machine": machine, "graph": {"nodes": nodes, "edges": edges}}


def fa_backward_problem(calibrated=False, fused=False, exb_spill=16, q_staging=False):
    """FA-backward loop body on sm_100a (the paper's second workload,
    PAPER.md:1073-1148; the single-pass algorithm of FA3): one CTA owns a
    128-key K/V tile (K, V resident in shared memory, dK and dV accumulated
    in tensor memory) and iterates over the 128-row Q tiles of its head:

      LDQ, LDO  TMA loads of Q_i and dO_i (streamed rings)
      ST        S^T = K Q_i^T            tcgen05.mma SS -> TMEM (keys on lanes)
      EXB       P^T = exp2(S^T - LSE_i)  MUFU; P^T (bf16) -> TMEM over S^T
      DP        dP^T = V dO_i^T          tcgen05.mma SS -> TMEM
      DS        dS^T = P^T (dP^T - D_i)  FMA; bf16 -> TMEM over dP^T and -> smem
      DV        dV += P^T dO_i           tcgen05.mma TS
      DK        dK += dS^T Q_i           tcgen05.mma TS
      DQ        dQ_i = dS K              tcgen05.mma SS -> TMEM over S^T
      RD        dQ_i -> global           tcgen05.ld + TMA reduce-add (fp32)

    Tensor memory (512 columns): dK, dV, S^T (P^T), dP^T (dS^T, then dQ_i),
    128 each. The aliasing is carried by edges: DV -> ST (delta 1: S^T(i+1)
    overwrites the P^T DV(i) reads; in order on the issuing thread), DK -> DQ
    (DQ overwrites the dS^T DK reads; in order), RD -> DP (delta 1: dP^T(i+1)
    needs dQ_i read out), RD -> DS (delta 1: dS(i+1) reuses the smem buffer
    RD stages dQ_i in). S^T(i+1) thus only waits for DV(i): the exponentials
    of the next tile overlap DS, DK, DQ and RD of this one.
    EXB -> DS carries P in registers (spill cost: a re-read of P from tensor
    memory in bf16 changes the numerics, so a large cost keeps them on one
    warpgroup). The tensor-core ops are variable latency (the production
    forward model): they go to the reserved warp with the loads.
    Costs (datasheet, units of 256 clk): GEMMs 2, EXB 4 (16384 exp2 at
    16/clk/SM), DS 2 (TMEM read of dP^T + FMA + two stores), RD 2 (TMEM read
    of dQ_i + staging + bulk reduce issue)."""
    T = 256
    machine = {
        "units": [{"name": "TC", "capacity": 1}, {"name": "TMA", "capacity": 1},
                  {"name": "MUFU", "capacity": 1}, {"name": "ALU", "capacity": 1},
                  {"name": "FMA", "capacity": 1}],
        "memories": [{"name": "tmem", "capacity": 512}],
        "num_warps": 16,
        "reg_limit": 224,
        "vl_warp": 15,
    }
    g = 2  # one 128x128x128 tcgen05 GEMM
    # calibrated: the in-kernel clock profile of the realized loop
    # (TWFA_BWD_PROF): EXB ~1500 clk incl. the TMEM read of S^T, DS ~1000
    ex, dsc = (6, 4) if calibrated else (4, 2)
    nodes = [node("LDQ", "TMA", 2, variable_latency=True), node("LDO", "TMA", 2, variable_latency=True)]
    for v in ("ST", "DP"):
        nodes.append(node(v, "TC", g, footprint={"tmem": 128}, variable_latency=True))
    if fused:
        # EXB and DS as one warpgroup op (P^T is carried in registers from the
        # exponentials into dS^T, so they cannot sit on different warps). Its
        # consumers read through memory: P^T (TMEM) after the exponential part
        # (edge delay ex < the op's duration), dS^T (TMEM + smem) at the end,
        # each behind an mbarrier handoff (spill cost 1 = 256 clk). dP^T is
        # only needed by the DS part: DP -> EXDS with delay 0 is conservative.
        nodes.append(node("EXDS", "MUFU", ex + dsc, regs=128, spill_cost=1, warps_required=4))
    else:
        nodes += [
            node("EXB", "MUFU", ex, regs=128, spill_cost=exb_spill, warps_required=4),
            node("DS", "FMA", dsc, regs=64, warps_required=4),
        ]
    nodes += [
        node("DV", "TC", g, variable_latency=True),
        node("DK", "TC", g, variable_latency=True),
        node("DQ", "TC", g, variable_latency=True),
        node("RD", "ALU", 2, regs=128, warps_required=4),
    ]
    edges = [
        edge("LDQ", "ST", 0, blocking=True), edge("LDQ", "DK", 0, blocking=True),
        edge("LDO", "DP", 0, blocking=True), edge("LDO", "DV", 0, blocking=True),
    ]
    if fused:
        edges += [
            edge("ST", "EXDS", g, blocking=True), edge("DP", "EXDS", 0, blocking=True),
            edge("EXDS", "DV", ex, blocking=True),
            edge("EXDS", "DK", ex + dsc, blocking=True), edge("EXDS", "DQ", ex + dsc, blocking=True),
            edge("RD", "EXDS", 2, delta=1, blocking=True), edge("EXDS", "EXDS", ex + dsc, delta=1),
        ]
    else:
        edges += [
            edge("ST", "EXB", g, blocking=True),
            edge("EXB", "DV", ex, blocking=True), edge("EXB", "DS", ex),
            edge("DP", "DS", g, blocking=True),
            edge("DS", "DK", dsc, blocking=True), edge("DS", "DQ", dsc, blocking=True),
            # RD stages dQ_i in shared memory: in the dS buffer (DS(i+1) then
            # waits for RD(i)), or -- q_staging -- in Q_i's ring slot, which
            # DK(i) has finished reading once DQ(i) completed: DS(i+1) then
            # only waits for DQ(i) to have read dS(i), and RD(i) holds the Q
            # slot (edge LDQ -> RD) until its bulk reductions have read it
            *([edge("DQ", "DS", g, delta=1, blocking=True), edge("LDQ", "RD", 0)] if q_staging
              else [edge("RD", "DS", 2, delta=1, blocking=True)]),
            edge("EXB", "EXB", ex, delta=1), edge("DS", "DS", dsc, delta=1),
        ]
        if exb_spill < ex:
            # a DS on another warpgroup reads P^T back from tensor memory
            # (bf16) at its start: S^T(i+1) may overwrite it only after that
            edges.append(edge("DS", "ST", 1, delta=1, blocking=True))
    edges += [
        edge("DQ", "RD", g, blocking=True),
        edge("DV", "ST", 0, delta=1),
        edge("DK", "DQ", 0),
        edge("RD", "DP", 2, delta=1, blocking=True),
        edge("DV", "DV", g, delta=1), edge("DK", "DK", g, delta=1), edge("RD", "RD", 2, delta=1),
    ]
    for n in nodes:
        n["cycles"] *= T
        n["rrt"] = {u: [1] * n["cycles"] for u in n["rrt"]}
        if n.get("spill_cost"):
            n["spill_cost"] *= T
    for e in edges:
        e["d"] *= T
    return {"machine": machine, "graph": {"nodes": nodes, "edges": edges}}


def fa_backward_pp_problem():
    """FA-backward loop body with two 64-query sub-tiles per iteration (the
    paper's Blackwell strategy: two exponential
    warpgroups ping-pong over alternating query tiles, a third stages the dQ
    reduction). One CTA owns a 128-key K/V tile (K, V resident in shared
    memory; dK, dV accumulated in tensor memory) and iterates over 128-row
    Q / dO tiles (LDQ, LDO, streamed); sub-tile k = queries 64k .. 64k + 63:

      ST_k   S^T_k  = K Q_k^T        M 128 keys, N 64 queries, K 128 d (SS)
      EXB_k  P^T_k  = exp2(S^T_k - LSE)  -> bf16 over S^T_k        (MUFU)
      DP_k   dP^T_k = V dO_k^T       M 128, N 64, K 128 (SS)
      DS_k   dS^T_k = P^T_k (dP^T_k - D) -> bf16 over dP^T_k and to smem
      DV_k   dV    += P^T_k dO_k     M 128 keys, N 128 d, K 64 (TS)
      DK_k   dK    += dS^T_k Q_k     M 128, N 128, K 64 (TS)
      DQ_k   dQ^T_k = K^T dS^T_k     M 128 d, N 64 queries, K 128 keys (SS)
      RD_k   dQ^T_k -> smem (transposed) -> TMA reduce-add into fp32 dQ

    Tensor memory (512 columns): dK 128, dV 128, and per sub-tile 128: S^T_k
    (64, P^T_k over it, then dQ^T_k over it once DV_k has read P^T_k) and
    dP^T_k (64, dS^T_k over it). Aliasing edges: DV_k -> DQ_k (in order on
    the issuing thread), RD_k -> ST_k (delta 1: S^T_k(i+1) overwrites the
    dQ^T_k RD_k(i) reads), DK_k -> DP_k (delta 1, in order), DQ_k -> DS_k
    (delta 1: dS^T_k(i+1) overwrites the shared-memory operand DQ_k(i)
    reads), RD_k -> DS_k (delta 1: RD_k stages dQ^T_k in that buffer).
    EXB_k -> DS_k carries P^T_k in registers (a large spill cost keeps them
    on one warpgroup); a 192-register budget per warp keeps the two sub-tiles'
    EXB / DS on different warpgroups.
    Raw costs (B200 clk, multiples of 256 so the normalization is exact at
    U = 14): SS GEMMs with N = 64 read 6 KiB of shared memory per 32-clk
    K-step (192 B/clk against 128): 384, priced 512; TS GEMMs 256; EXB 768
    (8192 exp2 at 16/clk + the S^T read); DS 512; RD 512; spill 2048."""
    ss, ts, ex, dsc, rd = 512, 256, 768, 512, 512
    machine = {
        "units": [{"name": "TC", "capacity": 1}, {"name": "TMA", "capacity": 1},
                  {"name": "MUFU", "capacity": 1}, {"name": "ALU", "capacity": 1},
                  {"name": "FMA", "capacity": 1}],
        "memories": [{"name": "tmem", "capacity": 512}],
        "num_warps": 16,
        "reg_limit": 192,
        "vl_warp": 15,
    }
    nodes = [node("LDQ", "TMA", 256, variable_latency=True), node("LDO", "TMA", 256, variable_latency=True)]
    edges = []
    for k in (0, 1):
        nodes += [
            node(f"ST{k}", "TC", ss, footprint={"tmem": 64}, variable_latency=True),
            node(f"DP{k}", "TC", ss, footprint={"tmem": 64}, variable_latency=True),
            node(f"EXB{k}", "MUFU", ex, regs=128, spill_cost=2048, warps_required=4),
            node(f"DS{k}", "FMA", dsc, regs=64, warps_required=4),
            node(f"DV{k}", "TC", ts, variable_latency=True),
            node(f"DK{k}", "TC", ts, variable_latency=True),
            node(f"DQ{k}", "TC", ss, variable_latency=True),
            node(f"RD{k}", "ALU", rd, regs=64, warps_required=4),
        ]
        edges += [
            edge("LDQ", f"ST{k}", 0, blocking=True), edge("LDQ", f"DK{k}", 0, blocking=True),
            edge("LDO", f"DP{k}", 0, blocking=True), edge("LDO", f"DV{k}", 0, blocking=True),
            edge(f"ST{k}", f"EXB{k}", ss, blocking=True),
            edge(f"EXB{k}", f"DV{k}", ex, blocking=True), edge(f"EXB{k}", f"DS{k}", ex),
            edge(f"DP{k}", f"DS{k}", ss, blocking=True),
            edge(f"DS{k}", f"DK{k}", dsc, blocking=True), edge(f"DS{k}", f"DQ{k}", dsc, blocking=True),
            edge(f"DQ{k}", f"RD{k}", ss, blocking=True),
            edge(f"DV{k}", f"DQ{k}", 0),
            edge(f"RD{k}", f"ST{k}", rd, delta=1, blocking=True),
            edge(f"DK{k}", f"DP{k}", 0, delta=1),
            edge(f"DQ{k}", f"DS{k}", ss, delta=1, blocking=True),
            edge(f"RD{k}", f"DS{k}", rd, delta=1, blocking=True),
            edge(f"EXB{k}", f"EXB{k}", ex, delta=1), edge(f"DS{k}", f"DS{k}", dsc, delta=1),
            edge(f"RD{k}", f"RD{k}", rd, delta=1),
        ]
    for n in nodes:
        n["rrt"] = {u: [1] * n["cycles"] for u in n["rrt"]}
    return {"machine": machine, "graph": {"nodes": nodes, "edges": edges}}


def gemm_problem():
    """GEMM mainloop (BASELINE config 2): per k-block, TMA loads of the A and B
    tiles feed one 256x256x64 tcgen05 MMA chain (cta_group::2: a CTA pair on
    two SMs, each holding 128 rows of A and 128 rows of B) into a TMEM
    accumulator. Per SM 128x256x64 = 2 MMAC = 512 clk on TC; TMA of 32 KiB
    per SM per k-block."""
    T = 512
    machine = {
        "units": [{"name": "TC", "capacity": 1}, {"name": "TMA", "capacity": 1}],
        "memories": [{"name": "smem", "capacity": 6}],
        "num_warps": 2,
        "reg_limit": 0,
        "vl_warp": 1,
    }
    nodes = [
        node("LDA", "TMA", T, variable_latency=True, footprint={"smem": 1}),
        node("LDB", "TMA", T, variable_latency=True, footprint={"smem": 1}),
        node("MMA", "TC", T),
    ]
    nodes[0]["rrt"] = {"TMA": [1] * T}
    nodes[1]["rrt"] = {"TMA": [1] * T}
    edges = [
        edge("LDA", "MMA", 0, blocking=True),
        edge("LDB", "MMA", 0, blocking=True),
        edge("MMA", "MMA", T, delta=1),
    ]
    return {"machine": machine, "graph": {"nodes": nodes, "edges": edges}}


def load_ref():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    import _weftsched  # noqa: E402  (oracle: the unmodified reference)
    return _weftsched


def solver_version(solver):
    """`z3 --version` of the external backend (pinned with the schedule)."""
    if not solver or solver == "internal":
        return "internal DPLL (solverio.cpp)"
    exe = solver.split()[0]
    cand = os.path.join(os.path.dirname(sys.executable), exe)
    try:
        out = subprocess.run([cand if os.path.exists(cand) else exe, "--version"], capture_output=True, text=True,
                             timeout=30).stdout.strip()
    except OSError as e:
        out = f"unavailable: {e}"
    return out


def solve(name, raw, resolution, stream_depth, solver=""):
    w = load_ref()
    os.makedirs(OUT, exist_ok=True)
    raw_text = json.dumps(raw, indent=2) + "\n"
    open(os.path.join(OUT, name + ".raw.json"), "w").write(raw_text)
    t0 = time.time()
    norm = w.normalize(raw_text, resolution)
    t1 = time.time()
    prob = json.dumps(json.loads(norm["problem"]), indent=2) + "\n"
    open(os.path.join(OUT, name + ".json"), "w").write(prob)
    r = w.joint(prob, 0, stream_depth, solver)
    t2 = time.time()
    meta = {
        "resolution": resolution,
        "cost_map": {str(k): v for k, v in norm["cost_map"].items()},
        "F": norm["F"],
        "backend": solver or "internal",
        "backend_version": solver_version(solver),
        # SolveOptions defaults of the reference binding (solverio.hpp:75-81;
        # py_joint, bindings/module.cpp:95-101): only external_command is set
        "max_decisions": 28,
        "stream_depth": stream_depth,
        "normalize_s": round(t1 - t0, 4),
        "joint_s": round(t2 - t1, 4),
        "status": r["status"],
    }
    if r["status"] != "sat":
        meta["message"] = r.get("message")
        print(name, json.dumps(meta), file=sys.stderr)
        return meta
    open(os.path.join(OUT, name + ".solution.json"), "w").write(r["solution_json"])
    listing = w.codegen(prob, r["solution_json"], "text")
    open(os.path.join(OUT, name + ".listing.txt"), "w").write(listing)
    meta.update({"I": r["I"], "L": r["L"], "M": r["M"], "A": r["A"]})
    meta["validate"] = w.validate(prob, r["solution_json"])
    json.dump(meta, open(os.path.join(OUT, name + ".meta.json"), "w"), indent=2)
    print(name, json.dumps(meta))
    return meta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--resolution", type=int, default=7)
    ap.add_argument("--solver", default="")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    # name: (raw problem, stream depth, normalization resolution U or None = --resolution)
    probs = {
        "gemm_mainloop": (gemm_problem(), 6, None),  # 32 KiB stages per SM (CTA pair)
        # production: tcgen05.mma modeled as variable latency (see
        # fa_forward_problem) with the B200-calibrated costs (EX 6, MX 2
        # units of 256 clk, measured by the in-kernel trace); U = 9 normalizes
        # {256, 512, 1536} exactly (F = 0)
        "fa_fwd": (fa_forward_problem(tc_variable_latency=True, calibrated=True), 2, 9),
        # (stream_depth 3 and 4 give the same M / A with deeper K / V rings,
        # which fit with the CTA-pair realization: measured equal, not kept;
        # profiles/r02c_notes.md)
        # variable latency with the datasheet costs (EX 4, MX 1)
        "fa_fwd_vl": (fa_forward_problem(tc_variable_latency=True), 2, None),
        # comparison: MMAs as fixed-latency ops (the solver scatters them over warps)
        "fa_fwd_fixedtc": (fa_forward_problem(), 2, None),
        "fa_fwd_cal": (fa_forward_problem(calibrated=True), 2, 9),
        # production model with S_k split into SA_k + SB_k (half of S(i+1) overlaps EX(i))
        "fa_fwd_split": (fa_forward_problem(tc_variable_latency=True, calibrated=True, split_s=True), 2, 9),
        # double-buffered S (64-key K/V tiles): S_k(i+1) independent of PV_k(i)
        "fa_fwd_ring2": (fa_forward_problem(tc_variable_latency=True, s_ring=2), 4, None),
        # FA backward (single pass, K/V-stationary), datasheet costs; P^T
        # carried in registers from EXB to DS (a large spill cost keeps them
        # on one warpgroup)
        "fa_bwd": (fa_backward_problem(), 2, 11),  # {512, 1024, 4096} clk exactly (F = 0)
        # EXB's consumers read P^T through tensor memory behind an mbarrier
        # (spill cost 256 clk): the solver splits EXB and DS over two
        # warpgroups and pipelines across iterations (I = 12 x 256 clk); the
        # realized loop is slower (DESIGN 12: the dS / dQ-staging buffer)
        "fa_bwd_split": (fa_backward_problem(exb_spill=1), 2, 13),
        # the split model with dQ staged in the Q ring slot (no RD -> DS chain)
        "fa_bwd_qstage": (fa_backward_problem(exb_spill=1, q_staging=True), 2, 13),
        "fa_bwd_cal": (fa_backward_problem(calibrated=True), 2, 14),
        # two 64-query sub-tiles per iteration, ping-ponging EXB / DS warpgroups
        "fa_bwd_pp": (fa_backward_pp_problem(), 2, 14),
    }
    for name, (raw, depth, res) in probs.items():
        if args.only and name != args.only:
            continue
        if args.solve:
            solve(name, raw, res or args.resolution, depth, args.solver)
        else:
            print(json.dumps(raw, indent=2))


if __name__ == "__main__":
    main()
