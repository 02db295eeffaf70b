// FA-backward on sm_100a, realized from a Twill joint schedule.
//
// The paper's second workload: the single-pass backward
// of FA3 -- five GEMMs, one exponential, and an atomic reduction of dQ into
// global memory. The loop graph is tools/make_problems.py:fa_backward_problem;
// its solution (schedules/fa_bwd.solution.json, z3) gives the warp roles and
// the issue order that the lowering (lowering.cpp:derive_bwd) turns into the
// per-warp trip programs this kernel walks.
//
// One CTA owns a 128-key K/V tile of one (b, h) -- K and V stay in shared
// memory, dK and dV accumulate in tensor memory -- and iterates over the
// 128-row Q tiles i (causal: the tiles on and below the diagonal):
//   LDQ, LDO  Q_i, dO_i -> smem rings (TMA)
//   ST        S^T  = K Q_i^T            TMEM cols 256.. (keys on lanes)
//   EXB       P^T  = exp2(S^T * scale*log2e - LSE_i*log2e) -> bf16 over S^T
//   DP        dP^T = V dO_i^T           TMEM cols 384..
//   DS        dS^T = P^T (dP^T - D_i)   -> bf16 over dP^T, and into smem
//             (MN-major, the A operand of DQ); P^T stays in registers
//   DV        dV  += P^T dO_i           TS, TMEM cols 128..
//   DK        dK  += dS^T Q_i           TS, TMEM cols 0..
//   DQ        dQ_i = dS K               SS (A MN-major) -> TMEM cols 384..
//   RD        dQ_i (fp32) -> smem -> TMA reduce-add into the global dQ
//             accumulator
// after the last tile: dK * scale, dV -> bf16 -> global (RD warpgroup).
// A pre-pass computes D_i = rowsum(dO_i * O_i); a post-pass scales dQ.
//
// Every cross-warp edge of the loop graph is an mbarrier; the aliasing edges
// (DV -> ST(i+1): S^T(i+1) overwrites P^T(i); DK -> DQ: dQ_i overwrites
// dS^T) are realized by tcgen05 in-order execution on the single issuing
// thread, which the lowering checks. S^T(i+1) never waits for the dQ_i
// read-out, so the next tile's exponentials overlap this tile's DS .. RD.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "fa_bwd.h"
#include "sm100.cuh"

namespace twfa {

namespace {

constexpr int kT = 128;                 // keys per K/V tile = rows per Q tile
constexpr uint32_t kTile = 32768;       // 128 x 128 bf16: two 64-column SW128 halves
constexpr uint32_t kHalf = 16384;
constexpr uint32_t kColDK = 0, kColDV = 128, kColS = 256, kColP = 384;  // TMEM columns
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kIdescKK = idesc_bf16_f32(128, 128, 0);  // A, B K-major
constexpr uint32_t kIdescKM = idesc_bf16_f32(128, 128, 1);  // A K-major (or TMEM), B MN-major
constexpr uint32_t kIdescMM = idesc_bf16_f32(128, 128, 1) | (1u << 15);  // A and B MN-major
constexpr uint32_t kSdHi = sdesc_hi(1024);
// timing-only experiments (results WRONG when set): 1 = RD skips the
// reduce-add; 2 = no shared-memory traffic from DS (dS) and RD (staging)
#ifndef TWFA_BWD_WHATIF
#define TWFA_BWD_WHATIF 0
#endif
// dQ reduction: 0 = staged through shared memory (the dS buffer) and
// cp.reduce.async.bulk.tensor; 1 = red.global.add.v4.f32 straight from
// registers (no staging buffer, so DS(i+1) does not wait for RD(i))
#ifndef TWFA_BWD_RED
#define TWFA_BWD_RED 0
#endif
// debug variant: CTA 0 prints per-op enter / exit clocks of iterations 20-21
// Skip an MMA-warp wait on a barrier phase this warp already saw complete
// (DK / DQ / DV after ST / DP / DK of the same iteration). An mbarrier wait
// costs the MMA warp ~160 clk even on a completed phase, and it queues behind
// the warp's own tcgen05 instructions, so each redundant wait delays the
// next op's issue while the tensor core drains its short queue.
#ifndef TWFA_BWD_MEMO
#define TWFA_BWD_MEMO 0  // measured neutral (688 vs 690); off: every p_full phase keeps a waiter (synccheck)
#endif
// RD reads the whole dQ_i row out of tensor memory before staging it
// (TWFA_BWD_RD_FULL), so q_free -- which DP_(i+1) waits for -- is signalled
// right after the read instead of after half of the staging and reduction
#ifndef TWFA_BWD_RD_FULL
#define TWFA_BWD_RD_FULL 0  // measured with TWFA_BWD_FIXED: 749 vs 766-770 TF/s (C3 shape)
#endif
#ifndef TWFA_BWD_CDEPTH
#define TWFA_BWD_CDEPTH 1
#endif
#ifndef TWFA_BWD_HEAVY_SPEC
#define TWFA_BWD_HEAVY_SPEC 1
#endif
#ifndef TWFA_BWD_CFLAGS
#define TWFA_BWD_CFLAGS 1
#endif
#ifndef TWFA_BWD_FIXED
#define TWFA_BWD_FIXED 1
#endif
#ifndef TWFA_BWD_SOLO
#define TWFA_BWD_SOLO 0  // measured: 680 vs 693 TF/s (C3); with the loads on warp 14 699
#endif
#ifndef TWFA_BWD_LOAD_WARP
#define TWFA_BWD_LOAD_WARP -1
#endif
#ifndef TWFA_BWD_PROF
#define TWFA_BWD_PROF 0
#endif

struct __align__(8) BwdBarriers {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[2], q_empty[2], o_full[2], o_empty[2];
  uint64_t s_full, dp_full, dq_full;  // tcgen05.commit
  uint64_t p_full, ds_full;           // EXB / DS warpgroup (4 warp arrivals)
  uint64_t p_read;                    // DS on its own warpgroup read P^T back (4)
  uint64_t q_free;                    // RD warpgroup read dQ_i out of TMEM (4)
  uint64_t ds_free;                   // RD is done with the dS buffer as staging (1)
  uint64_t acc_full;                  // dK, dV final for the work item (commit)
  uint64_t acc_free;                  // RD warpgroup read dK, dV (4)
  uint32_t tmem_base;
};
__shared__ BwdBarriers g_bb;
// LSE * log2(e) and D of the current Q tile, broadcast to the EXB / DS
// warpgroup (thread t stages query q0 + t)
__shared__ __align__(16) float g_lse2[kT];
__shared__ __align__(16) float g_dvec[kT];
#if TWFA_BWD_PROF
__shared__ int g_prof_n;
__shared__ long long g_prof[24][4];
__device__ long long g_prof_ready;  // per-op "inputs ready" clock (MMA warp, debug variant)
#endif

struct BwdCtx {
  uint8_t* k;
  uint8_t* v;
  uint8_t* q;   // ring of Q tiles
  uint8_t* o;   // ring of dO tiles
  uint8_t* ds;  // dS (A operand of DQ), then the dQ staging of RD
  uint32_t warp, lane, quad, lane_off;
  int S, BH, nq, num_work;
  uint64_t pol;
};

struct BwdItem {
  int bh, kv0, q_first, N;  // N = Q tiles of this work item
  uint32_t gbase;           // global iteration index of its iteration 0
  uint32_t icount;          // work items done by this CTA
};

__device__ __forceinline__ BwdItem bwd_item(const BwdCtx& c, const FaBwdArgs& a, int work, uint32_t gbase,
                                            uint32_t icount) {
  BwdItem t;
  int j;
  if (a.causal) {  // K/V tile j sees Q tiles j..nq-1: longest first
    j = work / c.BH;
    t.bh = work % c.BH;
  } else {
    t.bh = work / c.nq;
    j = work % c.nq;
  }
  t.kv0 = j * kT;
  t.q_first = a.causal ? j : 0;
  t.N = c.nq - t.q_first;
  t.gbase = gbase;
  t.icount = icount;
  return t;
}

struct BwdState {
  int q_next, o_next;      // next Q / dO iteration to load (TMA warp)
  int q_target, o_target;  // loads the trip program has asked for so far
  uint32_t trace_n;        // records of this warp in the issue trace
  uint32_t* rec;           // the current op's trace record (t_ready stamped after its waits)
  // MMA warp: iteration + 1 whose Q_i / dO_i / P^T / dS^T this warp has already
  // seen land (TWFA_BWD_MEMO): a later op of the same iteration skips its wait
  uint32_t q_seen, o_seen, p_seen, ds_seen;
};
// t_ready of the current op's trace record: its inputs have been awaited
__device__ __forceinline__ void bwd_ready(BwdState& st) {
  if (st.rec != nullptr) st.rec[4] = static_cast<uint32_t>(clock64());
}

// Issue trace (CTA 0, lane 0 of every warp): one record per op instance,
// the same layout as the forward's (fa_fwd_kernel.cuh)
__device__ __forceinline__ uint32_t* bwd_trace(const FaBwdArgs& a, const BwdCtx& c, BwdState& st, int node, int it,
                                               int trip, const BwdItem& t) {
  if (a.trace == nullptr || blockIdx.x != 0 || c.lane != 0 || st.trace_n + 1 >= a.trace_cap) return nullptr;
  uint32_t* base = a.trace + static_cast<size_t>(c.warp) * a.trace_cap * 8;
  uint32_t* e = base + (st.trace_n + 1) * 8;
  e[0] = static_cast<uint32_t>(node);
  e[1] = static_cast<uint32_t>(it);
  e[2] = static_cast<uint32_t>(trip);
  e[3] = static_cast<uint32_t>(clock64());
  e[6] = t.icount;
  e[7] = static_cast<uint32_t>(t.N);
  base[0] = ++st.trace_n;
  return e;
}

// Streamed Q / dO loads (LDQ / LDO). A load issues at its trip-program
// position if its ring slot is already free; otherwise it is deferred
// instead of stalling the warp (the TMA warp is also the MMA warp, and the
// slot is released by an MMA commit that may still be in flight), retried
// before every later op of the warp, and forced only when an op needs that
// very iteration. Streamed loads are zero-cycle ops: issuing them anywhere
// between their slot and their consumer realizes the same schedule.
#ifndef TWFA_BWD_LAZY_LOADS
#define TWFA_BWD_LAZY_LOADS 0  // measured: 712 vs 764 TFLOP/s (C3 shape), eager is faster
#endif
template <bool kSolo, int kDepth = 0>
__device__ __forceinline__ void bwd_top_up(const BwdCtx& c, const FaBwdArgs& a, const BwdItem& t, BwdState& st,
                                           const TwfaDevicePlan& plan, bool is_q, int upto, bool blocking) {
  BwdBarriers& bar = g_bb;
  int& next = is_q ? st.q_next : st.o_next;
  const int depth = kDepth > 0 ? kDepth : is_q ? plan.k_depth : plan.v_depth;  // kDepth: known ring depth
  while (next <= upto) {
    const int lit = next;
    const uint32_t g = t.gbase + static_cast<uint32_t>(lit);
    const uint32_t s = g % depth, ph = (g / depth) & 1;
    uint64_t* empty = is_q ? &bar.q_empty[s] : &bar.o_empty[s];
    if (blocking) {
      mbar_wait(empty, ph ^ 1);
    } else if (kSolo ? !mbar_try_wait(empty, ph ^ 1) : !__all_sync(0xffffffffu, mbar_try_wait(empty, ph ^ 1))) {
      return;
    }
    ++next;
    uint64_t* full = is_q ? &bar.q_full[s] : &bar.o_full[s];
    if (lead<kSolo>()) {
      uint8_t* dst = (is_q ? c.q : c.o) + s * kTile;
      const CUtensorMap* map = is_q ? &a.tm_q : &a.tm_do;
      const int row = (t.q_first + lit) * kT;
      mbar_arrive_expect_tx(full, kTile);
      tma_load_3d(dst, map, full, 0, row, t.bh, c.pol);
      tma_load_3d(dst + kHalf, map, full, 64, row, t.bh, c.pol);
    }
    wsync<kSolo>();
  }
}

__device__ __forceinline__ uint32_t sd_lo(const void* p, uint32_t lbo) { return sdesc_lo(smem_u32(p), lbo); }

// Stage one per-query vector of the current Q tile (LSE * log2e or D) in
// shared memory for the warpgroup: thread t loads query q0 + t, the group
// synchronizes on its named barrier before (previous tile's readers done)
// and after the store.
__device__ __forceinline__ void stage_tile_vec(float* dst, float v, uint32_t r, uint32_t bar_id) {
  named_bar_sync(bar_id, 128);
  dst[r] = v;
  named_bar_sync(bar_id, 128);
}

// EXB: P^T row of this thread (key kv0 + r) for Q tile q0, stored to TMEM as
// bf16 over S^T; the fp32 values stay in p[] for a fused DS.
__device__ __forceinline__ void exb_part(const BwdCtx& c, const FaBwdArgs& a, const BwdItem& t, int it, uint32_t g,
                                         uint32_t (&p)[kT], BwdState& st) {
  BwdBarriers& bar = g_bb;
  const int q0 = (t.q_first + it) * kT;
  const uint32_t r = c.quad * 32 + c.lane;
  const int key = t.kv0 + static_cast<int>(r);
  const int64_t row0 = static_cast<int64_t>(t.bh) * c.S + q0;
  // this tile's LSE: one coalesced load per thread, issued before the S^T
  // wait, then broadcast through shared memory
  const int qt = q0 + static_cast<int>(r);
  const float my_lse2 = qt < c.S ? a.lse[row0 + r] * kLog2e : INFINITY;  // rows past S: P = 0
  mbar_wait(&bar.s_full, g & 1);
  tc_fence_after();
  bwd_ready(st);
  // chunk 0 of the S^T row first; the rest streams in from tensor memory
  // while chunk 0 is exponentiated (and while the LSE is staged)
  tmem_ld32(c.lane_off + kColS, *reinterpret_cast<uint32_t(*)[32]>(&p[0]));
  tmem_ld_wait();
#pragma unroll
  for (int cc = 1; cc < 4; ++cc)
    tmem_ld32(c.lane_off + kColS + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&p[cc * 32]));
  stage_tile_vec(g_lse2, my_lse2, r, 1 + (c.warp >> 2));
  // P^T[key][q] = exp2(S^T * scale*log2e - LSE_q * log2e)
  const float sl = a.scale_log2;
  const bool diag = a.causal && it == 0;  // the diagonal tile (q0 == kv0)
#pragma unroll
  for (int j4 = 0; j4 < kT / 4; ++j4) {
    if (j4 == 8) tmem_ld_wait();  // chunks 1..3
    const float4 l = reinterpret_cast<const float4*>(g_lse2)[j4];
    const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 4 * j4 + u;
      float e = fast_exp2(fmaf(__uint_as_float(p[j]), sl, -lv[u]));
      if (diag && key > q0 + j) e = 0.f;
      p[j] = __float_as_uint(e);
    }
  }
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      pk[i] = pack_bf16(__uint_as_float(p[cc * 32 + 2 * i]), __uint_as_float(p[cc * 32 + 2 * i + 1]));
    tmem_st16(c.lane_off + kColS + cc * 16, pk);
  }
  tmem_st_wait();
  tc_fence_before();
  warp_arrive(&bar.p_full);
}

// DS: dS^T = P^T (dP^T - D_q), chunk by chunk over the dP^T columns; the
// bf16 chunk goes to TMEM (over dP^T columns already read) for DK and to the
// smem A operand of DQ (MN-major: row = key, 64 queries per SW128 half).
// kFused: P^T in fp32 registers from the EXB just before on this warpgroup;
// otherwise DS runs on its own warpgroup and reads P^T (bf16) back from
// tensor memory first, then releases the columns to S^T(i+1) (p_read).
template <bool kFused>
__device__ __forceinline__ void ds_part(const BwdCtx& c, const FaBwdArgs& a, const BwdItem& t, int it, uint32_t g,
                                        const uint32_t (&p)[kT]) {
  BwdBarriers& bar = g_bb;
  const int q0 = (t.q_first + it) * kT;
  const uint32_t r = c.quad * 32 + c.lane;
  const int64_t row0 = static_cast<int64_t>(t.bh) * c.S + q0;
  const int qt = q0 + static_cast<int>(r);
  const float my_d = qt < c.S ? a.dvec[row0 + r] : 0.f;
  uint32_t pp[kFused ? 1 : kT / 2];  // packed bf16 P^T (unfused)
  if constexpr (!kFused) {
    mbar_wait(&bar.p_full, g & 1);
    tc_fence_after();
    tmem_ld32(c.lane_off + kColS, *reinterpret_cast<uint32_t(*)[32]>(&pp[0]));
    tmem_ld32(c.lane_off + kColS + 32, *reinterpret_cast<uint32_t(*)[32]>(&pp[32]));
    tmem_ld_wait();
    tc_fence_before();
    warp_arrive(&bar.p_read);
  }
  if (g > 0) mbar_wait(&bar.ds_free, (g - 1) & 1);
  stage_tile_vec(g_dvec, my_d, r, 1 + (c.warp >> 2));
  mbar_wait(&bar.dp_full, g & 1);
  tc_fence_after();
  const uint32_t ds_base = smem_u32(c.ds) + r * 128;
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t dp[32];
    tmem_ld32(c.lane_off + kColP + cc * 32, dp);
    tmem_ld_wait();
    uint32_t pk[16];
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4) {
      const int j = cc * 32 + 4 * j4;
      const float4 d = reinterpret_cast<const float4*>(g_dvec)[j / 4];
      float pv[4];
      if constexpr (kFused) {
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = __uint_as_float(p[j + u]);
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t w = pp[j / 2 + u];
          pv[2 * u] = __uint_as_float(w << 16);
          pv[2 * u + 1] = __uint_as_float(w & 0xffff0000u);
        }
      }
      const float s0 = pv[0] * (__uint_as_float(dp[4 * j4 + 0]) - d.x);
      const float s1 = pv[1] * (__uint_as_float(dp[4 * j4 + 1]) - d.y);
      const float s2 = pv[2] * (__uint_as_float(dp[4 * j4 + 2]) - d.z);
      const float s3 = pv[3] * (__uint_as_float(dp[4 * j4 + 3]) - d.w);
      pk[2 * j4] = pack_bf16(s0, s1);
      pk[2 * j4 + 1] = pack_bf16(s2, s3);
    }
    tmem_st16(c.lane_off + kColP + cc * 16, pk);
    // queries 32cc .. 32cc+31: SW128 half cc/2, 16-byte chunks 4(cc%2) .. +3
    if (TWFA_BWD_WHATIF == 2) continue;  // timing only: no dS in shared memory
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint32_t ch = (cc & 1) * 4 + m;
      st_shared_v4(ds_base + (cc >> 1) * kHalf + ((ch ^ (r & 7)) << 4), pk[4 * m], pk[4 * m + 1], pk[4 * m + 2],
                   pk[4 * m + 3]);
    }
  }
  tmem_st_wait();
  tc_fence_before();
  fence_proxy_async_shared();
  warp_arrive(&bar.ds_full);
}

// RD: dQ_i from TMEM (row = query) -> smem staging (fp32, SW128 boxes of
// 128 rows x 32 columns) -> cp.reduce.async.bulk add into the fp32 dQ
// accumulator (the atomic reduction of the paper's backward loop).
template <bool kFull, bool kKnown = false>
__device__ __forceinline__ void rd_op(const BwdCtx& c, const FaBwdArgs& a, const BwdItem& t, int it, uint32_t g,
                                      const TwfaDevicePlan& plan, BwdState& st) {
  // staging buffer: Q_i's ring slot when the schedule says so (plan.s_split
  // for the backward family; DK_i is complete once DQ_i is), else dS's.
  // kKnown: the specialized kernel's host-checked plan (dS staging, depth 2)
  const bool q_stage = kKnown ? false : plan.s_split != 0;
  const uint32_t qs = g % (kKnown ? 2u : static_cast<uint32_t>(plan.k_depth));
  uint8_t* const stage_buf = q_stage ? c.q + qs * kTile : c.ds;
  BwdBarriers& bar = g_bb;
  const int q0 = (t.q_first + it) * kT;
  const uint32_t r = c.quad * 32 + c.lane;
  const bool leader = (c.warp & 3u) == 0 && c.lane == 0;
  const uint32_t nb = 1 + (c.warp >> 2);  // named barrier of this warpgroup
  mbar_wait(&bar.dq_full, g & 1);
  tc_fence_after();
  bwd_ready(st);
  if (TWFA_BWD_RED) {
    // the dS buffer is not used for staging: DS(i+1) may proceed (with Q-slot
    // staging DQ's commit frees it, and RD releases the unused Q slot)
    if (leader) mbar_arrive(q_stage ? &bar.q_empty[qs] : &bar.ds_free);
    float* dst = a.dq_acc + (static_cast<int64_t>(t.bh) * c.S + q0 + r) * 128;
    const bool in = q0 + static_cast<int>(r) < c.S;
#pragma unroll 1
    for (int h = 0; h < 4; ++h) {
      uint32_t v[32];
      tmem_ld32(c.lane_off + kColP + h * 32, v);
      tmem_ld_wait();
      if (h == 3) {
        tc_fence_before();
        warp_arrive(&bar.q_free);
      }
      if (in) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + h * 32 + 4 * j),
                       "f"(__uint_as_float(v[4 * j])), "f"(__uint_as_float(v[4 * j + 1])),
                       "f"(__uint_as_float(v[4 * j + 2])), "f"(__uint_as_float(v[4 * j + 3]))
                       : "memory");
      }
    }
    return;
  }
  if (TWFA_BWD_WHATIF == 2) {  // timing only: read dQ_i out, no staging / reduction
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      uint32_t v[64];
      tmem_ld32(c.lane_off + kColP + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      tmem_ld32(c.lane_off + kColP + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      asm volatile("" ::"r"(v[0]), "r"(v[63]));
    }
    tc_fence_before();
    warp_arrive(&bar.q_free);
    if (leader) mbar_arrive(q_stage ? &bar.q_empty[qs] : &bar.ds_free);
    return;
  }
  if constexpr (kFull) {
    // the whole dQ_i row comes out of tensor memory first (128 registers),
    // so DP_(i+1) may overwrite the columns before any staging starts; the
    // four 32-column boxes then alternate over the two staging halves
    uint32_t v[128];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      tmem_ld32(c.lane_off + kColP + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[cc * 32]));
    tmem_ld_wait();
    tc_fence_before();
    warp_arrive(&bar.q_free);
#pragma unroll
    for (int box = 0; box < 4; ++box) {
      const int hb = box & 1;
      if (box >= 2) {
        if (leader) bulk_wait_read_1();  // the reduce of box - 2 has read this half
        named_bar_sync(nb, 128);
      }
      const uint32_t base = smem_u32(stage_buf) + hb * kHalf + r * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        st_shared_v4(base + ((ch ^ (r & 7)) << 4), v[box * 32 + 4 * ch], v[box * 32 + 4 * ch + 1],
                     v[box * 32 + 4 * ch + 2], v[box * 32 + 4 * ch + 3]);
      fence_proxy_async_shared();
      named_bar_sync(nb, 128);
      if (leader) {
        tma_reduce_add_3d(&a.tm_dq, stage_buf + hb * kHalf, 32 * box, q0, t.bh);
        bulk_commit();
      }
    }
    if (leader) {
      bulk_wait_read();
      mbar_arrive(q_stage ? &bar.q_empty[qs] : &bar.ds_free);
    }
    return;
  }
  // DQ_i has completed (dq_full): the dS buffer is free for staging. Its two
  // 16 KiB halves alternate as staging for the four 32-column boxes of the
  // dQ tile, so the bulk reduction of one box overlaps the staging of the
  // next; the row is read in two 64-column halves (64 registers).
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    uint32_t v[64];
    tmem_ld32(c.lane_off + kColP + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
    tmem_ld32(c.lane_off + kColP + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
    tmem_ld_wait();
    if (h == 1) {
      tc_fence_before();
      warp_arrive(&bar.q_free);  // dP^T(i+1) may overwrite the columns
    }
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int box = 2 * h + hb;  // staging half = hb
      if (box >= 2) {
        if (leader) bulk_wait_read_1();  // the reduce of box - 2 has read this half
        named_bar_sync(nb, 128);
      }
      const uint32_t base = smem_u32(stage_buf) + hb * kHalf + r * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        st_shared_v4(base + ((ch ^ (r & 7)) << 4), v[hb * 32 + 4 * ch], v[hb * 32 + 4 * ch + 1],
                     v[hb * 32 + 4 * ch + 2], v[hb * 32 + 4 * ch + 3]);
      fence_proxy_async_shared();
      named_bar_sync(nb, 128);
      if (leader) {
        if (TWFA_BWD_WHATIF != 1) tma_reduce_add_3d(&a.tm_dq, stage_buf + hb * kHalf, 32 * box, q0, t.bh);
        bulk_commit();
      }
    }
  }
  if (leader) {
    bulk_wait_read();
    mbar_arrive(q_stage ? &bar.q_empty[qs] : &bar.ds_free);
  }
}

// dK (scaled) and dV of the work item: TMEM (row = key) -> bf16 -> global
__device__ __forceinline__ void kv_epilogue(const BwdCtx& c, const FaBwdArgs& a, const BwdItem& t) {
  BwdBarriers& bar = g_bb;
  mbar_wait(&bar.acc_full, t.icount & 1);
  tc_fence_after();
  const int key = t.kv0 + static_cast<int>(c.quad * 32 + c.lane);
  const int64_t off = (static_cast<int64_t>(t.bh) * c.S + key) * 128;
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    const uint32_t col = which == 0 ? kColDK : kColDV;
    const float mul = which == 0 ? a.scale : 1.f;
    __nv_bfloat16* dst = (which == 0 ? a.dk : a.dv) + off;
#pragma unroll 1
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t x[32];
      tmem_ld32(c.lane_off + col + cc * 32, x);
      tmem_ld_wait();
      if (key < c.S) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(x[8 * i + 0]) * mul, __uint_as_float(x[8 * i + 1]) * mul);
          w.y = pack_bf16(__uint_as_float(x[8 * i + 2]) * mul, __uint_as_float(x[8 * i + 3]) * mul);
          w.z = pack_bf16(__uint_as_float(x[8 * i + 4]) * mul, __uint_as_float(x[8 * i + 5]) * mul);
          w.w = pack_bf16(__uint_as_float(x[8 * i + 6]) * mul, __uint_as_float(x[8 * i + 7]) * mul);
          d4[i] = w;
        }
      }
    }
  }
  tc_fence_before();
  warp_arrive(&bar.acc_free);
}

// Register classes (each compiled under its setmaxnreg budget): the TMA / MMA
// warps, the RD warpgroup (RD + the dK / dV epilogue), and the EXB and DS
// warpgroups -- one warpgroup running both (P^T carried in registers) or
// one each (DS reads P^T back from tensor memory), as the schedule places
// them.
enum BwdRole { kLight = 0, kReduce = 1, kExbDs = 2, kExb = 3, kDs = 4, kReduceFull = 5, kLightSolo = 6 };
// kLightSolo: the TMA / MMA warp's trip program runs on one elected lane
// (TWFA_BWD_SOLO). Measured (tools/calib/ubench_mmaloop.cu): a warp that
// waits, elects a lane for each op's MMAs and re-converges with __syncwarp
// keeps the tensor core 65-72 % busy on 8-MMA ops of 64 clk each; one lane
// issuing the same ops (with the same waits) keeps it 89-96 % busy. In the
// kernels it does not carry over (backward 680 vs 693 TF/s, forward -4 to
// -9 % per clock), so both default to the warp-wide form.
__host__ __device__ constexpr bool is_light(int role) { return role == kLight || role == kLightSolo; }

// dS^T(g) has landed. With EXB and DS on one warpgroup, the same warps
// arrived P^T(g) (p_full) before dS^T(g) (ds_full), so P^T(g) has landed too.
__device__ __forceinline__ void bwd_wait_ds(BwdState& st, const TwfaDevicePlan& plan, uint32_t g) {
  mbar_wait(&g_bb.ds_full, g & 1);
  st.ds_seen = g + 1;
  if (plan.sm_warp[0] == plan.sm_warp[1]) st.p_seen = g + 1;
}

// One op of the trip program on this warp, trip r.
template <int kRole, int kKind = -1, bool kTrace = true>
__device__ __forceinline__ void bwd_exec(const TwfaPlanOp op, const int r, const BwdCtx& c, const BwdItem& t,
                                         BwdState& st, const TwfaDevicePlan& plan, const FaBwdArgs& a) {
  BwdBarriers& bar = g_bb;
  // kKind >= 0: a call site that knows the op's kind at compile time (the
  // TMA / MMA warp's fixed program, TWFA_BWD_FIXED): every other branch folds
  const int kind = kKind >= 0 ? kKind : static_cast<int>(op.kind);
  if (kind == TWFA_OP_LDQ || kind == TWFA_OP_LDO) {
    if constexpr (is_light(kRole)) {
      const bool is_q = kind == TWFA_OP_LDQ;
      const int target = (kKind >= 0 && TWFA_BWD_CFLAGS)
                             ? min(t.N - 1, r + 1)  // stage 0, prefetch 1: host-checked
                             : min(t.N - 1, r - static_cast<int>(op.stage) + (is_q ? plan.k_prefetch : plan.v_prefetch));
      (is_q ? st.q_target : st.o_target) = target;
      const int before = is_q ? st.q_next : st.o_next;
      if constexpr (kKind >= 0 && TWFA_BWD_CDEPTH) bwd_top_up<kRole == kLightSolo, 2>(c, a, t, st, plan, is_q, target, !TWFA_BWD_LAZY_LOADS);
      else bwd_top_up<kRole == kLightSolo>(c, a, t, st, plan, is_q, target, !TWFA_BWD_LAZY_LOADS);
      if (kTrace && a.trace != nullptr)
        for (int lit = before; lit < (is_q ? st.q_next : st.o_next); ++lit) {
          uint32_t* e = bwd_trace(a, c, st, op.node, lit, r, t);
          if (e) e[5] = e[3];
        }
    }
    return;
  }
  if constexpr (is_light(kRole)) {
    if (TWFA_BWD_LAZY_LOADS) {  // deferred loads: retry without blocking
      bwd_top_up<kRole == kLightSolo>(c, a, t, st, plan, true, st.q_target, false);
      bwd_top_up<kRole == kLightSolo>(c, a, t, st, plan, false, st.o_target, false);
    }
  }
  const int it = r - ((kKind >= 0 && TWFA_BWD_CFLAGS) ? 0 : static_cast<int>(op.stage));  // stage 0: host-checked
  if (it < 0 || it >= t.N) return;
  const uint32_t g = t.gbase + static_cast<uint32_t>(it);
  // one record per op instance; t_done stamped when the op body returns
  struct TraceDone {
    uint32_t* e;
    __device__ ~TraceDone() {
      if (e) e[5] = static_cast<uint32_t>(clock64());
    }
  } trace_done_{kTrace && a.trace != nullptr ? bwd_trace(a, c, st, op.node, it, r, t) : nullptr};
  st.rec = trace_done_.e;
#if TWFA_BWD_PROF
  const bool prof = blockIdx.x == 0 && c.lane == 0 && (c.warp & 3u) == 3 && t.icount == 0 && (it == 20 || it == 21);
  struct Out {
    bool on; int kind, it; long long t0;
    __device__ ~Out() {
      if (on) {
        const int n = atomicAdd(&g_prof_n, 1);
        if (n < 24) {
          g_prof[n][0] = (int)(threadIdx.x / 32) * 1000 + kind * 10 + (it - 20);
          g_prof[n][1] = t0;
          g_prof[n][2] = clock64();
          g_prof[n][3] = g_prof_ready;
        }
      }
    }
  } out_{prof, op.kind, it, clock64()};
#endif
  if (kind == TWFA_OP_EXB || kind == TWFA_OP_DS) {
    if constexpr (kRole == kExbDs || kRole == kExb || kRole == kDs) {
      uint32_t p[kT];
      if (kind == TWFA_OP_EXB) {
        exb_part(c, a, t, it, g, p, st);
        if constexpr (kRole == kExbDs) ds_part<true>(c, a, t, it, g, p);  // fused (lowering guarantees)
      } else if constexpr (kRole == kDs) {
        ds_part<false>(c, a, t, it, g, p);
      }
    }
    return;
  }
  if (kind == TWFA_OP_RD) {
    if constexpr (kRole == kReduce || kRole == kReduceFull)
      rd_op<kRole == kReduceFull, kKind >= 0 && TWFA_BWD_CFLAGS>(c, a, t, it, g, plan, st);
    return;
  }
  if constexpr (!is_light(kRole)) return;
  constexpr bool kSolo = kRole == kLightSolo;
  // tensor-core ops: warp-uniform descriptors, one elected lane issues
  if (TWFA_BWD_LAZY_LOADS) {  // a deferred load this op needs is forced now
    if (kind == TWFA_OP_ST || kind == TWFA_OP_DK) bwd_top_up<kRole == kLightSolo>(c, a, t, st, plan, true, it, true);
    if (kind == TWFA_OP_DP || kind == TWFA_OP_DV) bwd_top_up<kRole == kLightSolo>(c, a, t, st, plan, false, it, true);
  }
  // ring depths: compile-time 2 on the fixed production program (checked
  // before it is taken), the plan's otherwise
  const uint32_t kd = kKind >= 0 && TWFA_BWD_CDEPTH ? 2u : static_cast<uint32_t>(plan.k_depth);
  const uint32_t vd = kKind >= 0 && TWFA_BWD_CDEPTH ? 2u : static_cast<uint32_t>(plan.v_depth);
  const uint32_t qs = g % kd, os = g % vd;
  // the fixed production program's flags are host-checked (bwd_fixed_program):
  // DK releases Q_i, DV releases dO_i, nothing else releases or waits on p_read
  const bool release = (kKind >= 0 && TWFA_BWD_CFLAGS) ? (kind == TWFA_OP_DK || kind == TWFA_OP_DV)
                                                      : static_cast<bool>(op.flags & TWFA_OPF_RELEASE);
  if (kind == TWFA_OP_ST) {
    if (it == 0) mbar_wait(&bar.kv_full, t.icount & 1);
    // P^T(g-1) was read by DV(g-1) (in order) and, with DS on its own
    // warpgroup, by DS(g-1) (p_read)
    if (g > 0 && !(kKind >= 0 && TWFA_BWD_CFLAGS) && (op.flags & TWFA_OPF_WAIT_PREAD))
      mbar_wait_all(&bar.q_full[qs], (g / kd) & 1, &bar.p_read, (g - 1) & 1);
    else if (!(TWFA_BWD_MEMO && st.q_seen == g + 1))
      mbar_wait(&bar.q_full[qs], (g / kd) & 1);
    st.q_seen = g + 1;
    tc_fence_after();
    if (kTrace) bwd_ready(st);
#if TWFA_BWD_PROF
    g_prof_ready = clock64();
#endif
    const uint32_t ad = sd_lo(c.k, 16), bd = sd_lo(c.q + qs * kTile, 16);
    if (lead<kSolo>()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * kHalf + (kk & 3) * 32) / 16;
        mma_ss(kColS, sdesc_join(ad + off, kSdHi), sdesc_join(bd + off, kSdHi), kIdescKK, kk > 0);
      }
      mma_commit(&bar.s_full);
      if (release) mma_commit(&bar.q_empty[qs]);
    }
    wsync<kSolo>();
  } else if (kind == TWFA_OP_DP) {
    if (it == 0) mbar_wait(&bar.kv_full, t.icount & 1);
    const bool o_need = !(TWFA_BWD_MEMO && st.o_seen == g + 1);
    if (g > 0 && o_need)  // dQ_(g-1) (over dP^T) has been read out
      mbar_wait_all(&bar.o_full[os], (g / vd) & 1, &bar.q_free, (g - 1) & 1);
    else if (g > 0)
      mbar_wait(&bar.q_free, (g - 1) & 1);
    else if (o_need)
      mbar_wait(&bar.o_full[os], (g / vd) & 1);
    st.o_seen = g + 1;
    tc_fence_after();
    if (kTrace) bwd_ready(st);
#if TWFA_BWD_PROF
    g_prof_ready = clock64();
#endif
    const uint32_t ad = sd_lo(c.v, 16), bd = sd_lo(c.o + os * kTile, 16);
    if (lead<kSolo>()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * kHalf + (kk & 3) * 32) / 16;
        mma_ss(kColP, sdesc_join(ad + off, kSdHi), sdesc_join(bd + off, kSdHi), kIdescKK, kk > 0);
      }
      mma_commit(&bar.dp_full);
      if (release) mma_commit(&bar.o_empty[os]);
    }
    wsync<kSolo>();
  } else if (kind == TWFA_OP_DV || kind == TWFA_OP_DK) {
    const bool dv = kind == TWFA_OP_DV;
    // the accumulator is overwritten at iteration 0: the previous work
    // item's dK / dV must have been read out
    if (it == 0 && t.icount > 0) mbar_wait(&bar.acc_free, (t.icount - 1) & 1);
    if (!TWFA_BWD_MEMO) {
      if (dv)
        mbar_wait_all(&bar.p_full, g & 1, &bar.o_full[os], (g / vd) & 1);
      else
        mbar_wait_all(&bar.ds_full, g & 1, &bar.q_full[qs], (g / kd) & 1);
    } else if (dv) {
      if (st.p_seen != g + 1) mbar_wait(&bar.p_full, g & 1);
      if (st.o_seen != g + 1) mbar_wait(&bar.o_full[os], (g / vd) & 1);
      st.p_seen = st.o_seen = g + 1;
    } else {
      if (st.ds_seen != g + 1) bwd_wait_ds(st, plan, g);
      if (st.q_seen != g + 1) mbar_wait(&bar.q_full[qs], (g / kd) & 1);
      st.q_seen = g + 1;
    }
    tc_fence_after();
    if (kTrace) bwd_ready(st);
#if TWFA_BWD_PROF
    g_prof_ready = clock64();
#endif
    // B = dO_i / Q_i as [K = query][N = d], MN-major
    const uint32_t bd = dv ? sd_lo(c.o + os * kTile, kHalf) : sd_lo(c.q + qs * kTile, kHalf);
    const uint32_t a_t = dv ? kColS : kColP, d_t = dv ? kColDV : kColDK;
    if (lead<kSolo>()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)  // 16 queries per K-step: 8 packed bf16 columns of P^T / dS^T
        mma_ts(d_t, a_t + kk * 8, sdesc_join(bd + kk * 2048 / 16, kSdHi), kIdescKM, (it > 0 || kk > 0) ? 1u : 0u);
      if (release) mma_commit(dv ? &bar.o_empty[os] : &bar.q_empty[qs]);
    }
    wsync<kSolo>();
  } else if (kind == TWFA_OP_DQ) {
    if (!(TWFA_BWD_MEMO && st.ds_seen == g + 1)) bwd_wait_ds(st, plan, g);
    tc_fence_after();
    if (kTrace) bwd_ready(st);
#if TWFA_BWD_PROF
    g_prof_ready = clock64();
#endif
    // A = dS as [M = query][K = key], MN-major (row = key in smem);
    // B = K as [K = key][N = d], MN-major
    const uint32_t ad = sd_lo(c.ds, kHalf), bd = sd_lo(c.k, kHalf);
    if (lead<kSolo>()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(kColP, sdesc_join(ad + kk * 2048 / 16, kSdHi), sdesc_join(bd + kk * 2048 / 16, kSdHi), kIdescMM,
               kk > 0);
      mma_commit(&bar.dq_full);
      if (!(kKind >= 0 && TWFA_BWD_CFLAGS) && (op.flags & TWFA_OPF_RELEASE))
        mma_commit(&bar.ds_free);  // dQ staged in the Q slot: dS is free
    }
    wsync<kSolo>();
  }
}

template <int kRole, bool kSpec, bool kTrace>
__device__ __forceinline__ void bwd_run(const BwdCtx& c, const TwfaDevicePlan& plan, const FaBwdArgs& a) {
  BwdBarriers& bar = g_bb;
  // TWFA_BWD_LOAD_WARP >= 0: that warp runs the load warp's streamed loads
  // (and the K / V item loads), the load warp keeps only its other ops
  const bool loads_only = TWFA_BWD_LOAD_WARP >= 0 && c.warp == static_cast<uint32_t>(TWFA_BWD_LOAD_WARP);
  const bool skip_loads = TWFA_BWD_LOAD_WARP >= 0 && c.warp == static_cast<uint32_t>(plan.load_warp);
  const int src = loads_only ? plan.load_warp : static_cast<int>(c.warp);
  const int plen = plan.prog_len[src];
  const bool is_load = TWFA_BWD_LOAD_WARP >= 0 ? loads_only : c.warp == static_cast<uint32_t>(plan.load_warp);
  const bool is_mma = c.warp == static_cast<uint32_t>(plan.mma_warp);
  // TWFA_BWD_FIXED: the TMA / MMA warp whose program is the production order
  // runs it unrolled with every op's kind known at compile time
  constexpr int kFixed[7] = {TWFA_OP_ST, TWFA_OP_LDQ, TWFA_OP_LDO, TWFA_OP_DP, TWFA_OP_DK, TWFA_OP_DQ, TWFA_OP_DV};
  bool fixed = false;
  TwfaPlanOp fx[7];
  if constexpr (kSpec && TWFA_BWD_HEAVY_SPEC && (kRole == kExbDs || kRole == kReduce)) {
    // the production warpgroup programs [EXB DS] and [RD] (host-checked)
    fixed = true;
    fx[0] = plan.ops[plan.prog[src][0]];
    if (kRole == kExbDs) fx[1] = plan.ops[plan.prog[src][1]];
  }
  if constexpr (kRole == kLight) {
    fixed = kSpec && plen == 7 && is_load && is_mma && !loads_only && !skip_loads && plan.k_depth == 2 &&
            plan.v_depth == 2;
    for (int j = 0; j < 7 && fixed; ++j) {
      fx[j] = plan.ops[plan.prog[src][j]];
      fixed = fx[j].kind == kFixed[j];
    }
  }
  BwdState st{0, 0, -1, -1, 0, nullptr, 0, 0, 0, 0};
  uint32_t gbase = 0, icount = 0;
  for (int i = 0;; ++i, ++icount) {
    int work;
    if (a.work_list != nullptr) {
      const int o = a.work_off[blockIdx.x] + i;
      if (o >= a.work_off[blockIdx.x + 1]) break;
      work = a.work_list[o];
    } else {
      work = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
      if (work >= c.num_work) break;
    }
    const BwdItem t = bwd_item(c, a, work, gbase, icount);
    if constexpr (is_light(kRole)) {
      if (is_load) {  // K and V of the work item
        mbar_wait(&bar.kv_empty, (icount & 1) ^ 1);
        if (lead<kRole == kLightSolo>()) {
          mbar_arrive_expect_tx(&bar.kv_full, 2 * kTile);
          tma_load_3d(c.k, &a.tm_k, &bar.kv_full, 0, t.kv0, t.bh, c.pol);
          tma_load_3d(c.k + kHalf, &a.tm_k, &bar.kv_full, 64, t.kv0, t.bh, c.pol);
          tma_load_3d(c.v, &a.tm_v, &bar.kv_full, 0, t.kv0, t.bh, c.pol);
          tma_load_3d(c.v + kHalf, &a.tm_v, &bar.kv_full, 64, t.kv0, t.bh, c.pol);
        }
        wsync<kRole == kLightSolo>();
      }
    }
    st.q_next = st.o_next = 0;
    st.q_target = st.o_target = -1;
    const int trips = t.N + ((kSpec && TWFA_BWD_CFLAGS) ? 0 : plan.max_stage);
    if (kSpec && TWFA_BWD_HEAVY_SPEC && kRole == kExbDs) {
      for (int rr = -1; rr < trips; ++rr) {
        bwd_exec<kRole, TWFA_OP_EXB, kTrace>(fx[0], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_DS, kTrace>(fx[1], rr, c, t, st, plan, a);
      }
    } else if (kSpec && TWFA_BWD_HEAVY_SPEC && kRole == kReduce) {
      for (int rr = -1; rr < trips; ++rr) bwd_exec<kRole, TWFA_OP_RD, kTrace>(fx[0], rr, c, t, st, plan, a);
    } else if (fixed) {
      // the production TMA / MMA program [ST LDQ LDO DP DK DQ DV], each op
      // compiled for its own kind (TWFA_BWD_FIXED)
      for (int rr = -1; rr < trips; ++rr) {
        bwd_exec<kRole, TWFA_OP_ST, kTrace>(fx[0], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_LDQ, kTrace>(fx[1], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_LDO, kTrace>(fx[2], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_DP, kTrace>(fx[3], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_DK, kTrace>(fx[4], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_DQ, kTrace>(fx[5], rr, c, t, st, plan, a);
        bwd_exec<kRole, TWFA_OP_DV, kTrace>(fx[6], rr, c, t, st, plan, a);
      }
    } else if (kSpec && kRole == kLight && is_mma) {
      __trap();  // the host launches the specialized kernel only for the fixed program
    } else
    for (int rr = -1; rr < trips; ++rr)
      for (int j = 0; j < plen; ++j) {
        const TwfaPlanOp& op = plan.ops[plan.prog[src][j]];
        const bool ld = op.kind == TWFA_OP_LDQ || op.kind == TWFA_OP_LDO;
        if ((loads_only && !ld) || (skip_loads && ld)) continue;
        bwd_exec<kRole, -1, kTrace>(op, rr, c, t, st, plan, a);
      }
    if constexpr (is_light(kRole)) {
      if (is_mma) {  // every MMA of the item issued: dK, dV final; K, V free
        if (lead<kRole == kLightSolo>()) {
          mma_commit(&bar.acc_full);
          mma_commit(&bar.kv_empty);
        }
        wsync<kRole == kLightSolo>();
      }
    } else if constexpr (kRole == kReduce || kRole == kReduceFull) {
      kv_epilogue(c, a, t);
    }
    gbase += static_cast<uint32_t>(t.N);
  }
}

// kSpec: the production TMA / MMA program [ST LDQ LDO DP DK DQ DV] compiled
// for its op kinds (TWFA_BWD_FIXED), and no generic op loop in that role --
// the generic loop's code alone costs the role 5 % (810 vs 775 TF/s, C3
// shape). The host picks the instantiation (bwd_fixed_program).
template <bool kSpec, bool kTrace>
__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_bwd_kernel(const __grid_constant__ TwfaDevicePlan plan, const __grid_constant__ FaBwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  BwdCtx c;
  c.k = smem;
  c.v = c.k + kTile;
  c.q = c.v + kTile;
  c.o = c.q + plan.k_depth * kTile;
  c.ds = c.o + plan.v_depth * kTile;
  c.warp = warp_id();
  c.lane = lane_id();
  c.quad = c.warp & 3u;
  c.lane_off = (c.quad * 32u) << 16;
  c.S = a.S;
  c.BH = a.B * a.H;
  c.nq = (a.S + kT - 1) / kT;
  c.num_work = c.BH * c.nq;
  BwdBarriers& bar = g_bb;
  if (threadIdx.x == 0) {
#if TWFA_BWD_PROF
    g_prof_n = 0;
#endif
    mbar_init(&bar.kv_full, 1);
    mbar_init(&bar.kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar.q_full[s], 1);
      mbar_init(&bar.q_empty[s], 1);
      mbar_init(&bar.o_full[s], 1);
      mbar_init(&bar.o_empty[s], 1);
    }
    mbar_init(&bar.s_full, 1);
    mbar_init(&bar.dp_full, 1);
    mbar_init(&bar.dq_full, 1);
    mbar_init(&bar.p_full, 4);
    mbar_init(&bar.ds_full, 4);
    mbar_init(&bar.p_read, 4);
    mbar_init(&bar.q_free, 4);
    mbar_init(&bar.ds_free, 1);
    mbar_init(&bar.acc_full, 1);
    mbar_init(&bar.acc_free, 4);
    fence_mbar_init();
  }
  if (c.warp == static_cast<uint32_t>(plan.load_warp) && c.lane == 0) {
    tma_prefetch_desc(&a.tm_q);
    tma_prefetch_desc(&a.tm_k);
    tma_prefetch_desc(&a.tm_v);
    tma_prefetch_desc(&a.tm_do);
  }
  if (c.warp == 0) tmem_alloc<512>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (bar.tmem_base != 0) __trap();  // one CTA per SM owns all 512 columns from 0
  c.pol = policy_evict_last();
  const int wg = static_cast<int>(c.warp >> 2);
  const bool exb = wg * 4 == plan.sm_warp[0], ds = wg * 4 == plan.sm_warp[1], rd = wg * 4 == plan.cr_warp[0];
  // registers: EXB carries the 128-float S^T / P^T row, DS the packed P^T
  // (64) and a dP^T chunk, RD half a dQ row; the TMA / MMA warps need few
  if (exb && ds) {
    setmaxnreg_inc<200>();
    bwd_run<kExbDs, kSpec, kTrace>(c, plan, a);
  } else if (exb) {
    setmaxnreg_inc<168>();
    bwd_run<kExb, kSpec, kTrace>(c, plan, a);
  } else if (ds) {
    setmaxnreg_inc<144>();
    bwd_run<kDs, kSpec, kTrace>(c, plan, a);
  } else if (rd) {
    // with EXB and DS fused on one warpgroup the register file has room for
    // the whole dQ row in RD (200 + 176 + 8 x 64 per thread-warp class)
    if (TWFA_BWD_RD_FULL && plan.sm_warp[0] == plan.sm_warp[1]) {
      setmaxnreg_inc<176>();
      bwd_run<kReduceFull, kSpec, kTrace>(c, plan, a);
    } else {
      setmaxnreg_dec<128>();
      bwd_run<kReduce, kSpec, kTrace>(c, plan, a);
    }
  } else {
    setmaxnreg_dec<64>();
    if (TWFA_BWD_SOLO) {
      if (elect_one()) bwd_run<kLightSolo, false, kTrace>(c, plan, a);
      __syncwarp();
    } else {
      bwd_run<kLight, kSpec, kTrace>(c, plan, a);
    }
  }
  if (c.lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
#if TWFA_BWD_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < g_prof_n && i < 24; ++i)
      printf("PROF %lld %lld %lld %lld\n", g_prof[i][0], g_prof[i][1], g_prof[i][2], g_prof[i][3]);
#endif
  if (c.warp == 0) {
    tc_fence_after();
#if TWFA_BWD_PROF
    g_prof_ready = clock64();
#endif
    tmem_dealloc<512>(0);
  }
}

// D = rowsum(dO * O) in fp32: 16 threads per row, 8 bf16 each
__global__ void fa_bwd_pre(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                           float* __restrict__ dvec, int64_t rows) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 16) + threadIdx.x / 16;
  const int part = threadIdx.x % 16;
  float acc = 0.f;
  if (row < rows) {
    const uint4 x = reinterpret_cast<const uint4*>(o + row * 128)[part];
    const uint4 y = reinterpret_cast<const uint4*>(dout + row * 128)[part];
    const __nv_bfloat162* xa = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* ya = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __bfloat1622float2(xa[i]), b = __bfloat1622float2(ya[i]);
      acc = fmaf(a.x, b.x, fmaf(a.y, b.y, acc));
    }
  }
#pragma unroll
  for (int m = 8; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (row < rows && part == 0) dvec[row] = acc;
}

// dQ = scale * accumulator -> bf16, 8 per thread
__global__ void fa_bwd_post(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq, float scale, int64_t n8) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const float4 a = reinterpret_cast<const float4*>(acc)[2 * i];
  const float4 b = reinterpret_cast<const float4*>(acc)[2 * i + 1];
  uint4 w;
  w.x = pack_bf16(a.x * scale, a.y * scale);
  w.y = pack_bf16(a.z * scale, a.w * scale);
  w.z = pack_bf16(b.x * scale, b.y * scale);
  w.w = pack_bf16(b.z * scale, b.w * scale);
  reinterpret_cast<uint4*>(dq)[i] = w;
}

}  // namespace

size_t fa_bwd_smem_bytes(const TwfaDevicePlan& plan) {
  return static_cast<size_t>(3 + plan.k_depth + plan.v_depth) * kTile + 1024;
}

size_t fa_bwd_workspace_bytes(int B, int H, int S) {
  const size_t rows = static_cast<size_t>(B) * H * S;
  return rows * 128 * sizeof(float) + rows * sizeof(float);
}

// host mirror of the device-side condition of the fixed program: the TMA /
// MMA warp (one warp) holds exactly [ST LDQ LDO DP DK DQ DV], Q and dO rings
// two deep, the default one-warp roles
bool bwd_fixed_program(const TwfaDevicePlan& plan) {
  if (plan.num_tiles != 1 || plan.k_depth != 2 || plan.v_depth != 2 || plan.mma_warp != plan.load_warp ||
      TWFA_BWD_SOLO || TWFA_BWD_LOAD_WARP >= 0)
    return false;
  if (TWFA_BWD_CFLAGS && (plan.max_stage != 0 || plan.k_prefetch != 1 || plan.v_prefetch != 1 || plan.s_split != 0))
    return false;
  if (TWFA_BWD_CFLAGS)
    for (int v = 0; v < plan.num_nodes; ++v)
      if (plan.ops[v].stage != 0) return false;
  if (TWFA_BWD_HEAVY_SPEC) {  // the fused [EXB DS] warpgroup and the [RD] warpgroup
    const int e = plan.sm_warp[0], r = plan.cr_warp[0];
    if (e != plan.sm_warp[1] || e < 0 || r < 0 || plan.prog_len[e] != 2 || plan.prog_len[r] != 1 ||
        plan.ops[plan.prog[e][0]].kind != TWFA_OP_EXB || plan.ops[plan.prog[e][1]].kind != TWFA_OP_DS ||
        plan.ops[plan.prog[r][0]].kind != TWFA_OP_RD)
      return false;
  }
  const int w = plan.mma_warp;
  static const int kinds[7] = {TWFA_OP_ST, TWFA_OP_LDQ, TWFA_OP_LDO, TWFA_OP_DP, TWFA_OP_DK, TWFA_OP_DQ, TWFA_OP_DV};
  if (w < 0 || w >= TWFA_MAX_WARPS || plan.prog_len[w] != 7) return false;
  for (int j = 0; j < 7; ++j) {
    const TwfaPlanOp& op = plan.ops[plan.prog[w][j]];
    if (op.kind != kinds[j]) return false;
    if (TWFA_BWD_CFLAGS) {  // the flags the specialized kernel assumes
      const bool rel = op.kind == TWFA_OP_DK || op.kind == TWFA_OP_DV;
      if (((op.flags & TWFA_OPF_RELEASE) != 0) != rel || (op.flags & TWFA_OPF_WAIT_PREAD)) return false;
    }
  }
  return true;
}

cudaError_t fa_bwd_launch(const TwfaDevicePlan& plan, const FaBwdArgs& args, const __nv_bfloat16* o,
                          const __nv_bfloat16* dout, __nv_bfloat16* dq, int grid, cudaStream_t stream) {
  const int64_t rows = static_cast<int64_t>(args.B) * args.H * args.S;
  fa_bwd_pre<<<static_cast<unsigned>((rows + 15) / 16), 256, 0, stream>>>(o, dout, args.dvec, rows);
  cudaError_t e = cudaMemsetAsync(args.dq_acc, 0, static_cast<size_t>(rows) * 128 * sizeof(float), stream);
  if (e != cudaSuccess) return e;
  if (plan.num_tiles == 2) {
    e = fa_bwd_pp_main_launch(plan, args, grid, stream);
  } else {
    const size_t smem = fa_bwd_smem_bytes(plan);
    const bool spec = TWFA_BWD_FIXED && bwd_fixed_program(plan);
    // traced launches run the instantiation with the issue-trace code; the
    // others have it compiled out (+3 %, C3 shape)
    const bool tr = args.trace != nullptr;
    const void* kern = spec ? (tr ? reinterpret_cast<const void*>(&fa_bwd_kernel<true, true>)
                                  : reinterpret_cast<const void*>(&fa_bwd_kernel<true, false>))
                            : (tr ? reinterpret_cast<const void*>(&fa_bwd_kernel<false, true>)
                                  : reinterpret_cast<const void*>(&fa_bwd_kernel<false, false>));
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (spec && tr)
      fa_bwd_kernel<true, true><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
    else if (spec)
      fa_bwd_kernel<true, false><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
    else if (tr)
      fa_bwd_kernel<false, true><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
    else
      fa_bwd_kernel<false, false><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  const int64_t n8 = rows * 16;
  fa_bwd_post<<<static_cast<unsigned>((n8 + 255) / 256), 256, 0, stream>>>(args.dq_acc, dq, args.scale, n8);
  return cudaGetLastError();
}

}  // namespace twfa
