// FA-forward on sm_100a, realized from a Twill joint schedule (kernel bodies).
//
// Loop body (reference: proj/tests/testutil.hpp:13-15, PAPER.md:185-191,
// Blackwell strategy PAPER.md:1015-1046), per 128-key K/V tile and per
// 128-row Q sub-tile k of the CTA's 256-row query block:
//   LDK, LDV  TMA loads into smem rings (depth = streaming_depths)
//   S_k       S_k = Q_k K^T           tcgen05.mma SS -> TMEM cols [128k, 128k+128)
//   MX_k      m_new = max(m, rowmax(S_k) * scale*log2e); alpha = exp2(m - m_new)
//   EX_k      P_k = exp2(S_k*scale*log2e - m_new) -> bf16 over S_k in TMEM; l = l*alpha + rowsum
//   CR_k      O_k *= alpha            tcgen05.ld / st on TMEM cols [256+128k, ...)
//   PV_k      O_k += P_k V            tcgen05.mma TS (A = P from TMEM)
//
// Which warp runs which op, in which order and in which pipeline stage is
// NOT hard-coded: every warp walks its trip program from the TwfaDevicePlan
// (lowering.cpp), i.e. the solver's A(v) and M(v). Trip r runs op v on
// iteration r - stage(v); trips before max_stage are the prologue and trips
// past the last iteration the epilogue, exactly the region split of the
// reference's program synthesis (codegen.cpp:43-189). Every edge of the loop
// graph that the schedule places across warps is an mbarrier (the
// reference's `spill_recv` / xfer sites); same-warp edges that go through the
// asynchronous tensor core still wait on the MMA commit barrier, except
// PV_k -> S_k when one thread issues both (tcgen05 ops of a thread execute in
// order).
//
// Two kernels realize a plan, sharing every op body (exec_op):
//  * fa_fwd_spec<P>: one instantiation per schedule generated at build time
//    from the committed solution JSON (twfa-gen, gen/fa_plans.inc). Each
//    warp's trip program is a compile-time sequence, so op dispatch, ring
//    arithmetic and flags fold away.
//  * fa_fwd_interp: walks the trip programs at run time (any other plan).
//
// Register classes: warpgroups that run softmax ops (MX/EX) raise their
// register budget with setmaxnreg and keep a 128-column S row resident; the
// other warpgroups (TMA, MMA issue, correction) lower theirs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "fa_fwd.h"
#include <gen/fa_plans.inc>
#include "sm100.cuh"

// Kernel bodies of the FA-forward executor. Included by fa_fwd_sm100.cu (the
// interpreter and the launch dispatch) and by one generated translation unit
// per specialized schedule (gen/fa_spec_<id>.cu), compiled in parallel.
#pragma once

namespace twfa {

namespace {

constexpr int kBlockQ = 128;  // rows per Q sub-tile (= TMEM lanes)
constexpr int kHeadDim = 128;
constexpr uint32_t kTileBytes = kBlockQ * kHeadDim * 2;  // Q tile: 32 KiB, two 16 KiB SW128 column halves
constexpr uint32_t kHalfBytes = kTileBytes / 2;

// K/V tile of KV keys (128, or 64 when S is double-buffered in tensor memory:
// the plan's S ring depth is 128 / KV). S_k's buffer b of iteration g is
// g % depth at columns [128k + b*KV, ...); P_k (bf16) is aliased over it.
//
// CTA pair (P = true, cta_group::2): the two CTAs of a cluster run one work
// tile of 2 x 256 query rows; sub-tile k of CTA r holds rows 256k + 128r of
// it, and one M = 256 MMA computes S_k (PV_k) for both. Each CTA stages half
// of every K tile (keys 64r .. 64r + 63, both head-dim halves) and half of
// every V tile (head dims 64r .. 64r + 63, all keys), so the per-SM K/V ring
// slots, the TMA traffic and the tensor core's shared-memory reads per FLOP
// are halved.
template <int KV, bool P = false>
struct Kv {
  static constexpr int depth = 128 / KV;                        // S ring depth
  static constexpr uint32_t tile = KV * kHeadDim * 2;           // full K or V tile bytes
  static constexpr uint32_t half = tile / 2;                    // one 64-column SW128 half
  static constexpr uint32_t slot = P ? tile / 2 : tile;         // this CTA's ring slot (K or V)
  static constexpr uint32_t k_half = P ? half / 2 : half;       // K slot: one head-dim half of its keys
  static constexpr int rows = P ? 2 : 1;                        // CTAs per work tile
  static constexpr uint32_t idesc_s = idesc_bf16_f32(128 * rows, KV, 0);  // K-major Q, K-major K
  static constexpr uint32_t idesc_pv = idesc_bf16_f32(128 * rows, kHeadDim, 1);  // TMEM P, MN-major V
};
constexpr int kMaxRing = 4;
#ifndef TWFA_POLY_EVERY
#define TWFA_POLY_EVERY 1000  // measured: MUFU-only is fastest while the loop is latency-bound
#endif
constexpr int kPolyEvery = TWFA_POLY_EVERY;  // 1 in kPolyEvery exp2 pairs on the FMA pipe
// Online-softmax rescale threshold (log2 units): the running max is only
// moved when a row's max grows by more than 2^8, so P <= 256 and most
// iterations need no O correction. The final O / l is unchanged in exact
// arithmetic (m cancels); bf16 P and fp32 l stay far from overflow.
constexpr float kRescaleLog2 = 8.0f;
#ifndef TWFA_TMA_EPILOGUE
#define TWFA_TMA_EPILOGUE 1
#endif
// MX_k(g) hands its rescale factors to CR_k(g) through the double-buffered
// stats slot g % 2. The slot is free again by construction when MX_k(g + 2)
// writes it: CR_k(g) reads it before arriving o_ready, PV_k(g) waits for
// o_ready, S_k(g + 2) follows PV_k(g) (in order on one thread, or behind
// PV_k's commit), and MX_k(g + 2) waits for S_k(g + 2). The explicit
// slot-empty wait is kept (TWFA_ST_EMPTY = 1): dropping it measured 9 %
// slower, the mbarrier round trip paces the two softmax warpgroups' turns
// on MUFU (a MUFU token that makes them alternate strictly: -2 to -4 %).
#ifndef TWFA_ST_EMPTY
#define TWFA_ST_EMPTY 1
#endif
// What-if knobs for sensitivity experiments (timing only; results are WRONG
// when set): 1 = half the exponentials on MUFU (the rest reuse them),
// 3 = MX reads half the row, 4 = no K/V loads after the first ring fill,
// 5 = the MMA warp skips its steady-state waits on K, V and the correction
// (only P and Q are awaited), 6 = 5 and the loads skip their empty-slot waits
#ifndef TWFA_WHATIF
#define TWFA_WHATIF 0
#endif
// P_k is handed to PV_k in kPParts parts of 128 / kPParts keys: part j is
// released once its tcgen05.st completed (checked after the exponentials of
// part j + 1, so MUFU does not drain), and PV_k issues its K-steps over those
// keys. Finer parts start PV earlier and leave a shorter tail after EX.
#ifndef TWFA_P_PARTS
#define TWFA_P_PARTS 4  // measured: 4 parts >= halves >= 8 parts (C3, C4)
#endif
constexpr int kPParts = TWFA_P_PARTS;
static_assert(kPParts == 2 || kPParts == 4 || kPParts == 8, "P parts");
// CTA pairs hand P over in halves (TWFA_PAIR_P_PARTS; measured under the
// power cap, C3: 0.585 tensor-pipe fraction per clock with halves against
// 0.564 with 4 parts)
#ifndef TWFA_PAIR_P_PARTS
#define TWFA_PAIR_P_PARTS 2
#endif
static_assert(TWFA_PAIR_P_PARTS <= kPParts || TWFA_PAIR_P_PARTS == 2, "pair P parts");
template <bool P>
__host__ __device__ constexpr int p_parts() {
  return P ? (TWFA_PAIR_P_PARTS < kPParts ? TWFA_PAIR_P_PARTS : kPParts) : kPParts;
}
// MMA-warp input waits: probe all inputs of a PV op at once (1) instead of
// waiting for them one after the other (0); skip a second wait on a K / V
// tile this warp already saw land (TWFA_MEMO_WAITS)
#ifndef TWFA_PROBE_PARTS
#define TWFA_PROBE_PARTS 1
#endif
#ifndef TWFA_MEMO_WAITS
#define TWFA_MEMO_WAITS 1
#endif
#ifndef TWFA_SOFTMAX_TOKEN
#define TWFA_SOFTMAX_TOKEN 0  // measured: serializing MX+EX of the two tiles is 12% slower (C3)
#endif
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, kHeadDim, 1);  // TMEM P, MN-major V
constexpr uint32_t kIdescS64 = idesc_bf16_f32(128, 64, 0);       // split S: one 64-key half
constexpr uint32_t kSdescHi = sdesc_hi(1024);                     // SW128, 8-row groups 1 KiB apart

struct __align__(8) FaBarriers {
  uint64_t q_full[TWFA_MAX_TILES], q_empty[TWFA_MAX_TILES];
  uint64_t k_full[kMaxRing], k_empty[kMaxRing];
  uint64_t v_full[kMaxRing], v_empty[kMaxRing];
  // per S buffer (ring depth <= 2): a phase-parity barrier may only run one
  // phase ahead of its waiters, which the per-buffer split guarantees
  uint64_t s_full[TWFA_MAX_TILES][2];
  uint64_t p_part[TWFA_MAX_TILES][2][kPParts];  // P_k keys [j*128/kPParts, ...) in tensor memory
  uint64_t o_ready[TWFA_MAX_TILES][2], o_done[TWFA_MAX_TILES][2];
  uint64_t st_full[TWFA_MAX_TILES][2], st_empty[TWFA_MAX_TILES][2];
  uint64_t l_full[TWFA_MAX_TILES], l_empty[TWFA_MAX_TILES];
  uint64_t sm_tok[TWFA_MAX_TILES];  // softmax order token (TWFA_SOFTMAX_TOKEN)
  uint64_t s_half[TWFA_MAX_TILES];  // split S: SA_k committed
  uint64_t s_lo[TWFA_MAX_TILES][2];  // TWFA_S_HALVES: keys 0-63 of S_k committed
  uint64_t s_read[TWFA_MAX_TILES];  // split S: MX_k has the S row in registers
  uint32_t tmem_base;
};

struct FaShared {
  float stats[TWFA_MAX_TILES][2][kBlockQ];  // MX -> CR rescale factors, double-buffered
  float mrow[TWFA_MAX_TILES][2][kBlockQ];   // MX -> CR running max (TWFA_CR_EXP; NaN: no offload)
  float lbuf[TWFA_MAX_TILES][2][kBlockQ];   // EX -> epilogue: running max, row sum
  // per-warp trip programs (interpreted roles): one shared load per op
  TwfaPlanOp prog[TWFA_MAX_WARPS][TWFA_MAX_NODES];
  int prog_len[TWFA_MAX_WARPS];
  FaBarriers bar;
};

// Barriers, handoff buffers and trip programs live in static shared memory so
// every access compiles to LDS/STS/SYNCS on a known shared address.
__shared__ FaShared g_sh;

// Issue trace of CTA 0 (debug / schedule-realization evidence). Per warp:
// word 0 = record count, then records of kTraceWords uint32:
// {node, iteration, trip, t_issue, t_ready (inputs waited), t_done, work tile
// ordinal of the CTA, K/V iterations of that tile}. A streamed load that
// runs ahead into the next work tile records that tile and its iteration.
constexpr int kTraceWords = 8;
// Record 0 of warp 0 (unused by the op records, which start at 1) holds CTA
// 0's own clock: words 1 / 2 = clock64 / %globaltimer (ns) after the setup
// barrier, 3 / 4 = the same at teardown (low 32 bits): the SM clock the
// kernel ran at, independent of the other CTAs' finishing times.
__device__ __forceinline__ void trace_clock(const FaArgs& a, int word) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    a.trace[word] = static_cast<uint32_t>(clock64());
    a.trace[word + 1] = static_cast<uint32_t>(global_timer_ns());
  }
}

template <bool kTrace>
__device__ __forceinline__ uint32_t* trace_begin(const FaArgs& a, uint32_t warp, uint32_t& n, int node, int it,
                                                 int trip, uint32_t tile, int tile_n) {
  if (!kTrace || blockIdx.x != 0 || lane_id() != 0) return nullptr;
  uint32_t* base = a.trace + static_cast<size_t>(warp) * a.trace_cap * kTraceWords;
  if (n + 1 >= a.trace_cap) return nullptr;
  uint32_t* e = base + (n + 1) * kTraceWords;
  e[0] = static_cast<uint32_t>(node);
  e[1] = static_cast<uint32_t>(it);
  e[2] = static_cast<uint32_t>(trip);
  e[3] = static_cast<uint32_t>(clock64());
  e[6] = tile;
  e[7] = static_cast<uint32_t>(tile_n);
  base[0] = ++n;  // count kept in a register; the store is fire-and-forget
  return e;
}
template <bool kTrace>
__device__ __forceinline__ void trace_mark(uint32_t* e, int field) {
  if (kTrace && e != nullptr) e[field] = static_cast<uint32_t>(clock64());
}

// ---------------------------------------------------------------- barrier flavours
// With CTA pairs (P) the MMA-side barriers of the leader also receive
// arrivals from the peer CTA, and the tensor core reads and writes both
// CTAs' memory: waits acquire at cluster scope, the softmax / correction
// warps of both CTAs arrive on the leader's copy, commits multicast to both.
template <bool P>
__device__ __forceinline__ void wait_(uint64_t* b, uint32_t ph) {
  if constexpr (P) mbar_wait_cluster(b, ph); else mbar_wait(b, ph);
}
template <bool P>
__device__ __forceinline__ bool test_(uint64_t* b, uint32_t ph) {
  if constexpr (P) return mbar_test_cluster(b, ph); else return mbar_test(b, ph);
}
template <bool P>
__device__ __forceinline__ void wait_all_(uint64_t* b0, uint32_t p0, uint64_t* b1, uint32_t p1) {
  if constexpr (P) {
    bool d0 = mbar_try_wait_cluster(b0, p0);
    bool d1 = mbar_try_wait_cluster(b1, p1);
    while (!d0) d0 = mbar_try_wait_cluster(b0, p0);
    while (!d1) d1 = mbar_try_wait_cluster(b1, p1);
  } else {
    mbar_wait_all(b0, p0, b1, p1);
  }
}
// a warp's arrival on a barrier the MMA-issuing warp (of the leader) waits on
template <bool P>
__device__ __forceinline__ void arrive_mma_(uint64_t* b) {
  if constexpr (P) warp_arrive_cluster(b, 0); else warp_arrive(b);
}
template <bool P>
__device__ __forceinline__ void commit_(uint64_t* b) {
  if constexpr (P) mma_commit_pair(b, 0x3); else mma_commit(b);
}

// ---------------------------------------------------------------- softmax pieces
// all N scores of this thread's TMEM lane, one wait
template <int N>
__device__ __forceinline__ void load_row(uint32_t taddr, uint32_t (&s)[N]) {
#pragma unroll
  for (int c = 0; c < N / 32; ++c) tmem_ld32(taddr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
  tmem_ld_wait();
}

template <int N>
__device__ __forceinline__ void mask_row(uint32_t (&s)[N], int limit) {
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i >= limit) s[i] = __float_as_uint(-INFINITY);
}

// FMNMX3: three-operand max (sm_100), four independent chains
template <int N>
__device__ __forceinline__ float row_max(const uint32_t (&s)[N]) {
  float a[4] = {__uint_as_float(s[0]), __uint_as_float(s[1]), __uint_as_float(s[2]), __uint_as_float(s[3])};
#pragma unroll
  for (int i = 4; i < N - 4; i += 8) {
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = fmax3(a[j], __uint_as_float(s[i + 2 * j]), __uint_as_float(s[i + 2 * j + 1]));
  }
  a[0] = fmax3(a[0], __uint_as_float(s[N - 4]), __uint_as_float(s[N - 3]));
  a[1] = fmax3(a[1], __uint_as_float(s[N - 2]), __uint_as_float(s[N - 1]));
  return fmax3(a[0], a[1], fmaxf(a[2], a[3]));
}

// P = exp2(S*sl - m) for the resident scores: FFMA2 for the argument, MUFU
// ex2 or the FMA-pipe polynomial (1 in kPolyEvery pairs) for the exp, FADD2
// for the row sum, F2FP to bf16 pairs, stored as the TS-MMA A operand over
// the first N/2 columns of the S tile. Part j of P is released to PV_k on
// part_bar[j] (see kPParts). Returns the row sum.
template <int N, bool kMask, bool P>
__device__ __forceinline__ float exp_store_row(const uint32_t (&s)[N], uint32_t taddr, float sl, float m,
                                               uint64_t* part_bar) {
  constexpr int kParts = N == 128 ? p_parts<P>() : 2;  // 64-key tiles keep halves
  constexpr int kPartKeys = N / kParts;
  constexpr int kKeys = kPartKeys < 32 ? kPartKeys : 32;  // keys per tcgen05.st chunk
  constexpr int kRegs = kKeys / 2;
  const float2 sl2 = make_float2(sl, sl);
  const float2 nm2 = make_float2(-m, -m);
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < N / kKeys; ++c) {
    uint32_t pk[kRegs];
#pragma unroll
    for (int i = 0; i < kKeys; i += 2) {
      const int e = c * kKeys + i;
      const float2 x = ffma2(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2, nm2);
      float2 p;
      if (TWFA_WHATIF == 1 && e >= N / 2) {
        p = x;
      } else if (!kMask && ((e >> 1) % kPolyEvery) == kPolyEvery - 1) {
        // masked tiles (diagonal / sequence tail) hold -inf: MUFU maps it to 0
        p = poly_exp2x2(x);
      } else {
        p.x = fast_exp2(x.x);
        p.y = fast_exp2(x.y);
      }
      acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], p);
      pk[i >> 1] = pack_bf16(p.x, p.y);
    }
    if (c > 0 && (c * kKeys) % kPartKeys == 0) {
      // the part that ended with chunk c - 1 was stored one chunk of MUFU
      // work ago: release it
      tmem_st_wait();
      tc_fence_before();
      arrive_mma_<P>(&part_bar[c * kKeys / kPartKeys - 1]);
    }
    tmem_st<kRegs>(taddr + c * kRegs, pk);
  }
  tmem_st_wait();
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

// Fused MX_k + EX_k that starts the exponentials before the row max is
// known. With the rescale threshold the running max rarely moves after the
// first tiles, so chunk 0 of the S row is loaded first and exponentiated with
// m_old while the rest of the row is still in flight from tensor memory.
// Once the whole row is in registers its max decides, per row, whether m
// moves; if any row of the warp moved, chunk 0 is recomputed with the new max
// before anything is stored. The stored P and the row sum are therefore
// exactly those of MX_k followed by EX_k; only the TMEM read of the row and
// the max leave the S -> P critical path. `handoff(alpha)` passes the rescale
// factor to the correction warpgroup once the max is known.
#ifndef TWFA_SPEC_EX
#define TWFA_SPEC_EX 1
#endif
// S_k issued as two N = 64 halves with a commit after the first (the
// speculative EX starts on keys 0-63 while keys 64-127 are computed)
#ifndef TWFA_S_HALVES
#define TWFA_S_HALVES 0  // measured: -5 % C3 (twice the MMA issues for S outweigh the earlier start)
#endif
// TWFA_TRACE_SUB (diagnostic builds): the traced MX record's fields 6 / 7
// hold the clock after the row max / handoff and after the last exponential
// instead of the work tile
#ifndef TWFA_TRACE_SUB
#define TWFA_TRACE_SUB 0
#endif
// TWFA_LATE_SUM: the row sum of chunks 1.. is taken after the last P part is
// released (the fp32 P overwrites the consumed S registers), so the FADD2s
// leave the MUFU-bound path to PV
// The correction warps compute the last 32-key chunk of every row's P in
// the speculative iterations (TWFA_CR_EXP): exp2 by the FMA-pipe polynomial
// on warps that are otherwise idle with the rescale threshold, a quarter of
// the exponentials off the softmax warps' MUFU path. The last P part then
// waits for the softmax and the correction warps; the correction warps keep
// their part of the row sum and add it in the epilogue.
#ifndef TWFA_CR_WAIT_ALL
#define TWFA_CR_WAIT_ALL 0  // 1: synccheck-clean (every o_done phase awaited), measured -0.5 to -1 %
#endif
#ifndef TWFA_CR_EXP
#define TWFA_CR_EXP 0  // measured: -3.4 % per clock (pair, C3), -3 % (C4), -1 % (one CTA)
#endif
template <int KV>
constexpr bool kCrExp = TWFA_CR_EXP && KV == 128;
#ifndef TWFA_CHUNK_PHASED
#define TWFA_CHUNK_PHASED 0  // measured: all FFMA2 arguments of a chunk before its MUFU ops, -0.6 % (C3, C4)
#endif
#ifndef TWFA_LATE_SUM
#define TWFA_LATE_SUM 1  // measured: +0.9 % (pair) / +1.4 % (one CTA) per clock under the power cap, +4 % burst
#endif
static_assert(!TWFA_CR_EXP || TWFA_LATE_SUM, "TWFA_CR_EXP releases the last P part with the late row sum");
template <int N, bool P, bool kOff, class Handoff, class WaitRest>
__device__ __forceinline__ float mx_ex_spec(uint32_t (&s)[N], uint32_t taddr, float sl, float& m_io, float& alpha,
                                            uint64_t* part_bar, Handoff&& handoff, WaitRest&& wait_rest,
                                            uint32_t* trm = nullptr) {
  constexpr int kParts = p_parts<P>();
  constexpr int kPartKeys = N / kParts;
  constexpr int kKeys = kPartKeys < 32 ? kPartKeys : 32;
  constexpr int kRegs = kKeys / 2;
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
  tmem_ld_wait();
  // with S in halves, keys 64.. may still be in flight in the tensor core:
  // load the rest of the first half, then wait for the second
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
  wait_rest();
#pragma unroll
  for (int c = 2; c < N / 32; ++c) tmem_ld32(taddr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
  const float m_old = m_io;
  const float2 sl2 = make_float2(sl, sl);
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t pk0[kRegs];
  auto chunk = [&](int c, float m, uint32_t (&pk)[kRegs]) {
    const float2 nm2 = make_float2(-m, -m);
    if (TWFA_CHUNK_PHASED) {  // all exponent arguments first, so every MUFU input is ready when it issues
#pragma unroll
      for (int i = 0; i < kKeys; i += 2) {
        const int e = c * kKeys + i;
        const float2 x = ffma2(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2, nm2);
        s[e] = __float_as_uint(x.x);
        s[e + 1] = __float_as_uint(x.y);
      }
    }
#pragma unroll
    for (int i = 0; i < kKeys; i += 2) {
      const int e = c * kKeys + i;
      const float2 x = TWFA_CHUNK_PHASED
                           ? make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1]))
                           : ffma2(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2, nm2);
      float2 p;
      if (TWFA_WHATIF == 1 && e >= N / 2) {
        p = x;
      } else if (((e >> 1) % kPolyEvery) == kPolyEvery - 1) {  // unmasked rows only: x is finite
        p = poly_exp2x2(x);
      } else {
        p.x = fast_exp2(x.x);
        p.y = fast_exp2(x.y);
      }
      if (TWFA_LATE_SUM && c > 0) {  // S of chunk c is consumed: keep P there for the late row sum
        s[e] = __float_as_uint(p.x);
        s[e + 1] = __float_as_uint(p.y);
      } else {
        acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], p);
      }
      pk[i >> 1] = pack_bf16(p.x, p.y);
    }
  };
  chunk(0, m_old, pk0);
  tmem_ld_wait();
  const float mx = row_max<N>(s);
  const float m_cand = fmaxf(m_old, mx * sl);
  const float m_new = (m_cand - m_old > kRescaleLog2) ? m_cand : m_old;
  if (__any_sync(0xffffffffu, m_new != m_old)) {
    acc[0] = acc[1] = make_float2(0.f, 0.f);
    chunk(0, m_new, pk0);
  }
  alpha = m_new == m_old ? 1.f : fast_exp2(m_old - m_new);
  m_io = m_new;
  handoff(alpha);
  if (TWFA_TRACE_SUB && trm != nullptr) trm[6] = static_cast<uint32_t>(clock64());
  tmem_st<kRegs>(taddr, pk0);
  // kOff: the last chunk is the correction warps' (TWFA_CR_EXP)
  constexpr int kChunks = N / kKeys - (kOff ? 1 : 0);
#pragma unroll
  for (int c = 1; c < kChunks; ++c) {
    uint32_t pk[kRegs];
    chunk(c, m_new, pk);
    if ((c * kKeys) % kPartKeys == 0) {
      tmem_st_wait();
      tc_fence_before();
      arrive_mma_<P>(&part_bar[c * kKeys / kPartKeys - 1]);
    }
    tmem_st<kRegs>(taddr + c * kRegs, pk);
  }
  if (TWFA_TRACE_SUB && trm != nullptr) trm[7] = static_cast<uint32_t>(clock64());
  tmem_st_wait();
  if constexpr (TWFA_LATE_SUM) {
    tc_fence_before();
    // the parts from the one holding this warp's last chunk to the last,
    // before the row sum
#pragma unroll
    for (int j = (kChunks * kKeys - 1) / kPartKeys; j < kParts; ++j) arrive_mma_<P>(&part_bar[j]);
#pragma unroll
    for (int e = kKeys; e < kChunks * kKeys; e += 4) {
      acc[0] = fadd2(acc[0], make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])));
      acc[1] = fadd2(acc[1], make_float2(__uint_as_float(s[e + 2]), __uint_as_float(s[e + 3])));
    }
  }
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

// ---------------------------------------------------------------- state
struct FaCtx {
  uint8_t* q_smem;
  uint8_t* k_smem;
  uint8_t* v_smem;
  uint8_t* o_smem;  // 16 KiB epilogue staging (one 128 x 64 bf16 half-tile, SW128)
  uint32_t tmem;
  uint32_t warp, lane, quad, lane_off;
  uint32_t rank;  // CTA rank in the pair (0 = leader, issues the MMAs); 0 without pairs
  int unit, units;  // this CTA's work unit (CTA or CTA pair) and their number
  int S, BH, q_blocks, num_work;
  int q_warp;  // idle warp loading the Q tiles (-1: the load warp does)
  float scale_log2;
  uint64_t pol_q, pol_kv;
};

// the work tile (256 query rows of one (b, h)) a CTA is on
struct WorkTile {
  int bh, q0, N;    // N = K/V iterations of this tile
  uint32_t gbase;   // global iteration index of its iteration 0 (ring phases)
  uint32_t tcount;  // work tiles done by this CTA (Q / LSE buffer phases)
};

template <int KV, bool P>
__device__ __forceinline__ WorkTile work_tile(const FaCtx& c, const FaArgs& args, int work, uint32_t gbase,
                                              uint32_t tcount) {
  constexpr int kRows = 2 * kBlockQ * Kv<KV, P>::rows;  // query rows of a work tile
  WorkTile t;
  int qb;
  if (args.causal) {  // longest-processing-time first
    qb = c.q_blocks - 1 - work / c.BH;
    t.bh = work % c.BH;
  } else {
    t.bh = work / c.q_blocks;
    qb = work % c.q_blocks;
  }
  t.q0 = qb * kRows;
  const int kv_end = args.causal ? min(c.S, t.q0 + kRows) : c.S;
  t.N = (kv_end + KV - 1) / KV;
  t.gbase = gbase;
  t.tcount = tcount;
  return t;
}

// First query row of this CTA's sub-tile k of a work tile
template <int KV, bool P>
__device__ __forceinline__ int sub_tile_row(const FaCtx& c, const WorkTile& t, int k) {
  return t.q0 + k * kBlockQ * Kv<KV, P>::rows + static_cast<int>(c.rank) * kBlockQ;
}

// Number of leading keys of this K/V tile that row `row` may attend to
// (the rest are past the sequence end or above the causal diagonal).
template <int KV>
__device__ __forceinline__ int valid_keys(const FaArgs& a, int row, int key0) {
  const int end = a.causal ? min(a.S, row + 1) : a.S;
  return max(0, min(KV, end - key0));
}

// running per-warp state
struct WarpState {
  float m_run[TWFA_MAX_TILES], l_run[TWFA_MAX_TILES], alpha[TWFA_MAX_TILES];
  float l3[TWFA_MAX_TILES];  // correction warps: row-sum share of the offloaded chunk (TWFA_CR_EXP)
  int k_next, v_next;  // next K / V iteration to load (TMA warp); may run into the next tile
  // MMA warp: the last global iteration whose K (V) tile this warp already
  // saw land; a second tensor-core op on the same tile skips the wait
  uint32_t k_seen, v_seen;
  uint32_t trace_n;
  // TMA warp: the CTA's next work tile (its first K / V iterations are
  // prefetched while this tile's pipeline drains)
  int next_bh, next_N;  // next_N = 0: no next tile
};

// per-tile scalars indexed by a (possibly runtime) tile: selects keep the
// arrays in registers (a dynamic index would move them to local memory)
__device__ __forceinline__ float rd(const float (&a)[TWFA_MAX_TILES], int k) { return k == 0 ? a[0] : a[1]; }
__device__ __forceinline__ void wr(float (&a)[TWFA_MAX_TILES], int k, float x) {
  if (k == 0) a[0] = x; else a[1] = x;
}

// Ring geometry: depths and prefetch distances of the streamed loads
// (compile-time constants in the specialized kernels).
struct Rings {
  int kd, vd, kpf, vpf;
  // softmax order token (TWFA_SOFTMAX_TOKEN): the EX ops share the MUFU unit
  // and the schedule orders them inside the trip (ex_ring, slot order); the
  // softmax warpgroups then run MX_k + EX_k one after the other in that order
  int ring_len, ring0, ring1;
  int split;  // S_k issued as SA_k + SB_k; P_k at S columns 64-127
};

struct Maps {
  const CUtensorMap* q;
  const CUtensorMap* k;
  const CUtensorMap* v;
};

// ---------------------------------------------------------------- op bodies
// One op of the trip program on this warp, trip r. Shared by both kernels:
// with a compile-time `op` and `rg` every branch below folds.
template <int KV, bool kHeavy, bool kTrace, bool P, bool kSolo = false>
__device__ __forceinline__ void exec_op(const TwfaPlanOp op, const int r, const FaCtx& c, const WorkTile& t,
                                        WarpState& st, const Rings rg, const Maps& tm, const FaArgs& args) {
  FaBarriers& bar = g_sh.bar;
  const uint32_t warp = c.warp, lane = c.lane;
  const uint32_t tmem = c.tmem;
  const int N = t.N;
  using G = Kv<KV, P>;

  if (op.kind == TWFA_OP_LDK || op.kind == TWFA_OP_LDV) {
    if constexpr (!kHeavy) {
      // streamed load: top the ring up to iteration r - stage + prefetch.
      // Warp-uniform address arithmetic (uniform datapath); one elected lane
      // issues the TMA.
      const bool is_k = op.kind == TWFA_OP_LDK;
      const int pf = is_k ? rg.kpf : rg.vpf;
      // iterations past N belong to the next work tile (global iteration
      // numbering, and with it the ring slots and phases, runs on)
      const int target = min(N - 1 + min(pf, st.next_N), r - static_cast<int>(op.stage) + pf);
      int& next = is_k ? st.k_next : st.v_next;
      while (next <= target) {
        const int lit = next++;
        const bool cross = lit >= N;
        const int key0 = (cross ? lit - N : lit) * KV, bh = cross ? st.next_bh : t.bh;
        uint32_t* tr = trace_begin<kTrace>(args, warp, st.trace_n, op.node, cross ? lit - N : lit, r,
                                           t.tcount + (cross ? 1u : 0u), cross ? st.next_N : N);
        const uint32_t g = t.gbase + static_cast<uint32_t>(lit);
        const int depth = is_k ? rg.kd : rg.vd;
        const uint32_t s = g % depth, ph = (g / depth) & 1;
        uint64_t* full = is_k ? &bar.k_full[s] : &bar.v_full[s];
        uint64_t* empty = is_k ? &bar.k_empty[s] : &bar.v_empty[s];
        uint8_t* dst = (is_k ? c.k_smem : c.v_smem) + s * G::slot;
        const CUtensorMap* map = is_k ? tm.k : tm.v;
        if (!(TWFA_WHATIF == 6 && g >= 8u)) wait_<P>(empty, ph ^ 1);
        trace_mark<kTrace>(tr, 4);
        if (lead<kSolo>()) {
          if constexpr (P) {
            // this CTA's half: K keys 64r.. (both head-dim halves), V head
            // dims 64r.. (all keys); both halves land on the leader's barrier
            if (c.rank == 0) mbar_arrive_expect_tx(full, 2 * G::slot);
            const int r0 = static_cast<int>(c.rank);
            if (is_k) {
              tma_load_3d_pair(dst, map, full, 0, key0 + r0 * (KV / 2), bh, c.pol_kv);
              tma_load_3d_pair(dst + G::k_half, map, full, 64, key0 + r0 * (KV / 2), bh, c.pol_kv);
            } else {
              tma_load_3d_pair(dst, map, full, r0 * 64, key0, bh, c.pol_kv);
            }
          } else if (TWFA_WHATIF == 4 && g >= static_cast<uint32_t>(depth)) {
            mbar_arrive(full);  // what-if: the tile is already resident (no L2 -> SM traffic)
          } else {
            mbar_arrive_expect_tx(full, G::tile);
            tma_load_3d(dst, map, full, 0, key0, bh, c.pol_kv);
            tma_load_3d(dst + G::half, map, full, 64, key0, bh, c.pol_kv);
          }
        }
        wsync<kSolo>();
        trace_mark<kTrace>(tr, 5);
      }
    }
    return;
  }
  const int it = r - static_cast<int>(op.stage);
  if (it < 0 || it >= N) return;
  if (op.kind == TWFA_OP_EX && (op.flags & TWFA_OPF_FUSED)) return;  // done by MX_k
  // the leader issues the pair's tensor-core ops (its MMA warp is the peer's
  // load warp too, which only runs the loads of the program)
  if (P && c.rank != 0 && (op.kind == TWFA_OP_S || op.kind == TWFA_OP_PV || op.kind == TWFA_OP_SA ||
                           op.kind == TWFA_OP_SB))
    return;
  const uint32_t g = t.gbase + static_cast<uint32_t>(it);
  const int k = op.tile;
  const uint32_t b = g % G::depth, pb = (g / G::depth) & 1;  // S buffer of this iteration, its phase
  uint32_t* tr = trace_begin<kTrace>(args, warp, st.trace_n, op.node, it, r, t.tcount, N);

  if (op.kind == TWFA_OP_SA || op.kind == TWFA_OP_SB) {
    // split S_k (single 128-key S tile): SA_k = keys 0-63 into columns 0-63,
    // issued once MX_k(g-1) holds its row in registers; SB_k = keys 64-127
    // into columns 64-127, where P_k(g-1) lives, after PV_k(g-1)
    const bool a = op.kind == TWFA_OP_SA;
    const uint32_t s = g % rg.kd;
    if (it == 0) mbar_wait(&bar.q_full[k], t.tcount & 1);
    if (a && g >= 1)
      mbar_wait_all(&bar.k_full[s], (g / rg.kd) & 1, &bar.s_read[k], (g - 1) & 1);
    else if (!a && g >= 1 && !(op.flags & TWFA_OPF_INORDER))
      mbar_wait_all(&bar.k_full[s], (g / rg.kd) & 1, &bar.o_done[k][0], (g - 1) & 1);
    else
      mbar_wait(&bar.k_full[s], (g / rg.kd) & 1);
    trace_mark<kTrace>(tr, 4);
    tc_fence_after();
    const uint32_t qd = sdesc_lo(smem_u32(c.q_smem + k * kTileBytes), 16);
    // K rows 64.. (8 SW128 atoms)
    const uint32_t kd = sdesc_lo(smem_u32(c.k_smem + s * G::tile) + (a ? 0u : 64u * 128u), 16);
    const uint32_t d_s = tmem + k * 128 + (a ? 0u : 64u);
    if (lead<kSolo>()) {
#pragma unroll
      for (int kk = 0; kk < kHeadDim / 16; ++kk)
        mma_ss(d_s, sdesc_join(qd + ((kk >> 2) * kHalfBytes + (kk & 3) * 32) / 16, kSdescHi),
               sdesc_join(kd + ((kk >> 2) * G::half + (kk & 3) * 32) / 16, kSdescHi), kIdescS64, kk > 0);
      mma_commit(a ? &bar.s_half[k] : &bar.s_full[k][0]);
      mma_commit(&bar.k_empty[s]);
      if (it == N - 1) mma_commit(&bar.q_empty[k]);
    }
    wsync<kSolo>();
  } else if (op.kind == TWFA_OP_S) {
    // MMA issue: every lane waits and computes the (warp-uniform)
    // descriptors, so they live in uniform registers; one elected lane
    // issues the tcgen05.mma chain and the commits
    const uint32_t s = g % rg.kd;
    if (it == 0) wait_<P>(&bar.q_full[k], t.tcount & 1);
    if ((TWFA_WHATIF == 5 || TWFA_WHATIF == 6) && g >= 8u) {
    } else if (g >= G::depth && !(op.flags & TWFA_OPF_INORDER))  // K landed; P_k(g-depth) consumed by PV_k
      wait_all_<P>(&bar.k_full[s], (g / rg.kd) & 1, &bar.o_done[k][b], pb ^ 1);
    else if (!TWFA_MEMO_WAITS || st.k_seen != g + 1)  // (the other sub-tile's S on this warp saw K(g) land)
      wait_<P>(&bar.k_full[s], (g / rg.kd) & 1);
    st.k_seen = g + 1;
    trace_mark<kTrace>(tr, 4);
    tc_fence_after();
    const uint32_t qd = sdesc_lo(smem_u32(c.q_smem + k * kTileBytes), 16);
    const uint32_t kd = sdesc_lo(smem_u32(c.k_smem + s * G::slot), 16);
    const uint32_t d_s = tmem + k * 128 + b * KV;
    if constexpr (P) {
      // M = 256 (Q_k of both CTAs), N = 128 keys (64 from each CTA's half)
      if (lead<kSolo>()) {
#pragma unroll
        for (int kk = 0; kk < kHeadDim / 16; ++kk)
          mma_ss_pair(d_s, sdesc_join(qd + ((kk >> 2) * kHalfBytes + (kk & 3) * 32) / 16, kSdescHi),
                      sdesc_join(kd + ((kk >> 2) * G::k_half + (kk & 3) * 32) / 16, kSdescHi), G::idesc_s, kk > 0);
        commit_<P>(&bar.s_full[k][b]);
        commit_<P>(&bar.k_empty[s]);
        if (it == N - 1) commit_<P>(&bar.q_empty[k]);
      }
      wsync<kSolo>();
    } else if (lead<kSolo>()) {
      if (TWFA_S_HALVES && KV == 128) {
        // keys 0-63, committed on their own, then keys 64-127: the softmax
        // starts on the first half while the second is computed
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int kk = 0; kk < kHeadDim / 16; ++kk)
            mma_ss(d_s + 64 * h, sdesc_join(qd + ((kk >> 2) * kHalfBytes + (kk & 3) * 32) / 16, kSdescHi),
                   sdesc_join(kd + ((kk >> 2) * G::half + h * 64 * 128 + (kk & 3) * 32) / 16, kSdescHi), kIdescS64,
                   kk > 0);
          if (h == 0) mma_commit(&bar.s_lo[k][b]);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < kHeadDim / 16; ++kk)  // 16 head dims per step, 4 per SW128 half
          mma_ss(d_s, sdesc_join(qd + ((kk >> 2) * kHalfBytes + (kk & 3) * 32) / 16, kSdescHi),
                 sdesc_join(kd + ((kk >> 2) * G::half + (kk & 3) * 32) / 16, kSdescHi), G::idesc_s, kk > 0);
      }
      mma_commit(&bar.s_full[k][b]);
      mma_commit(&bar.k_empty[s]);
      if (it == N - 1) mma_commit(&bar.q_empty[k]);
    }
    wsync<kSolo>();
  } else if (op.kind == TWFA_OP_PV) {
    const uint32_t s = g % rg.vd;
    // P_k arrives in two halves (keys 0-63, 64-127): the first four
    // K-steps of PV_k overlap the exponentials of the second half
    constexpr int kParts = KV == 128 ? p_parts<P>() : 2;
    constexpr int kSteps = KV / 16 / kParts;  // K-steps (16 keys) per part
    // probe every input of the op at once (non-blocking test_wait: the
    // round trips overlap), then block only on what had not landed: a wait
    // on this warp costs a ~160-clk shared-memory round trip even when the
    // phase completed long ago, and the parts arriving one by one would
    // otherwise serialize four of them into PV's issue
    bool part_ready[kParts];
#if TWFA_PROBE_PARTS
    const bool skip = (TWFA_WHATIF == 5 || TWFA_WHATIF == 6) && g >= 8u;
    const bool v_ok = skip || (TWFA_MEMO_WAITS && st.v_seen == g + 1) ? true : test_<P>(&bar.v_full[s], (g / rg.vd) & 1);
    const bool o_ok = skip || test_<P>(&bar.o_ready[k][b], pb);
#pragma unroll
    for (int j = 0; j < kParts; ++j) part_ready[j] = test_<P>(&bar.p_part[k][b][j], pb);
    if (!v_ok) wait_<P>(&bar.v_full[s], (g / rg.vd) & 1);
    if (!o_ok) wait_<P>(&bar.o_ready[k][b], pb);
    if (!part_ready[0]) wait_<P>(&bar.p_part[k][b][0], pb);
#else
#pragma unroll
    for (int j = 0; j < kParts; ++j) part_ready[j] = false;
    mbar_wait_all(&bar.v_full[s], (g / rg.vd) & 1, &bar.p_part[k][b][0], pb, &bar.o_ready[k][b], pb);
#endif
    st.v_seen = g + 1;
    trace_mark<kTrace>(tr, 4);
    tc_fence_after();
    const uint32_t vd = sdesc_lo(smem_u32(c.v_smem + s * G::slot), G::half);
    const uint32_t d_o = tmem + 256 + k * 128, a_p = tmem + k * 128 + b * KV + (rg.split ? 64u : 0u);
    const uint32_t acc0 = it > 0 ? 1u : 0u;
#pragma unroll
    for (int j = 0; j < kParts; ++j) {
      if (j > 0 && !part_ready[j]) {
        wait_<P>(&bar.p_part[k][b][j], pb);
        tc_fence_after();
      }
      if (lead<kSolo>()) {
#pragma unroll
        for (int kk = j * kSteps; kk < (j + 1) * kSteps; ++kk) {  // V is MN-major: 16 keys = 16 rows of 128 B
          if constexpr (P)  // M = 256 (P_k of both CTAs), N = 128 head dims (64 from each CTA's half)
            mma_ts_pair(d_o, a_p + kk * 8, sdesc_join(vd + kk * 2048 / 16, kSdescHi), G::idesc_pv,
                        kk > 0 ? 1u : acc0);
          else
            mma_ts(d_o, a_p + kk * 8, sdesc_join(vd + kk * 2048 / 16, kSdescHi), kIdescPV, kk > 0 ? 1u : acc0);
        }
        if (j == kParts - 1) {
          commit_<P>(&bar.o_done[k][b]);
          commit_<P>(&bar.v_empty[s]);
        }
      }
      wsync<kSolo>();
    }
  } else if (op.kind == TWFA_OP_CR) {
    const uint32_t sb = g & 1;
    mbar_wait(&bar.st_full[k][sb], (g >> 1) & 1);
    const float alpha = g_sh.stats[k][sb][c.quad * 32 + lane];
    const float m_row = kCrExp<KV> ? g_sh.mrow[k][sb][c.quad * 32 + lane] : 0.f;
    if (TWFA_ST_EMPTY) warp_arrive(&bar.st_empty[k][sb]);
    if constexpr (kCrExp<KV>) {
      // the last 32 keys of the row's P when MX_k took the speculative path
      // (m_row finite for the whole warp; split-S plans never offload)
      float l3 = it == 0 ? 0.f : rd(st.l3, k) * alpha;
      if (!rg.split && __all_sync(0xffffffffu, m_row == m_row)) {
        trace_mark<kTrace>(tr, 4);
        const uint32_t s_addr = tmem + c.lane_off + k * 128 + b * KV;
        const float2 sl2 = make_float2(c.scale_log2, c.scale_log2), nm2 = make_float2(-m_row, -m_row);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[16], pk[8];
          tmem_ld16(s_addr + KV - 32 + h * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 x = ffma2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sl2, nm2);
            const float2 p = poly_exp2x2(x);
            acc = fadd2(acc, p);
            pk[i >> 1] = pack_bf16(p.x, p.y);
          }
          tmem_st8(s_addr + (KV - 32) / 2 + h * 8, pk);
        }
        tmem_st_wait();
        l3 += acc.x + acc.y;
      }
      wr(st.l3, k, l3);
      tc_fence_before();
      arrive_mma_<P>(&bar.p_part[k][b][p_parts<P>() - 1]);
    }
    // PV_k(g - 1) has completed: O may be read-modified-written. Awaited on
    // every iteration (TWFA_CR_WAIT_ALL), so every phase of o_done has a
    // waiter; the wait returns at once with 128-key tiles (S_k(g), which
    // MX_k(g) waited for, follows PV_k(g - 1) on the tensor pipe)
    if (TWFA_CR_WAIT_ALL && g > 0) wait_<P>(&bar.o_done[k][(g - 1) % G::depth], ((g - 1) / G::depth) & 1);
    // with the rescale threshold most iterations keep the max: then O is
    // not touched and the correction only forwards the handoff
    if (it > 0 && !__all_sync(0xffffffffu, alpha == 1.f)) {
      if (!TWFA_CR_WAIT_ALL) wait_<P>(&bar.o_done[k][(g - 1) % G::depth], ((g - 1) / G::depth) & 1);
      trace_mark<kTrace>(tr, 4);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        const uint32_t addr = tmem + c.lane_off + 256 + k * 128 + cc * 32;
        tmem_ld32(addr, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 o =
              fmul2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), make_float2(alpha, alpha));
          v[i] = __float_as_uint(o.x);
          v[i + 1] = __float_as_uint(o.y);
        }
        tmem_st32(addr, v);
      }
      tmem_st_wait();
    }
    tc_fence_before();
    arrive_mma_<P>(&bar.o_ready[k][b]);
  } else if (op.kind == TWFA_OP_MX || op.kind == TWFA_OP_EX) {
    if constexpr (kHeavy) {
      const uint32_t taddr = tmem + c.lane_off + k * 128 + b * KV;
      const int row = sub_tile_row<KV, P>(c, t, k) + c.quad * 32 + lane;
      const int limit = valid_keys<KV>(args, row, it * KV);
      const bool mask = !__all_sync(0xffffffffu, limit >= KV);
      uint32_t srow[KV];
      const bool tok = TWFA_SOFTMAX_TOKEN && rg.ring_len == 2 && (op.flags & TWFA_OPF_FUSE_NEXT);
      if (op.kind == TWFA_OP_MX) {
        if (tok) mbar_wait(&bar.sm_tok[k], (g & 1) ^ (k == rg.ring0 ? 1u : 0u));
        const bool spec = KV == 128 && TWFA_SPEC_EX && !rg.split && !mask && (op.flags & TWFA_OPF_FUSE_NEXT) &&
                          __all_sync(0xffffffffu, rd(st.m_run, k) != -INFINITY);
        if (rg.split)
          mbar_wait_all(&bar.s_half[k], g & 1, &bar.s_full[k][b], pb);
        else if (TWFA_S_HALVES && spec)
          mbar_wait(&bar.s_lo[k][b], pb);  // keys 0-63; the rest is awaited inside the speculative EX
        else
          wait_<P>(&bar.s_full[k][b], pb);
        trace_mark<kTrace>(tr, 4);
        tc_fence_after();
        if constexpr (KV == 128) {
          const float m_old = rd(st.m_run, k);
          if (spec) {
            float m = m_old, alpha = 1.f;
            const uint32_t sb = g & 1;
            const float sum = mx_ex_spec<KV, P, kCrExp<KV>>(srow, taddr, c.scale_log2, m, alpha, bar.p_part[k][b], [&](float al) {
              if (TWFA_ST_EMPTY) mbar_wait(&bar.st_empty[k][sb], ((g >> 1) & 1) ^ 1);
              g_sh.stats[k][sb][c.quad * 32 + lane] = al;
              if constexpr (kCrExp<KV>) g_sh.mrow[k][sb][c.quad * 32 + lane] = m;
              warp_arrive(&bar.st_full[k][sb]);
            }, [&] {
              if (TWFA_S_HALVES) {
                mbar_wait(&bar.s_full[k][b], pb);
                tc_fence_after();
              }
            }, tr);
            wr(st.m_run, k, m);
            wr(st.alpha, k, alpha);
            wr(st.l_run, k, rd(st.l_run, k) * alpha + sum);
            if (!TWFA_LATE_SUM) {
              tc_fence_before();
              arrive_mma_<P>(&bar.p_part[k][b][p_parts<P>() - 1]);
            }
            if (it == N - 1) {
              mbar_wait(&bar.l_empty[k], (t.tcount & 1) ^ 1);
              g_sh.lbuf[k][0][c.quad * 32 + lane] = m;
              g_sh.lbuf[k][1][c.quad * 32 + lane] = rd(st.l_run, k);
              warp_arrive(&bar.l_full[k]);
            }
            // the trace keeps one record per op: EX_k ran inside this MX_k
            trace_mark<kTrace>(tr, 5);
            uint32_t* tr_ex = trace_begin<kTrace>(args, warp, st.trace_n, op.node + 1, it, r, t.tcount, N);
            trace_mark<kTrace>(tr_ex, 4);
            trace_mark<kTrace>(tr_ex, 5);
            return;
          }
        }
        if (TWFA_WHATIF == 3) {
#pragma unroll
          for (int c2 = 0; c2 < KV / 64; ++c2)
            tmem_ld32(taddr + c2 * 32, *reinterpret_cast<uint32_t(*)[32]>(&srow[c2 * 32]));
          tmem_ld_wait();
#pragma unroll
          for (int i = KV / 2; i < KV; ++i) srow[i] = srow[i - KV / 2];
        } else {
          load_row<KV>(taddr, srow);
        }
        if (rg.split) {  // the row is in registers: SA_k(g+1) may overwrite columns 0-63
          tc_fence_before();
          warp_arrive(&bar.s_read[k]);
        }
        if (mask) mask_row<KV>(srow, limit);
        const float mx = row_max<KV>(srow);
        const float m_old = rd(st.m_run, k);
        const float m_cand = fmaxf(m_old, mx * c.scale_log2);
        const float m_new = (m_cand - m_old > kRescaleLog2) ? m_cand : m_old;  // m_old = -inf -> m_cand
        const float m_safe = m_new == -INFINITY ? 0.f : m_new;
        wr(st.alpha, k, m_new == m_old ? 1.f : fast_exp2(m_old - m_safe));
        wr(st.m_run, k, m_new);
        const uint32_t sb = g & 1;
        if (TWFA_ST_EMPTY) mbar_wait(&bar.st_empty[k][sb], ((g >> 1) & 1) ^ 1);
        g_sh.stats[k][sb][c.quad * 32 + lane] = rd(st.alpha, k);
        if constexpr (kCrExp<KV>) g_sh.mrow[k][sb][c.quad * 32 + lane] = __int_as_float(0x7fffffff);  // NaN: all chunks here
        warp_arrive(&bar.st_full[k][sb]);
        trace_mark<kTrace>(tr, 5);
        if (!(op.flags & TWFA_OPF_FUSE_NEXT)) return;
        // EX_k is this warp's next op: run it on the resident S row
        tr = trace_begin<kTrace>(args, warp, st.trace_n, op.node + 1, it, r, t.tcount, N);
        trace_mark<kTrace>(tr, 4);
      } else {
        // unfused EX (other ops run between MX_k and EX_k on this warp):
        // re-read S; the running max and alpha of MX_k are in registers
        trace_mark<kTrace>(tr, 4);
        load_row<KV>(taddr, srow);
        if (mask) mask_row<KV>(srow, limit);
      }
      const float m_run = rd(st.m_run, k);
      const float m_safe = m_run == -INFINITY ? 0.f : m_run;
      const uint32_t paddr = taddr + (rg.split ? 64u : 0u);  // P_k columns
      const float sum = mask ? exp_store_row<KV, true, P>(srow, paddr, c.scale_log2, m_safe, bar.p_part[k][b])
                             : exp_store_row<KV, false, P>(srow, paddr, c.scale_log2, m_safe, bar.p_part[k][b]);
      wr(st.l_run, k, rd(st.l_run, k) * rd(st.alpha, k) + sum);
      tc_fence_before();
      arrive_mma_<P>(&bar.p_part[k][b][(KV == 128 ? p_parts<P>() : 2) - 1]);
      if (tok) warp_arrive(&bar.sm_tok[k == rg.ring0 ? rg.ring1 : rg.ring0]);
      if (it == N - 1) {
        mbar_wait(&bar.l_empty[k], (t.tcount & 1) ^ 1);
        g_sh.lbuf[k][0][c.quad * 32 + lane] = m_run;
        g_sh.lbuf[k][1][c.quad * 32 + lane] = rd(st.l_run, k);
        warp_arrive(&bar.l_full[k]);
      }
    }
  }
  trace_mark<kTrace>(tr, 5);
}

// Q sub-tiles of a new work tile (TMA warp, before its trip loop). With CTA
// pairs each CTA loads its own sub-tile rows onto the leader's barrier.
template <int KV, bool P, bool kSolo = false>
__device__ __forceinline__ void load_q(const FaCtx& c, const WorkTile& t, int tiles, const Maps& tm) {
  FaBarriers& bar = g_sh.bar;
  for (int k = 0; k < tiles; ++k) {
    wait_<P>(&bar.q_empty[k], (t.tcount & 1) ^ 1);
    uint8_t* dst = c.q_smem + k * kTileBytes;
    const int row = sub_tile_row<KV, P>(c, t, k);
    if (lead<kSolo>()) {
      if constexpr (P) {
        if (c.rank == 0) mbar_arrive_expect_tx(&bar.q_full[k], 2 * kTileBytes);
        tma_load_3d_pair(dst, tm.q, &bar.q_full[k], 0, row, t.bh, c.pol_q);
        tma_load_3d_pair(dst + kHalfBytes, tm.q, &bar.q_full[k], 64, row, t.bh, c.pol_q);
      } else {
        mbar_arrive_expect_tx(&bar.q_full[k], kTileBytes);
        tma_load_3d(dst, tm.q, &bar.q_full[k], 0, row, t.bh, c.pol_q);
        tma_load_3d(dst + kHalfBytes, tm.q, &bar.q_full[k], 64, row, t.bh, c.pol_q);
      }
    }
    wsync<kSolo>();
  }
}

// Epilogue of sub-tile k on its correction warpgroup: O / l -> bf16 -> global,
// LSE (the accumulator is final after the last PV_k).
template <int KV, bool P>
__device__ __forceinline__ void epilogue(const FaCtx& c, const WorkTile& t, int k, const FaArgs& args,
                                         float l_cr = 0.f) {
  FaBarriers& bar = g_sh.bar;
  const uint32_t lane = c.lane;
  const uint32_t g_last = t.gbase + static_cast<uint32_t>(t.N - 1);
  wait_<P>(&bar.o_done[k][g_last % Kv<KV>::depth], (g_last / Kv<KV>::depth) & 1);
  mbar_wait(&bar.l_full[k], t.tcount & 1);
  const float m = g_sh.lbuf[k][0][c.quad * 32 + lane];
  const float l = g_sh.lbuf[k][1][c.quad * 32 + lane] + l_cr;  // + the correction warps' share (TWFA_CR_EXP)
  warp_arrive(&bar.l_empty[k]);
  tc_fence_after();
  const int row0 = sub_tile_row<KV, P>(c, t, k);
  const int row = row0 + c.quad * 32 + lane;
  const float inv = l > 0.f ? 1.f / l : 0.f;
#if TWFA_TMA_EPILOGUE
  // two 128 x 64 halves through the swizzled staging buffer and a bulk
  // tensor store each (rows past S are clipped by the tensor map): the
  // epilogue issues 16 shared stores per thread instead of 16 scattered
  // global ones, which otherwise flood the MIO queue the TMA / MMA warp
  // shares at the work-tile boundary
  const uint32_t wg_bar = 1 + (c.warp >> 2);  // named barrier of this warpgroup
  const bool leader = (c.warp & 3u) == 0 && lane == 0;
  const uint32_t r = c.quad * 32 + lane;  // row inside the sub-tile
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    uint32_t v[64];
    tmem_ld32(c.tmem + c.lane_off + 256 + k * 128 + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
    tmem_ld32(c.tmem + c.lane_off + 256 + k * 128 + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
    tmem_ld_wait();
    const uint32_t rbase = smem_u32(c.o_smem) + r * 128;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {  // 16-byte chunk ch of the row, SW128: chunk ^ (row % 8)
      st_shared_v4(rbase + ((ch ^ (r & 7)) << 4),
                   pack_bf16(__uint_as_float(v[8 * ch + 0]) * inv, __uint_as_float(v[8 * ch + 1]) * inv),
                   pack_bf16(__uint_as_float(v[8 * ch + 2]) * inv, __uint_as_float(v[8 * ch + 3]) * inv),
                   pack_bf16(__uint_as_float(v[8 * ch + 4]) * inv, __uint_as_float(v[8 * ch + 5]) * inv),
                   pack_bf16(__uint_as_float(v[8 * ch + 6]) * inv, __uint_as_float(v[8 * ch + 7]) * inv));
    }
    fence_proxy_async_shared();
    named_bar_sync(wg_bar, 128);
    if (leader) {
      tma_store_3d(&args.tm_o, c.o_smem, h * 64, row0, t.bh);
      bulk_commit();
      bulk_wait_read();  // the staging buffer is reusable
    }
    named_bar_sync(wg_bar, 128);
  }
#else
  __nv_bfloat16* orow = args.o + (static_cast<int64_t>(t.bh) * c.S + row) * kHeadDim;
#pragma unroll 1
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t v[32];
    tmem_ld32(c.tmem + c.lane_off + 256 + k * 128 + cc * 32, v);
    tmem_ld_wait();
    if (row < c.S) {
      uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(v[8 * i + 0]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
        w.y = pack_bf16(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
        w.z = pack_bf16(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
        w.w = pack_bf16(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
        dst[i] = w;
      }
    }
  }
#endif
  if (args.lse != nullptr && row < c.S)
    args.lse[static_cast<int64_t>(t.bh) * c.S + row] = (m + __log2f(l)) * 0.69314718055994531f;
  tc_fence_before();
}

// Work-tile loop of one warp. `trip` runs the warp's trip program for trip r.
// The i-th work tile of this CTA: from the host's per-CTA list (causal:
// load-balanced, (b, h)-grouped for L2 reuse of K / V), else round-robin
// over the persistent CTAs.
// A work unit is one CTA, or one CTA pair (both CTAs walk the same list).
__device__ __forceinline__ int work_of(const FaCtx& c, const FaArgs& args, int i) {
  if (args.work_list != nullptr) {
    const int o = args.work_off[c.unit] + i;
    return o < args.work_off[c.unit + 1] ? args.work_list[o] : c.num_work;
  }
  // causal without a list: longest first, alternating the direction of each
  // round over the persistent units ("snake") to balance their totals
  return i * c.units + ((args.causal && (i & 1)) ? c.units - 1 - c.unit : c.unit);
}

// cross-tile prefetch (Q on an idle warp, the next tile's first K / V
// iterations on the TMA warp); 0 = each tile starts from empty rings
#ifndef TWFA_SOLO
#define TWFA_SOLO 0  // measured: one-lane TMA / MMA warp -9 % per clock (pair), -4 % (one CTA)
#endif
#ifndef TWFA_XTILE
#define TWFA_XTILE 1
#endif
template <int KV, bool P, bool kSolo = false, class Trip>
__device__ __forceinline__ void work_loop(const FaCtx& c, const FaArgs& args, const Maps& tm, int tiles, int max_stage,
                                          bool is_load_warp, bool is_q_warp, const int* cr_warp, WarpState& st,
                                          Trip&& trip) {
  uint32_t gbase = 0, tcount = 0;
  st.k_next = st.v_next = 0;
  st.k_seen = st.v_seen = 0;
  for (int round = 0;; ++round, ++tcount) {
    const int work = work_of(c, args, round);
    if (work >= c.num_work) break;
    const WorkTile t = work_tile<KV, P>(c, args, work, gbase, tcount);
    if (TWFA_XTILE && is_q_warp) {  // Q of every tile, as soon as the previous tile's last S_k released it
      load_q<KV, P, kSolo>(c, t, tiles, tm);
      gbase += static_cast<uint32_t>(t.N);
      continue;
    }
    if (is_load_warp) {
      if (!TWFA_XTILE || !(c.q_warp >= 0)) load_q<KV, P, kSolo>(c, t, tiles, tm);
      const int nwork = work_of(c, args, round + 1);
      st.next_N = 0;
      if (TWFA_XTILE && nwork < c.num_work) {
        const WorkTile nt = work_tile<KV, P>(c, args, nwork, gbase + static_cast<uint32_t>(t.N), tcount + 1);
        st.next_bh = nt.bh;
        st.next_N = nt.N;
      }
    }
#pragma unroll
    for (int k = 0; k < TWFA_MAX_TILES; ++k) {
      st.m_run[k] = -INFINITY;
      st.l_run[k] = 0.f;
      st.alpha[k] = 1.f;
    }
    // trip -1 only tops up the streamed-load rings (every timed op has
    // iteration < 0 there): a consumer that precedes its load in the trip
    // program finds iteration 0 already in flight
    const int trips = t.N + max_stage;
    for (int r = -1; r < trips; ++r) trip(r, t);
    for (int k = 0; k < tiles; ++k)
      if (static_cast<int>(c.warp & ~3u) == cr_warp[k]) epilogue<KV, P>(c, t, k, args, kCrExp<KV> ? rd(st.l3, k) : 0.f);
    // iterations of the next tile already in flight keep their count
    st.k_next = max(0, st.k_next - t.N);
    st.v_next = max(0, st.v_next - t.N);
    gbase += static_cast<uint32_t>(t.N);
  }
}

// Shared prologue of both kernels: smem carve-up, barriers, TMEM allocation.
template <int KV, bool P>
__device__ __forceinline__ FaCtx fa_setup(int tiles, int kd, int vd, int load_warp, int q_warp, int split,
                                          const FaArgs& args, const Maps& tm, uint8_t* smem_raw) {
  // 1 KiB alignment of the tile buffers (SW128 atoms) by offset arithmetic on
  // the shared window address, keeping the pointer in the shared space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  FaCtx c;
  c.q_smem = smem;
  c.k_smem = c.q_smem + tiles * kTileBytes;
  c.v_smem = c.k_smem + kd * Kv<KV, P>::slot;
  c.o_smem = c.v_smem + vd * Kv<KV, P>::slot;
  FaBarriers& bar = g_sh.bar;
  c.warp = warp_id();
  c.lane = lane_id();
  c.q_warp = q_warp;
  if (threadIdx.x == 0) {
    for (int k = 0; k < tiles; ++k) {
      mbar_init(&bar.q_full[k], 1);
      mbar_init(&bar.q_empty[k], split ? 2 : 1);  // the last S GEMM(s) of the tile read Q_k
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bar.s_full[k][b], 1);
        // warp arrivals of a warpgroup (of both CTAs' warpgroups: the leader's copy)
        // the last part of a 128-key tile also waits for the correction
        // warps' chunk (TWFA_CR_EXP, every iteration: they arrive without
        // work when MX_k did all chunks)
        for (int j = 0; j < kPParts; ++j)
          mbar_init(&bar.p_part[k][b][j],
                    4 * Kv<KV, P>::rows * (kCrExp<KV> && !split && j == p_parts<P>() - 1 ? 2 : 1));
        mbar_init(&bar.o_ready[k][b], 4 * Kv<KV, P>::rows);
        mbar_init(&bar.o_done[k][b], 1);
      }
      for (int j = 0; j < 2; ++j) {
        mbar_init(&bar.st_full[k][j], 4);
        mbar_init(&bar.st_empty[k][j], 4);
      }
      mbar_init(&bar.sm_tok[k], 4);
      mbar_init(&bar.s_half[k], 1);
      mbar_init(&bar.s_lo[k][0], 1);
      mbar_init(&bar.s_lo[k][1], 1);
      mbar_init(&bar.s_read[k], 4);
      mbar_init(&bar.l_full[k], 4);
      mbar_init(&bar.l_empty[k], 4);
    }
    for (int s = 0; s < kd; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], tiles * (split ? 2 : 1));
    }
    for (int s = 0; s < vd; ++s) {
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], tiles);
    }
    fence_mbar_init();
  }
  if ((c.warp == static_cast<uint32_t>(load_warp) || static_cast<int>(c.warp) == q_warp) && c.lane == 0) {
    tma_prefetch_desc(tm.q);
    tma_prefetch_desc(tm.k);
    tma_prefetch_desc(tm.v);
  }
  if constexpr (P) {
    if (c.warp == 0) tmem_alloc_pair<512>(&bar.tmem_base);
    tc_fence_before();
    cluster_sync();  // both CTAs' barriers initialised and tensor memory allocated
  } else {
    if (c.warp == 0) tmem_alloc<512>(&bar.tmem_base);
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  // the CTA owns all 512 columns (one CTA per SM): the allocation starts at
  // column 0, lane 0, so the base is the compile-time constant 0
  if (bar.tmem_base != 0) __trap();
  c.tmem = 0;
  trace_clock(args, 1);
  c.scale_log2 = args.scale_log2;
  c.S = args.S;
  c.BH = args.B * args.H;
  c.rank = P ? cluster_ctarank() : 0u;
  c.unit = static_cast<int>(blockIdx.x) / Kv<KV, P>::rows;
  c.units = static_cast<int>(gridDim.x) / Kv<KV, P>::rows;
  constexpr int kRows = 2 * kBlockQ * Kv<KV, P>::rows;
  c.q_blocks = (c.S + kRows - 1) / kRows;
  c.num_work = c.BH * c.q_blocks;
  c.quad = c.warp & 3u;               // TMEM lane quadrant of this warp
  c.lane_off = (c.quad * 32u) << 16;  // TMEM address lane field
  c.pol_q = policy_evict_first();
  c.pol_kv = policy_evict_last();
  return c;
}

template <bool P>
__device__ __forceinline__ void fa_teardown(const FaCtx& c, const FaArgs& args) {
  if (c.lane == 0) bulk_wait_all();  // epilogue bulk stores of this warp (if any) are complete
  tc_fence_before();
  if constexpr (P) {
    cluster_sync();  // neither CTA leaves while the pair's MMAs may touch its memory
    trace_clock(args, 3);  // every warp of CTA 0 is done
    if (c.warp == 0) {
      tc_fence_after();
      tmem_dealloc_pair<512>(c.tmem);
    }
  } else {
    __syncthreads();
    trace_clock(args, 3);
    if (c.warp == 0) {
      tc_fence_after();
      tmem_dealloc<512>(c.tmem);
    }
  }
}

template <bool kHeavy>
__device__ __forceinline__ void set_register_class(int heavy_wgs) {
  if constexpr (kHeavy) {
    if (heavy_wgs == 2) setmaxnreg_inc<192>(); else setmaxnreg_inc<232>();
  } else {
    if (heavy_wgs == 2) setmaxnreg_dec<64>(); else setmaxnreg_dec<80>();
  }
}

// ---------------------------------------------------------------- interpreter
template <int KV, bool kHeavy, bool kTrace, bool P>
__device__ __forceinline__ void run_interp(const FaCtx& c, const Maps& tm, const FaArgs& args, int tiles,
                                           int max_stage, int load_warp, const int* cr_warp, const Rings rg) {
  WarpState st;
  st.trace_n = 0;
  int plen = 0;
  while (plen < TWFA_MAX_NODES && g_sh.prog_len[c.warp] > plen) ++plen;
  work_loop<KV, P>(c, args, tm, tiles, max_stage, !kHeavy && c.warp == static_cast<uint32_t>(load_warp),
                !kHeavy && static_cast<int>(c.warp) == c.q_warp, cr_warp, st,
                [&](int r, const WorkTile& t) {
                  for (int j = 0; j < plen; ++j)
                    exec_op<KV, kHeavy, kTrace, P>(g_sh.prog[c.warp][j], r, c, t, st, rg, tm, args);
            });
}

template <int KV, bool kTrace, bool P>
__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_fwd_interp(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ TwfaDevicePlan plan,
                  const __grid_constant__ FaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Maps tm{&tm_q, &tm_k, &tm_v};
  for (int i = threadIdx.x; i < TWFA_MAX_WARPS * TWFA_MAX_NODES; i += blockDim.x) {
    const int w = i / TWFA_MAX_NODES, j = i % TWFA_MAX_NODES;
    if (j < plan.prog_len[w]) g_sh.prog[w][j] = plan.ops[plan.prog[w][j]];
    if (j == 0) g_sh.prog_len[w] = plan.prog_len[w];
  }
  const FaCtx c = fa_setup<KV, P>(plan.num_tiles, plan.k_depth, plan.v_depth, plan.load_warp, plan.q_warp,
                                  plan.s_split, args, tm, smem_raw);
  const Rings rg{plan.k_depth,   plan.v_depth,    plan.k_prefetch, plan.v_prefetch,
                 plan.ex_ring_len, plan.ex_ring[0], plan.ex_ring[1], plan.s_split};
  const bool heavy = (plan.heavy_wg_mask >> (c.warp >> 2)) & 1;
  const int heavy_wgs = __popc(plan.heavy_wg_mask);
  if (heavy) {
    set_register_class<true>(heavy_wgs);
    run_interp<KV, true, kTrace, P>(c, tm, args, plan.num_tiles, plan.max_stage, plan.load_warp, plan.cr_warp, rg);
  } else {
    set_register_class<false>(heavy_wgs);
    run_interp<KV, false, kTrace, P>(c, tm, args, plan.num_tiles, plan.max_stage, plan.load_warp, plan.cr_warp, rg);
  }
  fa_teardown<P>(c, args);
}

// ---------------------------------------------------------------- specialized
// gen::PlanOf<I>::value is a host constexpr object: device code only reads
// its scalar fields in constant expressions (never binds a reference to it).
#define TWFA_PLAN(I) (gen::PlanOf<I>::value)

template <int I, int W, int J>
__device__ __forceinline__ TwfaPlanOp spec_op() {
  constexpr int v = TWFA_PLAN(I).prog[W][J];
  TwfaPlanOp op{};
  op.node = TWFA_PLAN(I).ops[v].node;
  op.kind = TWFA_PLAN(I).ops[v].kind;
  op.tile = TWFA_PLAN(I).ops[v].tile;
  op.stage = TWFA_PLAN(I).ops[v].stage;
  op.slot = TWFA_PLAN(I).ops[v].slot;
  op.warp_start = TWFA_PLAN(I).ops[v].warp_start;
  op.warp_count = TWFA_PLAN(I).ops[v].warp_count;
  op.order = TWFA_PLAN(I).ops[v].order;
  op.flags = TWFA_PLAN(I).ops[v].flags;
  return op;
}

// the interpreted roles read their trip programs from shared memory
template <int I, int W, int... J>
__device__ __forceinline__ void fill_warp_prog(int j, std::integer_sequence<int, J...>) {
  ((j == J ? (void)(g_sh.prog[W][J] = spec_op<I, W, J>()) : void()), ...);
  if (j == 0) g_sh.prog_len[W] = TWFA_PLAN(I).prog_len[W];
}
template <int I, int... W>
__device__ __forceinline__ void fill_progs(int w, int j, std::integer_sequence<int, W...>) {
  ((w == W ? fill_warp_prog<I, W>(j, std::make_integer_sequence<int, TWFA_PLAN(I).prog_len[W]>{}) : void()), ...);
}

template <int I, int W, bool kTrace, bool P, bool kSolo, int... J>
__device__ __forceinline__ void spec_trip(int r, const FaCtx& c, const WorkTile& t, WarpState& st, const Maps& tm,
                                          const FaArgs& args, std::integer_sequence<int, J...>) {
  constexpr bool kHeavy = (TWFA_PLAN(I).heavy_wg_mask >> (W / 4)) & 1;
  constexpr Rings rg{TWFA_PLAN(I).k_depth,    TWFA_PLAN(I).v_depth,    TWFA_PLAN(I).k_prefetch,
                     TWFA_PLAN(I).v_prefetch, TWFA_PLAN(I).ex_ring_len, TWFA_PLAN(I).ex_ring[0],
                     TWFA_PLAN(I).ex_ring[1], TWFA_PLAN(I).s_split};
  (exec_op<TWFA_PLAN(I).kv_tile, kHeavy, kTrace, P, kSolo>(spec_op<I, W, J>(), r, c, t, st, rg, tm, args), ...);
}

// A light role runs on one elected lane (TWFA_SOLO) when its program holds
// only TMA loads and tensor-core issues: no correction, no epilogue, not the
// Q warp (lead / wsync in sm100.cuh)
template <int I, int W>
__host__ __device__ constexpr bool solo_role() {
  if (!TWFA_SOLO || ((TWFA_PLAN(I).heavy_wg_mask >> (W / 4)) & 1) || W == TWFA_PLAN(I).q_warp ||
      TWFA_PLAN(I).prog_len[W] == 0)
    return false;
  for (int k = 0; k < TWFA_PLAN(I).num_tiles; ++k)
    if ((W & ~3) == TWFA_PLAN(I).cr_warp[k]) return false;
  for (int j = 0; j < TWFA_PLAN(I).prog_len[W]; ++j) {
    const int kind = TWFA_PLAN(I).ops[TWFA_PLAN(I).prog[W][j]].kind;
    if (kind != TWFA_OP_LDK && kind != TWFA_OP_LDV && kind != TWFA_OP_S && kind != TWFA_OP_PV &&
        kind != TWFA_OP_SA && kind != TWFA_OP_SB)
      return false;
  }
  return true;
}

template <int I, int W, bool kTrace, bool P>
__device__ __forceinline__ void run_spec(const FaCtx& c, const Maps& tm, const FaArgs& args) {
  constexpr bool kHeavy = (TWFA_PLAN(I).heavy_wg_mask >> (W / 4)) & 1;
  constexpr int plen = TWFA_PLAN(I).prog_len[W];
  constexpr bool kLoad = !kHeavy && W == TWFA_PLAN(I).load_warp;
  constexpr int cr_warp[TWFA_MAX_TILES] = {TWFA_PLAN(I).cr_warp[0], TWFA_PLAN(I).cr_warp[1]};
  constexpr bool kSolo = solo_role<I, W>();
  WarpState st;
  st.trace_n = 0;
  auto body = [&] {
    work_loop<TWFA_PLAN(I).kv_tile, P, kSolo>(c, args, tm, TWFA_PLAN(I).num_tiles, TWFA_PLAN(I).max_stage, kLoad,
                                             !kHeavy && static_cast<int>(c.warp) == c.q_warp, cr_warp, st,
              [&](int r, const WorkTile& t) {
                spec_trip<I, W, kTrace, P, kSolo>(r, c, t, st, tm, args, std::make_integer_sequence<int, plen>{});
              });
  };
  if constexpr (kSolo) {
    if (elect_one()) body();
    __syncwarp();
  } else {
    body();
  }
}

// Light roles (TMA, MMA issue, correction) run their specialized trip
// program, one instantiation per distinct role; softmax warpgroups run the
// runtime interpreter over the same plan (a single shared copy of the large
// MX/EX bodies keeps the kernel within the instruction cache).
template <int I, bool kTrace, bool P, int... W>
__device__ __forceinline__ void spec_dispatch_light(const FaCtx& c, const Maps& tm, const FaArgs& args,
                                                    std::integer_sequence<int, W...>) {
  int role = -1;
  ((c.warp == static_cast<uint32_t>(W) ? (void)(role = gen::PlanOf<I>::role[W]) : void()), ...);
  ((!((TWFA_PLAN(I).heavy_wg_mask >> (W / 4)) & 1) && gen::PlanOf<I>::role[W] == W && role == W
        ? run_spec<I, W, kTrace, P>(c, tm, args)
        : void()),
   ...);
}

template <int I, bool kTrace, bool P>
__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_fwd_spec(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ FaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Maps tm{&tm_q, &tm_k, &tm_v};
  for (int i = threadIdx.x; i < TWFA_MAX_WARPS * TWFA_MAX_NODES; i += blockDim.x)
    fill_progs<I>(i / TWFA_MAX_NODES, i % TWFA_MAX_NODES, std::make_integer_sequence<int, TWFA_MAX_WARPS>{});
  constexpr int cr_warp[TWFA_MAX_TILES] = {TWFA_PLAN(I).cr_warp[0], TWFA_PLAN(I).cr_warp[1]};
  constexpr int KV = TWFA_PLAN(I).kv_tile;
  const FaCtx c = fa_setup<KV, P>(TWFA_PLAN(I).num_tiles, TWFA_PLAN(I).k_depth, TWFA_PLAN(I).v_depth,
                               TWFA_PLAN(I).load_warp, TWFA_PLAN(I).q_warp, TWFA_PLAN(I).s_split, args, tm, smem_raw);
  // the register class is per warpgroup; the warp roles of each class are
  // dispatched inside its branch so ptxas allocates them under that budget
  constexpr int mask = TWFA_PLAN(I).heavy_wg_mask;
  const int heavy_wgs = __popc(mask);
  constexpr int nw = TWFA_PLAN(I).num_warps;
  if ((mask >> (c.warp >> 2)) & 1) {
    set_register_class<true>(heavy_wgs);
    run_interp<KV, true, kTrace, P>(c, tm, args, TWFA_PLAN(I).num_tiles, TWFA_PLAN(I).max_stage, TWFA_PLAN(I).load_warp,
                             cr_warp, Rings{TWFA_PLAN(I).k_depth, TWFA_PLAN(I).v_depth, TWFA_PLAN(I).k_prefetch,
                                            TWFA_PLAN(I).v_prefetch, TWFA_PLAN(I).ex_ring_len,
                                            TWFA_PLAN(I).ex_ring[0], TWFA_PLAN(I).ex_ring[1],
                                            TWFA_PLAN(I).s_split});
  } else {
    set_register_class<false>(heavy_wgs);
    spec_dispatch_light<I, kTrace, P>(c, tm, args, std::make_integer_sequence<int, nw>{});
  }
  fa_teardown<P>(c, args);
}

bool same_plan(const TwfaDevicePlan& a, const TwfaDevicePlan& b) {
  if (a.family != b.family || a.ii != b.ii || a.max_stage != b.max_stage || a.num_nodes != b.num_nodes ||
      a.num_warps != b.num_warps || a.num_tiles != b.num_tiles || a.k_depth != b.k_depth || a.v_depth != b.v_depth ||
      a.load_warp != b.load_warp || a.k_prefetch != b.k_prefetch || a.v_prefetch != b.v_prefetch ||
      a.q_warp != b.q_warp ||
      a.heavy_wg_mask != b.heavy_wg_mask || a.s_depth != b.s_depth || a.kv_tile != b.kv_tile ||
      a.s_split != b.s_split)
    return false;
  for (int k = 0; k < TWFA_MAX_TILES; ++k)
    if (a.cr_warp[k] != b.cr_warp[k] || a.sm_warp[k] != b.sm_warp[k]) return false;
  for (int v = 0; v < a.num_nodes; ++v) {
    const TwfaPlanOp &x = a.ops[v], &y = b.ops[v];
    if (x.node != y.node || x.kind != y.kind || x.tile != y.tile || x.stage != y.stage || x.slot != y.slot ||
        x.warp_start != y.warp_start || x.warp_count != y.warp_count || x.flags != y.flags)
      return false;
  }
  for (int w = 0; w < TWFA_MAX_WARPS; ++w) {
    if (a.prog_len[w] != b.prog_len[w]) return false;
    for (int j = 0; j < a.prog_len[w]; ++j)
      if (a.prog[w][j] != b.prog[w][j]) return false;
  }
  return true;
}

// `cluster` = 2 launches CTA pairs (clusters of two CTAs on one TPC)
template <class Kernel, class... Args>
cudaError_t launch(Kernel kernel, size_t smem, int grid, int threads, cudaStream_t stream, int cluster,
                   Args... args) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (cluster <= 1) {
    kernel<<<grid, threads, smem, stream>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

}  // namespace twfa
