// FA-forward on sm_100a, realized from a Twill joint schedule.
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
// asynchronous tensor core still wait on the MMA commit barrier.
//
// Register classes: warpgroups that run softmax ops (MX/EX) raise their
// register budget with setmaxnreg and keep a 128-column S row resident; the
// other warpgroups (TMA, MMA issue, correction) lower theirs. The interpreter
// is instantiated once per class so each compiles within its budget.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fa_fwd.h"
#include "sm100.cuh"

namespace twfa {

namespace {

constexpr int kBlockQ = 128;  // rows per Q sub-tile (= TMEM lanes)
constexpr int kBlockK = 128;  // keys per K/V tile
constexpr int kHeadDim = 128;
constexpr uint32_t kTileBytes = kBlockQ * kHeadDim * 2;  // 32 KiB, two 16 KiB SW128 column halves
constexpr uint32_t kHalfBytes = kTileBytes / 2;
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
constexpr uint32_t kIdescS = idesc_bf16_f32(128, kBlockK, 0);    // K-major Q, K-major K
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, kHeadDim, 1);  // TMEM P, MN-major V

struct __align__(8) FaBarriers {
  uint64_t q_full[TWFA_MAX_TILES], q_empty[TWFA_MAX_TILES];
  uint64_t k_full[kMaxRing], k_empty[kMaxRing];
  uint64_t v_full[kMaxRing], v_empty[kMaxRing];
  uint64_t s_full[TWFA_MAX_TILES], p_full[TWFA_MAX_TILES];
  uint64_t o_ready[TWFA_MAX_TILES], o_done[TWFA_MAX_TILES];
  uint64_t st_full[TWFA_MAX_TILES][2], st_empty[TWFA_MAX_TILES][2];
  uint64_t l_full[TWFA_MAX_TILES], l_empty[TWFA_MAX_TILES];
  uint64_t mufu_tok[TWFA_MAX_TILES];  // EX_k may use MUFU (schedule's unit order)
  uint32_t tmem_base;
};

struct FaShared {
  float stats[TWFA_MAX_TILES][2][kBlockQ];  // MX -> CR rescale factors, double-buffered
  float lbuf[TWFA_MAX_TILES][2][kBlockQ];   // EX -> epilogue: running max, row sum
  // per-warp trip programs copied out of the kernel parameters once: one
  // 8-byte shared load per op instead of chained indexed constant loads
  TwfaPlanOp prog[TWFA_MAX_WARPS][TWFA_MAX_NODES];
  FaBarriers bar;
};

// Barriers, handoff buffers and trip programs live in static shared memory so
// every access compiles to LDS/STS/SYNCS on a known shared address (generic
// pointers carved out of the dynamic window cost generic-load latency on
// every op transition).
__shared__ FaShared g_sh;

// Issue trace of CTA 0 (debug / schedule-realization evidence). Per warp:
// word 0 = record count, then records of kTraceWords uint32:
// {node, iteration, trip, t_issue, t_ready (inputs waited), t_done}.
constexpr int kTraceWords = 8;

__device__ __forceinline__ uint32_t* trace_begin(const FaArgs& a, uint32_t warp, uint32_t& n, int node, int it,
                                                 int trip) {
  if (a.trace == nullptr || blockIdx.x != 0 || lane_id() != 0) return nullptr;
  uint32_t* base = a.trace + static_cast<size_t>(warp) * a.trace_cap * kTraceWords;
  if (n + 1 >= a.trace_cap) return nullptr;
  uint32_t* e = base + (n + 1) * kTraceWords;
  e[0] = static_cast<uint32_t>(node);
  e[1] = static_cast<uint32_t>(it);
  e[2] = static_cast<uint32_t>(trip);
  e[3] = static_cast<uint32_t>(clock64());
  base[0] = ++n;  // count kept in a register; the store is fire-and-forget
  return e;
}
__device__ __forceinline__ void trace_mark(uint32_t* e, int field) {
  if (e != nullptr) e[field] = static_cast<uint32_t>(clock64());
}

// Number of leading keys of this K/V tile that row `row` may attend to
// (the rest are past the sequence end or above the causal diagonal).
__device__ __forceinline__ int valid_keys(const FaArgs& a, int row, int key0) {
  const int end = a.causal ? min(a.S, row + 1) : a.S;
  return max(0, min(kBlockK, end - key0));
}

// ---------------------------------------------------------------- softmax pieces
// all 128 scores of this thread's TMEM lane, one wait
__device__ __forceinline__ void load_row(uint32_t taddr, uint32_t (&s)[128]) {
  tmem_ld32(taddr + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
  tmem_ld32(taddr + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
  tmem_ld32(taddr + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
  tmem_ld_wait();
}

__device__ __forceinline__ void mask_row(uint32_t (&s)[128], int limit) {
#pragma unroll
  for (int i = 0; i < 128; ++i)
    if (i >= limit) s[i] = __float_as_uint(-INFINITY);
}

__device__ __forceinline__ float row_max(const uint32_t (&s)[128]) {
  float a[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int i = 0; i < 128; i += 8) {
    a[(i >> 3) & 3] = fmaxf(a[(i >> 3) & 3], fmaxf(fmaxf(__uint_as_float(s[i]), __uint_as_float(s[i + 1])),
                                                   fmaxf(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]))));
    a[(i >> 3) & 3] = fmaxf(a[(i >> 3) & 3], fmaxf(fmaxf(__uint_as_float(s[i + 4]), __uint_as_float(s[i + 5])),
                                                   fmaxf(__uint_as_float(s[i + 6]), __uint_as_float(s[i + 7]))));
  }
  return fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
}

// P = exp2(S*sl - m) for the 128 resident scores: FFMA2 for the argument,
// MUFU ex2 or the FMA-pipe polynomial (1 in kPolyEvery pairs) for the exp,
// FADD2 for the row sum, F2FP to bf16 pairs, stored as the TS-MMA A operand
// over the first 64 columns of the S tile. Returns the row sum.
template <bool kMask>
__device__ __forceinline__ float exp_store_row(const uint32_t (&s)[128], uint32_t taddr, float sl, float m) {
  const float2 sl2 = make_float2(sl, sl);
  const float2 nm2 = make_float2(-m, -m);
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 x =
          ffma2(make_float2(__uint_as_float(s[c * 32 + i]), __uint_as_float(s[c * 32 + i + 1])), sl2, nm2);
      float2 p;
      // masked tiles (diagonal / sequence tail) hold -inf: MUFU maps it to 0
      if (!kMask && ((i >> 1) % kPolyEvery) == kPolyEvery - 1) {
        p.x = poly_exp2(x.x);
        p.y = poly_exp2(x.y);
      } else {
        p.x = fast_exp2(x.x);
        p.y = fast_exp2(x.y);
      }
      acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], p);
      pk[i >> 1] = pack_bf16(p.x, p.y);
    }
    tmem_st16(taddr + c * 16, pk);
  }
  tmem_st_wait();
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

// ---------------------------------------------------------------- state
struct FaCtx {
  uint8_t* q_smem;
  uint8_t* k_smem;
  uint8_t* v_smem;
  uint32_t tmem;
  uint32_t warp, lane, quad, lane_off;
  int tiles, kd, vd;
  int S, BH, q_blocks, num_work;
  float scale_log2;
  uint64_t pol_q, pol_kv;
};

template <bool kHeavy>
__device__ __forceinline__ void run_warp(const FaCtx& c, const CUtensorMap* tm_q, const CUtensorMap* tm_k,
                                         const CUtensorMap* tm_v, const TwfaDevicePlan& plan, const FaArgs& args) {
  FaBarriers& bar = g_sh.bar;
  const uint32_t warp = c.warp, lane = c.lane;
  const uint32_t tmem = c.tmem;
  const int plen = plan.prog_len[warp];
  // running softmax state (used only by heavy warpgroups)
  float m_run0 = -INFINITY, m_run1 = -INFINITY, l_run0 = 0.f, l_run1 = 0.f;
  uint32_t gbase = 0;  // global K/V iteration index of this work tile's iteration 0
  uint32_t trace_n = 0;
  uint32_t tcount = 0;
  for (int work = blockIdx.x; work < c.num_work; work += gridDim.x, ++tcount) {
    int qb, bh;
    if (args.causal) {  // longest-processing-time first
      qb = c.q_blocks - 1 - work / c.BH;
      bh = work % c.BH;
    } else {
      bh = work / c.q_blocks;
      qb = work % c.q_blocks;
    }
    const int q0 = qb * 2 * kBlockQ;
    const int kv_end = args.causal ? min(c.S, q0 + 2 * kBlockQ) : c.S;
    const int N = (kv_end + kBlockK - 1) / kBlockK;

    if (!kHeavy && warp == static_cast<uint32_t>(plan.load_warp) && lane == 0) {
      for (int k = 0; k < c.tiles; ++k) {
        mbar_wait(&bar.q_empty[k], (tcount & 1) ^ 1);
        mbar_arrive_expect_tx(&bar.q_full[k], kTileBytes);
        uint8_t* dst = c.q_smem + k * kTileBytes;
        tma_load_3d(dst, tm_q, &bar.q_full[k], 0, q0 + k * kBlockQ, bh, c.pol_q);
        tma_load_3d(dst + kHalfBytes, tm_q, &bar.q_full[k], 64, q0 + k * kBlockQ, bh, c.pol_q);
      }
    }
    m_run0 = m_run1 = -INFINITY;
    l_run0 = l_run1 = 0.f;
    int k_next = 0, v_next = 0;  // next K / V iteration to load (load warp)

    const int trips = N + plan.max_stage;
    for (int r = 0; r < trips; ++r) {
      for (int j = 0; j < plen; ++j) {
        const TwfaPlanOp op = g_sh.prog[warp][j];
        if (!kHeavy && (op.kind == TWFA_OP_LDK || op.kind == TWFA_OP_LDV)) {
          // streamed load: top the ring up to iteration r - stage + prefetch
          const bool is_k = op.kind == TWFA_OP_LDK;
          const int target = min(N - 1, r - static_cast<int>(op.stage) + (is_k ? plan.k_prefetch : plan.v_prefetch));
          int& next = is_k ? k_next : v_next;
          while (next <= target) {
            const int lit = next++;
            uint32_t* tr = trace_begin(args, warp, trace_n, op.node, lit, r);
            if (lane == 0) {
              const uint32_t g = gbase + static_cast<uint32_t>(lit);
              const int depth = is_k ? c.kd : c.vd;
              const uint32_t s = g % depth, ph = (g / depth) & 1;
              uint64_t* full = is_k ? &bar.k_full[s] : &bar.v_full[s];
              uint64_t* empty = is_k ? &bar.k_empty[s] : &bar.v_empty[s];
              uint8_t* dst = (is_k ? c.k_smem : c.v_smem) + s * kTileBytes;
              const CUtensorMap* map = is_k ? tm_k : tm_v;
              mbar_wait(empty, ph ^ 1);
              trace_mark(tr, 4);
              mbar_arrive_expect_tx(full, kTileBytes);
              tma_load_3d(dst, map, full, 0, lit * kBlockK, bh, c.pol_kv);
              tma_load_3d(dst + kHalfBytes, map, full, 64, lit * kBlockK, bh, c.pol_kv);
            }
            trace_mark(tr, 5);
          }
          continue;
        }
        const int it = r - static_cast<int>(op.stage);
        if (it < 0 || it >= N) continue;
        const uint32_t g = gbase + static_cast<uint32_t>(it);
        const int k = op.tile;
        uint32_t* tr = trace_begin(args, warp, trace_n, op.node, it, r);
        if (op.kind == TWFA_OP_S) {
          if (lane == 0) {
            const uint32_t s = g % c.kd;
            if (it == 0) mbar_wait(&bar.q_full[k], tcount & 1);
            if (g > 0)  // K landed; P_k(g-1) consumed by PV_k(g-1)
              mbar_wait_all(&bar.k_full[s], (g / c.kd) & 1, &bar.o_done[k], (g - 1) & 1);
            else
              mbar_wait(&bar.k_full[s], (g / c.kd) & 1);
            trace_mark(tr, 4);
            tc_fence_after();
            const uint32_t qa = smem_u32(c.q_smem + k * kTileBytes);
            const uint32_t ka = smem_u32(c.k_smem + s * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < kHeadDim / 16; ++kk) {
              const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
              mma_ss(tmem + k * 128, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(ka + off, 16, 1024), kIdescS,
                     kk > 0);
            }
            mma_commit(&bar.s_full[k]);
            mma_commit(&bar.k_empty[s]);
            if (it == N - 1) mma_commit(&bar.q_empty[k]);
          }
          __syncwarp();
        } else if (op.kind == TWFA_OP_PV) {
          if (lane == 0) {
            const uint32_t s = g % c.vd;
#ifdef TWFA_SERIAL_WAITS
            mbar_wait(&bar.v_full[s], (g / c.vd) & 1);
            mbar_wait(&bar.p_full[k], g & 1);
            mbar_wait(&bar.o_ready[k], g & 1);
#else
            mbar_wait_all(&bar.v_full[s], (g / c.vd) & 1, &bar.p_full[k], g & 1, &bar.o_ready[k], g & 1);
#endif
            trace_mark(tr, 4);
            tc_fence_after();
            const uint32_t va = smem_u32(c.v_smem + s * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < kBlockK / 16; ++kk) {
              // V tile is MN-major (head dim contiguous): 16 keys = 16 rows of 128 B
              mma_ts(tmem + 256 + k * 128, tmem + k * 128 + kk * 8, sdesc_sw128(va + kk * 2048, kHalfBytes, 1024),
                     kIdescPV, (it > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&bar.o_done[k]);
            mma_commit(&bar.v_empty[s]);
          }
          __syncwarp();
        } else if (op.kind == TWFA_OP_CR) {
          const uint32_t sb = g & 1;
          mbar_wait(&bar.st_full[k][sb], (g >> 1) & 1);
          const float alpha = g_sh.stats[k][sb][c.quad * 32 + lane];
          warp_arrive(&bar.st_empty[k][sb]);
          // with the rescale threshold most iterations keep the max: then O is
          // not touched and the correction only forwards the handoff
          if (it > 0 && !__all_sync(0xffffffffu, alpha == 1.f)) {
            mbar_wait(&bar.o_done[k], (g - 1) & 1);
            trace_mark(tr, 4);
            tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
              uint32_t v[32];
              const uint32_t addr = tmem + c.lane_off + 256 + k * 128 + cc * 32;
              tmem_ld32(addr, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float2 o = fmul2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])),
                                       make_float2(alpha, alpha));
                v[i] = __float_as_uint(o.x);
                v[i + 1] = __float_as_uint(o.y);
              }
              tmem_st32(addr, v);
            }
            tmem_st_wait();
          }
          tc_fence_before();
          warp_arrive(&bar.o_ready[k]);
        } else if (kHeavy && op.kind == TWFA_OP_MX) {
          mbar_wait(&bar.s_full[k], g & 1);
          trace_mark(tr, 4);
          tc_fence_after();
          const uint32_t taddr = tmem + c.lane_off + k * 128;
          const int row = q0 + k * kBlockQ + c.quad * 32 + lane;
          const int limit = valid_keys(args, row, it * kBlockK);
          const bool mask = !__all_sync(0xffffffffu, limit >= kBlockK);
          uint32_t srow[128];
          load_row(taddr, srow);
          if (mask) mask_row(srow, limit);
          const float mx = row_max(srow);
          const float m_old = k == 0 ? m_run0 : m_run1;
          const float m_cand = fmaxf(m_old, mx * c.scale_log2);
          const float m_new = (m_cand - m_old > kRescaleLog2) ? m_cand : m_old;  // m_old = -inf -> m_cand
          const float m_safe = m_new == -INFINITY ? 0.f : m_new;
          const float alpha = m_new == m_old ? 1.f : fast_exp2(m_old - m_safe);
          if (k == 0) m_run0 = m_new; else m_run1 = m_new;
          const uint32_t sb = g & 1;
          mbar_wait(&bar.st_empty[k][sb], ((g >> 1) & 1) ^ 1);
          g_sh.stats[k][sb][c.quad * 32 + lane] = alpha;
          warp_arrive(&bar.st_full[k][sb]);
          trace_mark(tr, 5);
          if (!(op.flags & TWFA_OPF_FUSE_NEXT)) continue;
          // EX_k is this warp's next op: run it on the resident S row
          ++j;
          tr = trace_begin(args, warp, trace_n, g_sh.prog[warp][j].node, it, r);
          int ring_pos = -1;
#ifdef TWFA_MUFU_TOKEN
          for (int i = 0; i < plan.ex_ring_len; ++i)
            if (plan.ex_ring[i] == k) ring_pos = i;
          if (ring_pos >= 0) mbar_wait(&bar.mufu_tok[k], (g & 1) ^ (ring_pos == 0 ? 1u : 0u));
#endif
          trace_mark(tr, 4);
          const float sum = mask ? exp_store_row<true>(srow, taddr, c.scale_log2, m_safe)
                                 : exp_store_row<false>(srow, taddr, c.scale_log2, m_safe);
          if (ring_pos >= 0) warp_arrive(&bar.mufu_tok[plan.ex_ring[(ring_pos + 1) % plan.ex_ring_len]]);
          float& l_run = k == 0 ? l_run0 : l_run1;
          l_run = l_run * alpha + sum;
          tc_fence_before();
          warp_arrive(&bar.p_full[k]);
          if (it == N - 1) {
            mbar_wait(&bar.l_empty[k], (tcount & 1) ^ 1);
            g_sh.lbuf[k][0][c.quad * 32 + lane] = m_new;
            g_sh.lbuf[k][1][c.quad * 32 + lane] = l_run;
            warp_arrive(&bar.l_full[k]);
          }
        } else if (kHeavy && op.kind == TWFA_OP_EX) {
          // unfused EX (other ops run between MX_k and EX_k on this warp):
          // re-read S and use the running max MX_k left in registers
          const uint32_t taddr = tmem + c.lane_off + k * 128;
          const int row = q0 + k * kBlockQ + c.quad * 32 + lane;
          const int limit = valid_keys(args, row, it * kBlockK);
          const bool mask = !__all_sync(0xffffffffu, limit >= kBlockK);
          const float m = k == 0 ? m_run0 : m_run1;
          const float m_safe = m == -INFINITY ? 0.f : m;
          const float alpha = g_sh.stats[k][g & 1][c.quad * 32 + lane];
          trace_mark(tr, 4);
          uint32_t srow[128];
          load_row(taddr, srow);
          if (mask) mask_row(srow, limit);
          const float sum = mask ? exp_store_row<true>(srow, taddr, c.scale_log2, m_safe)
                                 : exp_store_row<false>(srow, taddr, c.scale_log2, m_safe);
          float& l_run = k == 0 ? l_run0 : l_run1;
          l_run = l_run * alpha + sum;
          tc_fence_before();
          warp_arrive(&bar.p_full[k]);
          if (it == N - 1) {
            mbar_wait(&bar.l_empty[k], (tcount & 1) ^ 1);
            g_sh.lbuf[k][0][c.quad * 32 + lane] = m;
            g_sh.lbuf[k][1][c.quad * 32 + lane] = l_run;
            warp_arrive(&bar.l_full[k]);
          }
        }
        trace_mark(tr, 5);
      }
    }

    // epilogue of the sub-tiles whose correction runs on this warpgroup:
    // O / l -> bf16 -> global, LSE (the accumulator is final after the last PV)
    for (int k = 0; k < c.tiles; ++k) {
      if (static_cast<int>(warp & ~3u) != plan.cr_warp[k]) continue;
      const uint32_t g_last = gbase + static_cast<uint32_t>(N - 1);
      mbar_wait(&bar.o_done[k], g_last & 1);
      mbar_wait(&bar.l_full[k], tcount & 1);
      const float m = g_sh.lbuf[k][0][c.quad * 32 + lane];
      const float l = g_sh.lbuf[k][1][c.quad * 32 + lane];
      warp_arrive(&bar.l_empty[k]);
      tc_fence_after();
      const int row = q0 + k * kBlockQ + c.quad * 32 + lane;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = args.o + (static_cast<int64_t>(bh) * c.S + row) * kHeadDim;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(tmem + c.lane_off + 256 + k * 128 + cc * 32, v);
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
      if (args.lse != nullptr && row < c.S)
        args.lse[static_cast<int64_t>(bh) * c.S + row] = (m + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
    }
    gbase += static_cast<uint32_t>(N);
  }
}

}  // namespace

__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ TwfaDevicePlan plan,
                  const __grid_constant__ FaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB alignment of the tile buffers (SW128 atoms) by offset arithmetic on
  // the shared window address, keeping the pointer in the shared space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  FaCtx c;
  c.tiles = plan.num_tiles;
  c.kd = plan.k_depth;
  c.vd = plan.v_depth;
  c.q_smem = smem;
  c.k_smem = c.q_smem + c.tiles * kTileBytes;
  c.v_smem = c.k_smem + c.kd * kTileBytes;
  FaBarriers& bar = g_sh.bar;
  c.warp = warp_id();
  c.lane = lane_id();

  for (int i = threadIdx.x; i < TWFA_MAX_WARPS * TWFA_MAX_NODES; i += blockDim.x) {
    const int w = i / TWFA_MAX_NODES, j = i % TWFA_MAX_NODES;
    if (j < plan.prog_len[w]) g_sh.prog[w][j] = plan.ops[plan.prog[w][j]];
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < c.tiles; ++k) {
      mbar_init(&bar.q_full[k], 1);
      mbar_init(&bar.q_empty[k], 1);
      mbar_init(&bar.s_full[k], 1);
      mbar_init(&bar.p_full[k], 4);  // warp arrivals of a warpgroup
      mbar_init(&bar.o_ready[k], 4);
      mbar_init(&bar.o_done[k], 1);
      for (int j = 0; j < 2; ++j) {
        mbar_init(&bar.st_full[k][j], 4);
        mbar_init(&bar.st_empty[k][j], 4);
      }
      mbar_init(&bar.l_full[k], 4);
      mbar_init(&bar.l_empty[k], 4);
      mbar_init(&bar.mufu_tok[k], 4);
    }
    for (int s = 0; s < c.kd; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], c.tiles);
    }
    for (int s = 0; s < c.vd; ++s) {
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], c.tiles);
    }
    fence_mbar_init();
  }
  if (c.warp == static_cast<uint32_t>(plan.load_warp) && c.lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (c.warp == 0) tmem_alloc<512>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  c.tmem = bar.tmem_base;
  c.scale_log2 = args.scale_log2;
  c.S = args.S;
  c.BH = args.B * args.H;
  c.q_blocks = (c.S + 2 * kBlockQ - 1) / (2 * kBlockQ);
  c.num_work = c.BH * c.q_blocks;
  c.quad = c.warp & 3u;               // TMEM lane quadrant of this warp
  c.lane_off = (c.quad * 32u) << 16;  // TMEM address lane field
  c.pol_q = policy_evict_first();
  c.pol_kv = policy_evict_last();

  const bool heavy = (plan.heavy_wg_mask >> (c.warp >> 2)) & 1;
  const int heavy_wgs = __popc(plan.heavy_wg_mask);
  if (heavy) {
    if (heavy_wgs == 2) setmaxnreg_inc<192>(); else setmaxnreg_inc<232>();
    run_warp<true>(c, &tm_q, &tm_k, &tm_v, plan, args);
  } else {
    if (heavy_wgs == 2) setmaxnreg_dec<64>(); else setmaxnreg_dec<80>();
    run_warp<false>(c, &tm_q, &tm_k, &tm_v, plan, args);
  }

  tc_fence_before();
  __syncthreads();
  if (c.warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(c.tmem);
  }
}

size_t fa_fwd_smem_bytes(const TwfaDevicePlan& plan) {
  // dynamic part only: tile buffers (+ alignment slack); FaShared is static
  return 1024 + static_cast<size_t>(plan.num_tiles + plan.k_depth + plan.v_depth) * kTileBytes;
}

cudaError_t fa_fwd_launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          const TwfaDevicePlan& plan, const FaArgs& args, int grid, cudaStream_t stream) {
  const size_t smem = fa_fwd_smem_bytes(plan);
  cudaError_t e = cudaFuncSetAttribute(fa_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fa_fwd_kernel<<<grid, plan.num_warps * 32, smem, stream>>>(tq, tk, tv, plan, args);
  return cudaGetLastError();
}

}  // namespace twfa
