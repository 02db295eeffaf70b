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
#define TWFA_POLY_EVERY 4
#endif
constexpr int kPolyEvery = TWFA_POLY_EVERY;  // 1 in kPolyEvery exp2 pairs on the FMA pipe
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
  FaBarriers bar;
};

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

template <bool kMask>
__device__ __forceinline__ void max_chunk(const uint32_t (&v)[32], int col0, int limit, float (&acc)[4]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float x = __uint_as_float(v[i]);
    if (kMask) x = (col0 + i < limit) ? x : -INFINITY;
    acc[i & 3] = fmaxf(acc[i & 3], x);
  }
}

// MX: row max of the 128 scores of this thread's TMEM lane (raw, unscaled).
template <bool kMask>
__device__ __forceinline__ float tile_row_max(uint32_t taddr, int limit) {
  float acc[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    uint32_t a[32], b[32];
    tmem_ld32(taddr + c * 32, a);
    tmem_ld32(taddr + (c + 1) * 32, b);
    tmem_ld_wait();
    max_chunk<kMask>(a, c * 32, limit, acc);
    max_chunk<kMask>(b, (c + 1) * 32, limit, acc);
  }
  return fmaxf(fmaxf(acc[0], acc[1]), fmaxf(acc[2], acc[3]));
}

template <bool kMask>
__device__ __forceinline__ void exp_chunk(const uint32_t (&v)[32], int col0, int limit, float sl, float neg_m,
                                          float (&acc)[4], uint32_t (&pk)[16]) {
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    // kPolyEvery-th pairs go to the FMA pipe, the rest to MUFU (ex2), to
    // balance the two pipes (MUFU alone co-bounds the loop at d = 128)
    const bool poly = (i >> 1) % kPolyEvery == 0;
    const float x0 = fmaf(__uint_as_float(v[i]), sl, neg_m);
    const float x1 = fmaf(__uint_as_float(v[i + 1]), sl, neg_m);
    float p0 = poly ? poly_exp2(x0) : fast_exp2(x0);
    float p1 = poly ? poly_exp2(x1) : fast_exp2(x1);
    if (kMask) {
      p0 = (col0 + i < limit) ? p0 : 0.f;
      p1 = (col0 + i + 1 < limit) ? p1 : 0.f;
    }
    acc[(i >> 1) & 3] += p0 + p1;
    pk[i >> 1] = pack_bf16(p0, p1);
  }
}

// EX: P = exp2(S * scale*log2e - m) written as bf16 pairs over the first 64
// columns of the S tile (the TS-MMA A operand); returns the row sum of P.
template <bool kMask>
__device__ __forceinline__ float tile_exp_to_p(uint32_t taddr, int limit, float sl, float m) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const float neg_m = -m;
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    uint32_t a[32], b[32];
    tmem_ld32(taddr + c * 32, a);
    tmem_ld32(taddr + (c + 1) * 32, b);
    tmem_ld_wait();
    uint32_t pa[16], pb[16];
    exp_chunk<kMask>(a, c * 32, limit, sl, neg_m, acc, pa);
    exp_chunk<kMask>(b, (c + 1) * 32, limit, sl, neg_m, acc, pb);
    tmem_st16(taddr + c * 16, pa);
    tmem_st16(taddr + (c + 1) * 16, pb);
  }
  tmem_st_wait();
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

}  // namespace

__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ TwfaDevicePlan plan,
                  const __grid_constant__ FaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tiles = plan.num_tiles;
  const int kd = plan.k_depth, vd = plan.v_depth;
  uint8_t* q_smem = smem;
  uint8_t* k_smem = q_smem + tiles * kTileBytes;
  uint8_t* v_smem = k_smem + kd * kTileBytes;
  FaShared* sh = reinterpret_cast<FaShared*>(v_smem + vd * kTileBytes);
  FaBarriers& bar = sh->bar;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (threadIdx.x == 0) {
    for (int k = 0; k < tiles; ++k) {
      mbar_init(&bar.q_full[k], 1);
      mbar_init(&bar.q_empty[k], 1);
      mbar_init(&bar.s_full[k], 1);
      mbar_init(&bar.p_full[k], 128);
      mbar_init(&bar.o_ready[k], 128);
      mbar_init(&bar.o_done[k], 1);
      for (int j = 0; j < 2; ++j) {
        mbar_init(&bar.st_full[k][j], 128);
        mbar_init(&bar.st_empty[k][j], 128);
      }
      mbar_init(&bar.l_full[k], 128);
      mbar_init(&bar.l_empty[k], 128);
      mbar_init(&bar.mufu_tok[k], 128);
    }
    for (int s = 0; s < kd; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], tiles);
    }
    for (int s = 0; s < vd; ++s) {
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], tiles);
    }
    fence_mbar_init();
  }
  if (warp == static_cast<uint32_t>(plan.load_warp) && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 0) tmem_alloc<512>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  const float scale_log2 = args.scale_log2;
  const int S = args.S;
  const int BH = args.B * args.H;
  const int q_blocks = (S + 2 * kBlockQ - 1) / (2 * kBlockQ);
  const int num_work = BH * q_blocks;
  const uint32_t quad = warp & 3u;                   // TMEM lane quadrant of this warp
  const uint32_t lane_off = (quad * 32u) << 16;      // TMEM address lane field
  const uint64_t pol_q = policy_evict_first();
  const uint64_t pol_kv = policy_evict_last();

  // per-thread running softmax state for the sub-tiles whose MX/EX run here
  float m_run[TWFA_MAX_TILES] = {-INFINITY, -INFINITY};
  float l_run[TWFA_MAX_TILES] = {0.f, 0.f};
  float alpha_cur[TWFA_MAX_TILES] = {0.f, 0.f};

  const int plen = plan.prog_len[warp];
  uint32_t gbase = 0;  // global K/V iteration index of this work tile's iteration 0
  uint32_t trace_n = 0;
  uint32_t tcount = 0;
  for (int work = blockIdx.x; work < num_work; work += gridDim.x, ++tcount) {
    int qb, bh;
    if (args.causal) {  // longest-processing-time first
      qb = q_blocks - 1 - work / BH;
      bh = work % BH;
    } else {
      bh = work / q_blocks;
      qb = work % q_blocks;
    }
    const int q0 = qb * 2 * kBlockQ;
    const int kv_end = args.causal ? min(S, q0 + 2 * kBlockQ) : S;
    const int N = (kv_end + kBlockK - 1) / kBlockK;

    if (warp == static_cast<uint32_t>(plan.load_warp) && lane == 0) {
      for (int k = 0; k < tiles; ++k) {
        mbar_wait(&bar.q_empty[k], (tcount & 1) ^ 1);
        mbar_arrive_expect_tx(&bar.q_full[k], kTileBytes);
        uint8_t* dst = q_smem + k * kTileBytes;
        tma_load_3d(dst, &tm_q, &bar.q_full[k], 0, q0 + k * kBlockQ, bh, pol_q);
        tma_load_3d(dst + kHalfBytes, &tm_q, &bar.q_full[k], 64, q0 + k * kBlockQ, bh, pol_q);
      }
    }
    for (int k = 0; k < tiles; ++k) {
      m_run[k] = -INFINITY;
      l_run[k] = 0.f;
    }
    int k_next = 0, v_next = 0;  // next K / V iteration to load (load warp)

    const int trips = N + plan.max_stage;
    for (int r = 0; r < trips; ++r) {
      for (int j = 0; j < plen; ++j) {
        const TwfaPlanOp op = plan.ops[plan.prog[warp][j]];
        if (op.kind == TWFA_OP_LDK || op.kind == TWFA_OP_LDV) {
          // streamed load: top the ring up to iteration r - stage + prefetch
          const bool is_k = op.kind == TWFA_OP_LDK;
          const int target = min(N - 1, r - static_cast<int>(op.stage) + (is_k ? plan.k_prefetch : plan.v_prefetch));
          int& next = is_k ? k_next : v_next;
          while (next <= target) {
            const int lit = next++;
            uint32_t* tr = trace_begin(args, warp, trace_n, op.node, lit, r);
            if (lane == 0) {
              const uint32_t g = gbase + static_cast<uint32_t>(lit);
              const int depth = is_k ? kd : vd;
              const uint32_t s = g % depth, ph = (g / depth) & 1;
              uint64_t* full = is_k ? &bar.k_full[s] : &bar.v_full[s];
              uint64_t* empty = is_k ? &bar.k_empty[s] : &bar.v_empty[s];
              uint8_t* dst = (is_k ? k_smem : v_smem) + s * kTileBytes;
              const CUtensorMap* map = is_k ? &tm_k : &tm_v;
              mbar_wait(empty, ph ^ 1);
              trace_mark(tr, 4);
              mbar_arrive_expect_tx(full, kTileBytes);
              tma_load_3d(dst, map, full, 0, lit * kBlockK, bh, pol_kv);
              tma_load_3d(dst + kHalfBytes, map, full, 64, lit * kBlockK, bh, pol_kv);
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
        switch (op.kind) {
          case TWFA_OP_S: {
            if (lane == 0) {
              const uint32_t s = g % kd;
              mbar_wait(&bar.k_full[s], (g / kd) & 1);
              if (it == 0) mbar_wait(&bar.q_full[k], tcount & 1);
              if (g > 0) mbar_wait(&bar.o_done[k], (g - 1) & 1);  // P_k(g-1) consumed
              trace_mark(tr, 4);
              tc_fence_after();
              const uint32_t qa = smem_u32(q_smem + k * kTileBytes);
              const uint32_t ka = smem_u32(k_smem + s * kTileBytes);
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
            break;
          }
          case TWFA_OP_MX: {
            mbar_wait(&bar.s_full[k], g & 1);
            trace_mark(tr, 4);
            tc_fence_after();
            const uint32_t taddr = tmem + lane_off + k * 128;
            const int limit = valid_keys(args, q0 + k * kBlockQ + quad * 32 + lane, it * kBlockK);
            const bool mask = !__all_sync(0xffffffffu, limit >= kBlockK);
            const float mx = mask ? tile_row_max<true>(taddr, limit) : tile_row_max<false>(taddr, limit);
            const float m_old = m_run[k];
            const float m_new = fmaxf(m_old, mx * scale_log2);
            const float m_safe = m_new == -INFINITY ? 0.f : m_new;
            const float alpha = fast_exp2(m_old - m_safe);
            m_run[k] = m_new;
            alpha_cur[k] = alpha;
            const uint32_t sb = g & 1;
            mbar_wait(&bar.st_empty[k][sb], ((g >> 1) & 1) ^ 1);
            sh->stats[k][sb][quad * 32 + lane] = alpha;
            mbar_arrive(&bar.st_full[k][sb]);
            break;
          }
          case TWFA_OP_EX: {
            const uint32_t taddr = tmem + lane_off + k * 128;
            const int limit = valid_keys(args, q0 + k * kBlockQ + quad * 32 + lane, it * kBlockK);
            const bool mask = !__all_sync(0xffffffffu, limit >= kBlockK);
            const float m_safe = m_run[k] == -INFINITY ? 0.f : m_run[k];
            int ring_pos = -1;
#ifndef TWFA_NO_MUFU_TOKEN
            for (int i = 0; i < plan.ex_ring_len; ++i)
              if (plan.ex_ring[i] == k) ring_pos = i;
#endif
            if (ring_pos >= 0) mbar_wait(&bar.mufu_tok[k], (g & 1) ^ (ring_pos == 0 ? 1u : 0u));
            trace_mark(tr, 4);
            const float sum = mask ? tile_exp_to_p<true>(taddr, limit, scale_log2, m_safe)
                                   : tile_exp_to_p<false>(taddr, limit, scale_log2, m_safe);
            if (ring_pos >= 0) mbar_arrive(&bar.mufu_tok[plan.ex_ring[(ring_pos + 1) % plan.ex_ring_len]]);
            l_run[k] = l_run[k] * alpha_cur[k] + sum;
            tc_fence_before();
            mbar_arrive(&bar.p_full[k]);
            if (it == N - 1) {
              mbar_wait(&bar.l_empty[k], (tcount & 1) ^ 1);
              sh->lbuf[k][0][quad * 32 + lane] = m_run[k];
              sh->lbuf[k][1][quad * 32 + lane] = l_run[k];
              mbar_arrive(&bar.l_full[k]);
            }
            break;
          }
          case TWFA_OP_CR: {
            const uint32_t sb = g & 1;
            mbar_wait(&bar.st_full[k][sb], (g >> 1) & 1);
            const float alpha = sh->stats[k][sb][quad * 32 + lane];
            mbar_arrive(&bar.st_empty[k][sb]);
            if (it > 0) {
              mbar_wait(&bar.o_done[k], (g - 1) & 1);
              trace_mark(tr, 4);
              tc_fence_after();
              if (!__all_sync(0xffffffffu, alpha == 1.f)) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                  uint32_t v[32];
                  const uint32_t addr = tmem + lane_off + 256 + k * 128 + c * 32;
                  tmem_ld32(addr, v);
                  tmem_ld_wait();
#pragma unroll
                  for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
                  tmem_st32(addr, v);
                }
                tmem_st_wait();
              }
            }
            tc_fence_before();
            mbar_arrive(&bar.o_ready[k]);
            break;
          }
          case TWFA_OP_PV: {
            if (lane == 0) {
              const uint32_t s = g % vd;
              mbar_wait(&bar.v_full[s], (g / vd) & 1);
              mbar_wait(&bar.p_full[k], g & 1);
              mbar_wait(&bar.o_ready[k], g & 1);
              trace_mark(tr, 4);
              tc_fence_after();
              const uint32_t va = smem_u32(v_smem + s * kTileBytes);
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
            break;
          }
          default:
            break;
        }
        trace_mark(tr, 5);
      }
    }

    // epilogue of the sub-tiles whose correction runs on this warpgroup:
    // O / l -> bf16 -> global, LSE (the accumulator is final after the last PV)
    for (int k = 0; k < tiles; ++k) {
      if (static_cast<int>(warp & ~3u) != plan.cr_warp[k]) continue;
      const uint32_t g_last = gbase + static_cast<uint32_t>(N - 1);
      mbar_wait(&bar.o_done[k], g_last & 1);
      mbar_wait(&bar.l_full[k], tcount & 1);
      const float m = sh->lbuf[k][0][quad * 32 + lane];
      const float l = sh->lbuf[k][1][quad * 32 + lane];
      mbar_arrive(&bar.l_empty[k]);
      tc_fence_after();
      const int row = q0 + k * kBlockQ + quad * 32 + lane;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = args.o + (static_cast<int64_t>(bh) * S + row) * kHeadDim;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + 256 + k * 128 + c * 32, v);
        tmem_ld_wait();
        if (row < S) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
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
      if (args.lse != nullptr && row < S)
        args.lse[static_cast<int64_t>(bh) * S + row] = (m + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
    }
    gbase += static_cast<uint32_t>(N);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

size_t fa_fwd_smem_bytes(const TwfaDevicePlan& plan) {
  return 1024 + static_cast<size_t>(plan.num_tiles + plan.k_depth + plan.v_depth) * kTileBytes +
         sizeof(FaShared);
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
