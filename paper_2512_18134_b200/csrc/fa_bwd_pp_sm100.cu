// FA-backward on sm_100a with two 64-query sub-tiles per iteration, realized
// from a Twill joint schedule (tools/make_problems.py:fa_backward_pp_problem,
// schedules/fa_bwd_pp.solution.json): the paper's Blackwell backward
// -- the exponential / dS work of the two halves of
// every Q tile runs on two warpgroups that ping-pong, while the tensor core
// works on the other half, and further warps stage the dQ reduction.
//
// One CTA owns a 128-key K/V tile of one (b, h) (K, V in shared memory; dK,
// dV accumulate in tensor memory) and iterates over 128-row Q / dO tiles.
// Sub-tile k = queries 64k .. 64k + 63 of the tile:
//   ST_k   S^T_k  = K Q_k^T      TMEM cols 256 + 128k (64 fp32, keys on lanes)
//   EXB_k  P^T_k  = exp2(S^T_k * scale*log2e - LSE*log2e) -> bf16 over S^T_k
//   DP_k   dP^T_k = V dO_k^T     TMEM cols 320 + 128k
//   DS_k   dS^T_k = P^T_k (dP^T_k - D) -> bf16 over dP^T_k (A of DK_k) and
//          into shared memory (MN-major B operand of DQ_k)
//   DV_k   dV    += P^T_k dO_k   TS, TMEM cols 128..255
//   DK_k   dK    += dS^T_k Q_k   TS, TMEM cols 0..127
//   DQ_k   dQ^T_k = K^T dS^T_k   SS (A = K MN-major, M = head dim), TMEM over S^T_k
//   RD_k   dQ^T_k (fp32, d on lanes) -> shared memory as [query][d] in two
//          64-column passes -> cp.reduce.async.bulk.tensor add into the fp32
//          dQ accumulator
// Each sub-tile has its own tensor-memory buffers (S^T_k / P^T_k / dQ^T_k
// and dP^T_k / dS^T_k), so the halves only meet in the dK / dV
// accumulators, which the tensor core updates in issue order. The aliasing
// edges of the loop graph (DV_k -> DQ_k, DK_k -> DP_k: in order on the
// issuing thread; RD_k -> ST_k, RD_k -> DS_k, DQ_k -> DS_k: mbarriers) are
// checked by the lowering.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fa_bwd.h"
#include "sm100.cuh"

namespace twfa {

namespace {

constexpr int kT = 128;                // keys per K/V tile = rows per Q tile
constexpr int kH = 64;                 // queries per sub-tile
constexpr uint32_t kTile = 32768;      // 128 x 128 bf16: two 64-column SW128 halves
constexpr uint32_t kHalf = 16384;
constexpr uint32_t kSubRows = kH * 128;  // byte offset of sub-tile 1's rows inside a tile half (8 KiB)
constexpr uint32_t kDsBytes = 16384;   // dS^T_k: 128 keys x 64 queries bf16 (MN-major B), or dQ staging
constexpr uint32_t kColDK = 0, kColDV = 128;
__host__ __device__ constexpr uint32_t col_s(int k) { return 256 + 128 * k; }  // S^T_k, P^T_k, dQ^T_k
__host__ __device__ constexpr uint32_t col_p(int k) { return 320 + 128 * k; }  // dP^T_k, dS^T_k
constexpr float kLog2e = 1.4426950408889634f;
constexpr uint32_t kIdescN64 = idesc_bf16_f32(128, 64, 0);                    // A, B K-major, N = 64
constexpr uint32_t kIdescTS = idesc_bf16_f32(128, 128, 1);                    // A TMEM, B MN-major, N = 128
constexpr uint32_t kIdescDQ = idesc_bf16_f32(128, 64, 1) | (1u << 15);       // A, B MN-major, N = 64
constexpr uint32_t kSdHi = sdesc_hi(1024);

struct __align__(8) PpBarriers {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[2], q_empty[2], o_full[2], o_empty[2];
  uint64_t s_full[2], dp_full[2], dq_full[2];  // tcgen05.commit
  uint64_t p_full[2], ds_full[2];              // EXB / DS warpgroup of sub-tile k (4 warp arrivals)
  uint64_t q_free[2];                          // RD_k read dQ^T_k out of TMEM (4)
  uint64_t ds_free[2];                         // RD_k is done with the dS_k buffer (1)
  uint64_t acc_full, acc_free;                 // dK, dV of the work item final / read out
  uint32_t tmem_base;
};
__shared__ PpBarriers g_pb;
// LSE * log2(e) and D of the current sub-tile's 64 queries, per sub-tile
__shared__ __align__(16) float g_pp_lse2[2][kH];
__shared__ __align__(16) float g_pp_dvec[2][kH];

struct PpCtx {
  uint8_t* k;
  uint8_t* v;
  uint8_t* q;   // ring of Q tiles (128 rows)
  uint8_t* o;   // ring of dO tiles
  uint8_t* ds;  // two dS^T buffers (MN-major B of DQ_k), then dQ staging of RD_k
  uint32_t warp, lane, quad, lane_off;
  int S, BH, nq, num_work;
  uint64_t pol;
};

struct PpItem {
  int bh, kv0, q_first, N;  // N = Q tiles of this work item
  uint32_t gbase;           // global iteration index of its iteration 0
  uint32_t icount;          // work items done by this CTA
};

struct PpState {
  int q_next, o_next;  // next Q / dO iteration to load (TMA warp)
  uint32_t trace_n;
  uint32_t* rec;       // current op's trace record
  bool dv_started, dk_started;  // the work item's first DV / DK MMA initialises the accumulator
  // 1 + the last global iteration whose Q (dO) tile the MMA warp has seen
  // land: later readers of the tile skip the wait
  uint32_t q_seen, o_seen;
};

__device__ __forceinline__ PpItem pp_item(const PpCtx& c, const FaBwdArgs& a, int work, uint32_t gbase,
                                          uint32_t icount) {
  PpItem t;
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

// issue trace of CTA 0 (lane 0 of every warp), the layout of the other kernels
__device__ __forceinline__ uint32_t* pp_trace(const FaBwdArgs& a, const PpCtx& c, PpState& st, int node, int it,
                                              int trip, const PpItem& t) {
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
__device__ __forceinline__ void pp_ready(PpState& st) {
  if (st.rec != nullptr) st.rec[4] = static_cast<uint32_t>(clock64());
}

// streamed Q / dO loads (128-row tiles): top the ring up to iteration `upto`
__device__ __forceinline__ void pp_top_up(const PpCtx& c, const FaBwdArgs& a, const PpItem& t, PpState& st,
                                          const TwfaDevicePlan& plan, bool is_q, int upto) {
  PpBarriers& bar = g_pb;
  int& next = is_q ? st.q_next : st.o_next;
  const int depth = is_q ? plan.k_depth : plan.v_depth;
  while (next <= upto) {
    const int lit = next++;
    const uint32_t g = t.gbase + static_cast<uint32_t>(lit);
    const uint32_t s = g % depth, ph = (g / depth) & 1;
    mbar_wait(is_q ? &bar.q_empty[s] : &bar.o_empty[s], ph ^ 1);
    uint64_t* full = is_q ? &bar.q_full[s] : &bar.o_full[s];
    if (elect_one()) {
      uint8_t* dst = (is_q ? c.q : c.o) + s * kTile;
      const CUtensorMap* map = is_q ? &a.tm_q : &a.tm_do;
      const int row = (t.q_first + lit) * kT;
      mbar_arrive_expect_tx(full, kTile);
      tma_load_3d(dst, map, full, 0, row, t.bh, c.pol);
      tma_load_3d(dst + kHalf, map, full, 64, row, t.bh, c.pol);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint32_t sd_lo(const void* p, uint32_t lbo) { return sdesc_lo(smem_u32(p), lbo); }

// EXB_k + DS_k on the sub-tile's warpgroup (thread = key row r): P^T_k row in
// fp32 registers from the exponentials into dS^T_k.
__device__ __forceinline__ void exb_ds(const PpCtx& c, const FaBwdArgs& a, const PpItem& t, int it, uint32_t g, int k,
                                       PpState& st) {
  PpBarriers& bar = g_pb;
  const int q0 = (t.q_first + it) * kT + k * kH;  // first query of the sub-tile
  const uint32_t r = c.quad * 32 + c.lane;
  const int key = t.kv0 + static_cast<int>(r);
  const int64_t row0 = static_cast<int64_t>(t.bh) * c.S + q0;
  const uint32_t nb = 1 + (c.warp >> 2);  // named barrier of this warpgroup
  // this sub-tile's LSE and D: threads 0..63 load one query each
  const bool vec_thread = r < static_cast<uint32_t>(kH);
  const bool in = vec_thread && q0 + static_cast<int>(r) < c.S;
  const float my_lse2 = in ? a.lse[row0 + r] * kLog2e : INFINITY;  // rows past S: P = 0
  const float my_d = in ? a.dvec[row0 + r] : 0.f;
  mbar_wait(&bar.s_full[k], g & 1);
  tc_fence_after();
  pp_ready(st);
  uint32_t p[kH];
  tmem_ld32(c.lane_off + col_s(k), *reinterpret_cast<uint32_t(*)[32]>(&p[0]));
  tmem_ld32(c.lane_off + col_s(k) + 32, *reinterpret_cast<uint32_t(*)[32]>(&p[32]));
  named_bar_sync(nb, 128);  // the previous sub-tile's readers of the staged vectors are done
  if (vec_thread) {
    g_pp_lse2[k][r] = my_lse2;
    g_pp_dvec[k][r] = my_d;
  }
  named_bar_sync(nb, 128);
  tmem_ld_wait();
  const float sl = a.scale_log2;
  const bool diag = a.causal && it == 0;  // the diagonal Q tile (first query q0 - 64k == kv0)
#pragma unroll
  for (int j4 = 0; j4 < kH / 4; ++j4) {
    const float4 l = reinterpret_cast<const float4*>(g_pp_lse2[k])[j4];
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
  for (int cc = 0; cc < 2; ++cc) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      pk[i] = pack_bf16(__uint_as_float(p[cc * 32 + 2 * i]), __uint_as_float(p[cc * 32 + 2 * i + 1]));
    tmem_st16(c.lane_off + col_s(k) + cc * 16, pk);
  }
  tmem_st_wait();
  tc_fence_before();
  warp_arrive(&bar.p_full[k]);
  // DS_k: the dS_k buffer must be free (RD_k(g-1) staged dQ^T in it after
  // DQ_k(g-1) read dS from it)
  if (g >= 1) mbar_wait(&bar.ds_free[k], (g - 1) & 1);  // one phase per iteration (RD_k(g - 1))
  mbar_wait(&bar.dp_full[k], g & 1);
  tc_fence_after();
  uint32_t dp[kH];
  tmem_ld32(c.lane_off + col_p(k), *reinterpret_cast<uint32_t(*)[32]>(&dp[0]));
  tmem_ld32(c.lane_off + col_p(k) + 32, *reinterpret_cast<uint32_t(*)[32]>(&dp[32]));
  tmem_ld_wait();
  uint32_t pk[kH / 2];
#pragma unroll
  for (int j4 = 0; j4 < kH / 4; ++j4) {
    const float4 d = reinterpret_cast<const float4*>(g_pp_dvec[k])[j4];
    const float s0 = __uint_as_float(p[4 * j4 + 0]) * (__uint_as_float(dp[4 * j4 + 0]) - d.x);
    const float s1 = __uint_as_float(p[4 * j4 + 1]) * (__uint_as_float(dp[4 * j4 + 1]) - d.y);
    const float s2 = __uint_as_float(p[4 * j4 + 2]) * (__uint_as_float(dp[4 * j4 + 2]) - d.z);
    const float s3 = __uint_as_float(p[4 * j4 + 3]) * (__uint_as_float(dp[4 * j4 + 3]) - d.w);
    pk[2 * j4] = pack_bf16(s0, s1);
    pk[2 * j4 + 1] = pack_bf16(s2, s3);
  }
  tmem_st16(c.lane_off + col_p(k), *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
  tmem_st16(c.lane_off + col_p(k) + 16, *reinterpret_cast<uint32_t(*)[16]>(&pk[16]));
  // dS^T_k row r (64 queries, 128 B) into the MN-major B operand of DQ_k:
  // SW128, 16-byte chunk ch of row r at ch ^ (r % 8)
  const uint32_t ds_row = smem_u32(c.ds + k * kDsBytes) + r * 128;
#pragma unroll
  for (int ch = 0; ch < 8; ++ch)
    st_shared_v4(ds_row + ((ch ^ (r & 7)) << 4), pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
  tmem_st_wait();
  tc_fence_before();
  fence_proxy_async_shared();
  warp_arrive(&bar.ds_full[k]);
}

// RD_k: dQ^T_k (thread = head dim d, 64 queries) -> shared memory [query][d]
// in two 64-dim passes through the dS_k buffer -> bulk tensor reduce-add.
__device__ __forceinline__ void rd_pp(const PpCtx& c, const FaBwdArgs& a, const PpItem& t, int it, uint32_t g, int k,
                                      PpState& st) {
  PpBarriers& bar = g_pb;
  const int q0 = (t.q_first + it) * kT + k * kH;
  const uint32_t d = c.quad * 32 + c.lane;  // TMEM lane = head dim
  const uint32_t nb = 1 + (c.warp >> 2);
  const bool leader = (c.warp & 3u) == 0 && c.lane == 0;
  mbar_wait(&bar.dq_full[k], g & 1);
  tc_fence_after();
  pp_ready(st);
  uint32_t v[kH];
  tmem_ld32(c.lane_off + col_s(k), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
  tmem_ld32(c.lane_off + col_s(k) + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
  tmem_ld_wait();
  tc_fence_before();
  warp_arrive(&bar.q_free[k]);  // S^T_k(g+1) may overwrite the columns
  float* stage = reinterpret_cast<float*>(c.ds + k * kDsBytes);  // [64 queries][64 dims] fp32
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {  // head dims 64h .. 64h + 63 live on warps 2h, 2h + 1
    if (h == 1) {
      if (leader) bulk_wait_read();  // pass 0's reduction has read the buffer
      named_bar_sync(nb, 128);
    }
    if ((d >> 6) == static_cast<uint32_t>(h)) {
      const uint32_t dd = d & 63u;
#pragma unroll
      for (int q = 0; q < kH; ++q) stage[q * 64 + dd] = __uint_as_float(v[q]);
    }
    fence_proxy_async_shared();
    named_bar_sync(nb, 128);
    if (leader) {
      tma_reduce_add_3d(&a.tm_dq64, stage, 64 * h, q0, t.bh);
      bulk_commit();
    }
  }
  if (leader) {
    bulk_wait_read();
    mbar_arrive(&bar.ds_free[k]);
  }
}

// dK (scaled) and dV of the work item: TMEM (row = key) -> bf16 -> global
__device__ __forceinline__ void kv_epilogue_pp(const PpCtx& c, const FaBwdArgs& a, const PpItem& t) {
  PpBarriers& bar = g_pb;
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

#ifndef TWFA_BWD_FIXED
#define TWFA_BWD_FIXED 1
#endif
enum PpRole { kPpLight = 0, kPpReduce = 1, kPpExbDs = 2 };

template <int kRole, int kKind = -1, bool kTrace = true>
__device__ __forceinline__ void pp_exec(const TwfaPlanOp op, const int r, const PpCtx& c, const PpItem& t,
                                        PpState& st, const TwfaDevicePlan& plan, const FaBwdArgs& a) {
  PpBarriers& bar = g_pb;
  const int kind = kKind >= 0 ? kKind : static_cast<int>(op.kind);  // kKind: known at the call site
  if (kind == TWFA_OP_LDQ || kind == TWFA_OP_LDO) {
    if constexpr (kRole == kPpLight) {
      const bool is_q = kind == TWFA_OP_LDQ;
      const int target = min(t.N - 1, r - static_cast<int>(op.stage) + (is_q ? plan.k_prefetch : plan.v_prefetch));
      const int before = is_q ? st.q_next : st.o_next;
      pp_top_up(c, a, t, st, plan, is_q, target);
      if (kTrace && a.trace != nullptr)
        for (int lit = before; lit < (is_q ? st.q_next : st.o_next); ++lit) {
          uint32_t* e = pp_trace(a, c, st, op.node, lit, r, t);
          if (e) e[4] = e[5] = e[3];
        }
    }
    return;
  }
  const int it = r - static_cast<int>(op.stage);
  if (it < 0 || it >= t.N) return;
  const uint32_t g = t.gbase + static_cast<uint32_t>(it);
  const int k = op.tile;
  struct TraceDone {
    uint32_t* e;
    __device__ ~TraceDone() {
      if (e) e[5] = static_cast<uint32_t>(clock64());
    }
  } trace_done_{kTrace && a.trace != nullptr ? pp_trace(a, c, st, op.node, it, r, t) : nullptr};
  st.rec = trace_done_.e;
  if (kind == TWFA_OP_EXB || kind == TWFA_OP_DS) {
    if constexpr (kRole == kPpExbDs)
      if (kind == TWFA_OP_EXB) exb_ds(c, a, t, it, g, k, st);  // DS_k fused (lowering guarantees)
    return;
  }
  if (kind == TWFA_OP_RD) {
    if constexpr (kRole == kPpReduce) rd_pp(c, a, t, it, g, k, st);
    return;
  }
  if constexpr (kRole != kPpLight) return;
  // tensor-core ops: warp-uniform descriptors, one elected lane issues
  const uint32_t qs = g % plan.k_depth, os = g % plan.v_depth;
  const bool release = op.flags & TWFA_OPF_RELEASE;
  uint8_t* const qk = c.q + qs * kTile + k * kSubRows;  // Q_k rows of the tile (both head-dim halves + kHalf)
  uint8_t* const ok = c.o + os * kTile + k * kSubRows;
  if (kind == TWFA_OP_ST || kind == TWFA_OP_DP) {
    const bool is_s = kind == TWFA_OP_ST;
    if (it == 0) mbar_wait(&bar.kv_full, t.icount & 1);
    if (is_s) {
      // S^T_k(g) overwrites dQ^T_k(g-1), which RD_k(g-1) must have read out
      if (g > 0 && st.q_seen == g + 1)
        mbar_wait(&bar.q_free[k], (g - 1) & 1);
      else if (g > 0)
        mbar_wait_all(&bar.q_full[qs], (g / plan.k_depth) & 1, &bar.q_free[k], (g - 1) & 1);
      else
        mbar_wait(&bar.q_full[qs], (g / plan.k_depth) & 1);
      st.q_seen = g + 1;
    } else {
      if (st.o_seen != g + 1) mbar_wait(&bar.o_full[os], (g / plan.v_depth) & 1);
      st.o_seen = g + 1;
    }
    tc_fence_after();
    if (kTrace) pp_ready(st);
    const uint32_t ad = sd_lo(is_s ? c.k : c.v, 16), bd = sd_lo(is_s ? qk : ok, 16);
    const uint32_t d_t = is_s ? col_s(k) : col_p(k);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * kHalf + (kk & 3) * 32) / 16;
        mma_ss(d_t, sdesc_join(ad + off, kSdHi), sdesc_join(bd + off, kSdHi), kIdescN64, kk > 0);
      }
      mma_commit(is_s ? &bar.s_full[k] : &bar.dp_full[k]);
      if (release) mma_commit(is_s ? &bar.q_empty[qs] : &bar.o_empty[os]);
    }
    __syncwarp();
  } else if (kind == TWFA_OP_DV || kind == TWFA_OP_DK) {
    const bool dv = kind == TWFA_OP_DV;
    bool& started = dv ? st.dv_started : st.dk_started;
    // the accumulator is overwritten by the item's first MMA: the previous
    // work item's dK / dV must have been read out
    if (!started && t.icount > 0) mbar_wait(&bar.acc_free, (t.icount - 1) & 1);
    uint32_t& seen = dv ? st.o_seen : st.q_seen;
    uint64_t* tile_full = dv ? &bar.o_full[os] : &bar.q_full[qs];
    const uint32_t tile_ph = dv ? (g / plan.v_depth) & 1 : (g / plan.k_depth) & 1;
    if (seen == g + 1)
      mbar_wait(dv ? &bar.p_full[k] : &bar.ds_full[k], g & 1);
    else
      mbar_wait_all(dv ? &bar.p_full[k] : &bar.ds_full[k], g & 1, tile_full, tile_ph);
    seen = g + 1;
    tc_fence_after();
    if (kTrace) pp_ready(st);
    // B = dO_k / Q_k as [K = query][N = d], MN-major (the two 64-dim halves kHalf apart)
    const uint32_t bd = sd_lo(dv ? ok : qk, kHalf);
    const uint32_t a_t = dv ? col_s(k) : col_p(k), d_t = dv ? kColDV : kColDK;
    const uint32_t first = started ? 1u : 0u;
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)  // 16 queries per K-step: 8 packed bf16 columns of P^T_k / dS^T_k
        mma_ts(d_t, a_t + kk * 8, sdesc_join(bd + kk * 2048 / 16, kSdHi), kIdescTS, (first || kk > 0) ? 1u : 0u);
      if (release) mma_commit(dv ? &bar.o_empty[os] : &bar.q_empty[qs]);
    }
    __syncwarp();
    started = true;
  } else if (kind == TWFA_OP_DQ) {
    mbar_wait(&bar.ds_full[k], g & 1);
    tc_fence_after();
    if (kTrace) pp_ready(st);
    // A = K^T as [M = d][K = key] (MN-major: the two 64-dim halves kHalf
    // apart), B = dS^T_k as [K = key][N = query] (MN-major, one 64-query atom)
    const uint32_t ad = sd_lo(c.k, kHalf), bd = sd_lo(c.ds + k * kDsBytes, kHalf);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(col_s(k), sdesc_join(ad + kk * 2048 / 16, kSdHi), sdesc_join(bd + kk * 2048 / 16, kSdHi), kIdescDQ,
               kk > 0);
      mma_commit(&bar.dq_full[k]);
    }
    __syncwarp();
  }
}

template <int kRole, bool kSpec, bool kTrace>
__device__ __forceinline__ void pp_run(const PpCtx& c, const TwfaDevicePlan& plan, const FaBwdArgs& a, int rd_k) {
  PpBarriers& bar = g_pb;
  const int plen = plan.prog_len[c.warp];
  const bool is_load = c.warp == static_cast<uint32_t>(plan.load_warp);
  const bool is_mma = c.warp == static_cast<uint32_t>(plan.mma_warp);
  PpState st{0, 0, 0, nullptr, false, false, 0, 0};
  constexpr int kFixed[12] = {TWFA_OP_ST, TWFA_OP_LDQ, TWFA_OP_ST, TWFA_OP_DP, TWFA_OP_LDO, TWFA_OP_DP,
                              TWFA_OP_DV, TWFA_OP_DQ, TWFA_OP_DV, TWFA_OP_DQ, TWFA_OP_DK, TWFA_OP_DK};
  bool fixed = false;
  TwfaPlanOp fx[12];
  if constexpr (kRole == kPpLight) {
    fixed = kSpec && plen == 12 && is_load && is_mma;
    for (int j = 0; j < 12 && fixed; ++j) {
      fx[j] = plan.ops[plan.prog[c.warp][j]];
      fixed = fx[j].kind == kFixed[j];
    }
  }
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
    const PpItem t = pp_item(c, a, work, gbase, icount);
    if constexpr (kRole == kPpLight) {
      if (is_load) {  // K and V of the work item
        mbar_wait(&bar.kv_empty, (icount & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&bar.kv_full, 2 * kTile);
          tma_load_3d(c.k, &a.tm_k, &bar.kv_full, 0, t.kv0, t.bh, c.pol);
          tma_load_3d(c.k + kHalf, &a.tm_k, &bar.kv_full, 64, t.kv0, t.bh, c.pol);
          tma_load_3d(c.v, &a.tm_v, &bar.kv_full, 0, t.kv0, t.bh, c.pol);
          tma_load_3d(c.v + kHalf, &a.tm_v, &bar.kv_full, 64, t.kv0, t.bh, c.pol);
        }
        __syncwarp();
      }
    }
    st.q_next = st.o_next = 0;
    st.dv_started = st.dk_started = false;
    const int trips = t.N + plan.max_stage;
    if (fixed) {
      // the committed TMA / MMA program, each op compiled for its kind
      // (TWFA_BWD_FIXED, as in fa_bwd_sm100.cu)
      for (int rr = -1; rr < trips; ++rr) {
        pp_exec<kRole, TWFA_OP_ST, kTrace>(fx[0], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_LDQ, kTrace>(fx[1], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_ST, kTrace>(fx[2], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DP, kTrace>(fx[3], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_LDO, kTrace>(fx[4], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DP, kTrace>(fx[5], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DV, kTrace>(fx[6], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DQ, kTrace>(fx[7], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DV, kTrace>(fx[8], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DQ, kTrace>(fx[9], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DK, kTrace>(fx[10], rr, c, t, st, plan, a);
        pp_exec<kRole, TWFA_OP_DK, kTrace>(fx[11], rr, c, t, st, plan, a);
      }
    } else if (kSpec && kRole == kPpLight && is_mma) {
      __trap();  // the host launches the specialized kernel only for the fixed program
    } else
    for (int rr = -1; rr < trips; ++rr)
      for (int j = 0; j < plen; ++j) pp_exec<kRole, -1, kTrace>(plan.ops[plan.prog[c.warp][j]], rr, c, t, st, plan, a);
    if constexpr (kRole == kPpLight) {
      if (is_mma) {  // every MMA of the item issued: dK, dV final; K, V free
        if (elect_one()) {
          mma_commit(&bar.acc_full);
          mma_commit(&bar.kv_empty);
        }
        __syncwarp();
      }
    } else if constexpr (kRole == kPpReduce) {
      if (rd_k == 0) kv_epilogue_pp(c, a, t);
    }
    gbase += static_cast<uint32_t>(t.N);
  }
}

template <bool kSpec, bool kTrace>  // the committed 12-op TMA / MMA program in its own instantiation; kTrace: issue trace compiled in
__global__ void __launch_bounds__(TWFA_MAX_WARPS * 32, 1)
    fa_bwd_pp_kernel(const __grid_constant__ TwfaDevicePlan plan, const __grid_constant__ FaBwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  PpCtx c;
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
  PpBarriers& bar = g_pb;
  if (threadIdx.x == 0) {
    mbar_init(&bar.kv_full, 1);
    mbar_init(&bar.kv_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar.q_full[s], 1);
      mbar_init(&bar.q_empty[s], 1);
      mbar_init(&bar.o_full[s], 1);
      mbar_init(&bar.o_empty[s], 1);
      mbar_init(&bar.s_full[s], 1);
      mbar_init(&bar.dp_full[s], 1);
      mbar_init(&bar.dq_full[s], 1);
      mbar_init(&bar.p_full[s], 4);
      mbar_init(&bar.ds_full[s], 4);
      mbar_init(&bar.q_free[s], 4);
      mbar_init(&bar.ds_free[s], 1);
    }
    mbar_init(&bar.acc_full, 1);
    mbar_init(&bar.acc_free, 4);
    fence_mbar_init();
  }
  if (c.warp == static_cast<uint32_t>(plan.load_warp) && c.lane == 0) {
    tma_prefetch_desc(&a.tm_q);
    tma_prefetch_desc(&a.tm_k);
    tma_prefetch_desc(&a.tm_v);
    tma_prefetch_desc(&a.tm_do);
    tma_prefetch_desc(&a.tm_dq64);
  }
  if (c.warp == 0) tmem_alloc<512>(&bar.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (bar.tmem_base != 0) __trap();  // one CTA per SM owns all 512 columns from 0
  c.pol = policy_evict_last();
  const int wg = static_cast<int>(c.warp >> 2) * 4;
  // registers (2 x 184 + 96 + 48 = 512 per thread slot, the 64 K register
  // file): an EXB / DS warpgroup carries the 64-float P^T row, the dP^T row
  // and the packed dS; RD a 64-float dQ^T row; the TMA / MMA warps few
  if (wg == plan.sm_warp[0] || wg == plan.sm_warp[1]) {
    setmaxnreg_inc<184>();
    pp_run<kPpExbDs, kSpec, kTrace>(c, plan, a, -1);
  } else if (wg == plan.cr_warp[0] || wg == plan.cr_warp[1]) {
    setmaxnreg_dec<96>();
    pp_run<kPpReduce, kSpec, kTrace>(c, plan, a, wg == plan.cr_warp[0] ? 0 : 1);
  } else {
    setmaxnreg_dec<48>();
    pp_run<kPpLight, kSpec, kTrace>(c, plan, a, -1);
  }
  if (c.lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (c.warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(0);
  }
}

}  // namespace

size_t fa_bwd_pp_smem_bytes(const TwfaDevicePlan& plan) {
  return static_cast<size_t>(2 + plan.k_depth + plan.v_depth) * kTile + 2 * kDsBytes + 1024;
}

// host mirror of the device-side condition of the fixed 12-op program
static bool pp_fixed_program(const TwfaDevicePlan& plan) {
  static const int kinds[12] = {TWFA_OP_ST, TWFA_OP_LDQ, TWFA_OP_ST, TWFA_OP_DP, TWFA_OP_LDO, TWFA_OP_DP,
                                TWFA_OP_DV, TWFA_OP_DQ, TWFA_OP_DV, TWFA_OP_DQ, TWFA_OP_DK, TWFA_OP_DK};
  const int w = plan.mma_warp;
  if (w != plan.load_warp || w < 0 || w >= TWFA_MAX_WARPS || plan.prog_len[w] != 12) return false;
  for (int j = 0; j < 12; ++j)
    if (plan.ops[plan.prog[w][j]].kind != kinds[j]) return false;
  return true;
}

cudaError_t fa_bwd_pp_main_launch(const TwfaDevicePlan& plan, const FaBwdArgs& args, int grid, cudaStream_t stream) {
  const size_t smem = fa_bwd_pp_smem_bytes(plan);
  const bool spec = TWFA_BWD_FIXED && pp_fixed_program(plan);
  const bool tr = args.trace != nullptr;
  const void* kern = spec ? (tr ? reinterpret_cast<const void*>(&fa_bwd_pp_kernel<true, true>)
                                : reinterpret_cast<const void*>(&fa_bwd_pp_kernel<true, false>))
                          : (tr ? reinterpret_cast<const void*>(&fa_bwd_pp_kernel<false, true>)
                                : reinterpret_cast<const void*>(&fa_bwd_pp_kernel<false, false>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (spec && tr)
    fa_bwd_pp_kernel<true, true><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
  else if (spec)
    fa_bwd_pp_kernel<true, false><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
  else if (tr)
    fa_bwd_pp_kernel<false, true><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
  else
    fa_bwd_pp_kernel<false, false><<<grid, TWFA_MAX_WARPS * 32, smem, stream>>>(plan, args);
  return cudaGetLastError();
}

}  // namespace twfa
