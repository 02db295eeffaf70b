// GEMM mainloop on sm_100a under the Twill schedule of the GEMM loop graph
// (BASELINE config 2; graph LDA, LDB -> MMA with a loop-carried accumulator).
// The solver's answer (I = 1, LDA/LDB streamed on the variable-latency warp,
// MMA on its own warp, ring depth = streaming depth) fixes the roles:
//   warp plan.load_warp  TMA producer: A [128 x 64] + B [128 x 64] per k-block
//                        and CTA (each CTA of the pair loads its own halves)
//   warp plan.mma_warp   single-thread tcgen05.mma.cta_group::2 256x256x16
//                        (leader CTA only), TMEM accumulator in both CTAs
//   4 extra warps        epilogue: tcgen05.ld -> bf16 -> swizzled shared
//                        memory -> TMA bulk tensor store (outside the loop graph)
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 output tile: each
// SM's tensor core reads 128 rows of A and 128 rows of B from its own shared
// memory per k-block (64 B/clk at full rate instead of the 96 B/clk of a
// single-CTA 128 x 256 tile) and the pair reads 64 KiB from L2 per 2 x 128 x
// 256 outputs instead of 96 KiB. Two TMEM accumulators (2 x 256 columns) let
// the epilogue of one output tile overlap the mainloop of the next.
// Persistent grid over pair tiles in groups of `group_m` tile rows, so the A
// panel of a group stays L2-resident while B streams.
//   C[M, N] = A[M, K] * B[N, K]^T, bf16 in, fp32 accumulate, bf16 out.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fa_fwd.h"
#include "sm100.cuh"

namespace twfa {
namespace {

constexpr int kBM = 128, kBN = 128, kBK = 64;  // per CTA: 128 rows of A, 128 rows (N half) of B
constexpr int kPairM = 2 * kBM, kPairN = 2 * kBN;  // output tile of the pair
constexpr uint32_t kABytes = kBM * kBK * 2;        // 16 KiB
constexpr uint32_t kBBytes = kBN * kBK * 2;        // 16 KiB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kMaxStages = 6;
constexpr uint32_t kEpiBox = 64;                        // output columns per TMA store box (128 B rows, SW128)
constexpr uint32_t kEpiBytes = kBM * kEpiBox * 2;        // 16 KiB staging per box
constexpr uint32_t kIdesc = idesc_bf16_f32(kPairM, kPairN, 0);

struct __align__(8) GemmBarriers {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_m, int& tm, int& tn) {
  const int per_group = group_m * tiles_n;
  const int group = t / per_group;
  const int first_m = group * group_m;
  const int gm = min(group_m, tiles_m - first_m);
  const int local = t % per_group;
  tm = first_m + local % gm;
  tn = local / gm;
  // odd groups sweep N backwards, so the B columns of the last wave of a
  // group are the first the next group reads (still in L2)
  if (group & 1) tn = tiles_n - 1 - tn;
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ TwfaDevicePlan plan,
                const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = plan.k_depth;
  uint8_t* epi = smem + stages * kStageBytes;  // 2 x 16 KiB output staging
  GemmBarriers* bar = reinterpret_cast<GemmBarriers*>(epi + 2 * kEpiBytes);
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t first_epi = static_cast<uint32_t>(plan.num_warps);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&bar->full[s], 1);   // leader: one expect_tx arrival for both CTAs' bytes
      mbar_init(&bar->empty[s], 1);  // one multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bar->acc_full[a], 1);
      mbar_init(&bar->acc_empty[a], 8);  // the 4 epilogue warps of both CTAs (leader's copy)
    }
    fence_mbar_init();
  }
  if (warp == static_cast<uint32_t>(plan.load_warp) && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_c);
  }
  if (warp == static_cast<uint32_t>(plan.mma_warp)) tmem_alloc_pair<512>(&bar->tmem_base);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, tensor memory allocated in both
  tc_fence_after();
  const uint32_t tmem = bar->tmem_base;

  const int tiles_m = args.M / kPairM, tiles_n = args.N / kPairN;
  const int num_tiles = tiles_m * tiles_n;
  const int kblocks = args.K / kBK;
  const int pair = static_cast<int>(blockIdx.x >> 1), num_pairs = static_cast<int>(gridDim.x >> 1);
  const int group_m = args.group_m > 0 ? args.group_m : 8;

  if (warp == static_cast<uint32_t>(plan.load_warp)) {
    // LDA, LDB: streamed loads into this CTA's ring (depth = streaming
    // depth). Both CTAs wait for their own slot to drain (the multicast
    // commit), then load their halves; the leader's full barrier counts both.
    // L2 policies (TWFA_GEMM_POL): 0 normal / normal, 1 A evict_last / B
    // evict_first, 2 last / last (default: 1.07 GB DRAM reads per 8192^3
    // launch against 2.2 GB for 1 and 3; profiles/r02b_gemm_policy.txt),
    // 3 normal / first, 4 last / normal
    const int pm = args.pol_mode;
    const uint64_t pol_a = (pm == 1 || pm == 2 || pm == 4) ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_b = pm == 2 ? policy_evict_last() : (pm == 1 || pm == 3) ? policy_evict_first()
                                                                                 : policy_evict_normal();
    // ring slot and phase advanced incrementally (no division per k-block)
    uint32_t s = 0, ph = 0;
    for (int t = pair; t < num_tiles; t += num_pairs) {
      int tm, tn;
      tile_coords(t, tiles_m, tiles_n, group_m, tm, tn);
      const int row_a = tm * kPairM + static_cast<int>(rank) * kBM;
      const int row_b = tn * kPairN + static_cast<int>(rank) * kBN;
      for (int kb = 0; kb < kblocks; ++kb, s = s + 1 == static_cast<uint32_t>(stages) ? (ph ^= 1u, 0u) : s + 1) {
        mbar_wait_cluster(&bar->empty[s], ph ^ 1);
        uint8_t* sa = smem + s * kStageBytes;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&bar->full[s], 2 * kStageBytes);
          tma_load_2d_pair(sa, &tm_a, &bar->full[s], kb * kBK, row_a, pol_a);
          tma_load_2d_pair(sa + kABytes, &tm_b, &bar->full[s], kb * kBK, row_b, pol_b);
        }
        __syncwarp();
      }
    }
  } else if (warp == static_cast<uint32_t>(plan.mma_warp)) {
    if (leader) {
      // MMA: D += A B^T, one 256x256x16 pair instruction per 16-wide k slice.
      // Every lane waits and computes the (uniform) descriptors; one elected
      // lane issues, so the operands stay in uniform registers.
      uint32_t s = 0, ph = 0, lt = 0;
      for (int t = pair; t < num_tiles; t += num_pairs, ++lt) {
        const uint32_t acc = lt & 1, acc_ph = (lt >> 1) & 1;
        mbar_wait_cluster(&bar->acc_empty[acc], acc_ph ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < kblocks; ++kb, s = s + 1 == static_cast<uint32_t>(stages) ? (ph ^= 1u, 0u) : s + 1) {
          mbar_wait_cluster(&bar->full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          // descriptors as base + 16-byte offset (see sdesc_lo)
          const uint32_t da = sdesc_lo(sa, 16), db = sdesc_lo(sa + kABytes, 16);
          constexpr uint32_t hi = sdesc_hi(1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              mma_ss_pair(tmem + acc * kPairN, sdesc_join(da + kk * 2, hi), sdesc_join(db + kk * 2, hi), kIdesc,
                          (kb | kk) != 0);
            mma_commit_pair(&bar->empty[s], 0x3);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit_pair(&bar->acc_full[acc], 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= first_epi && warp < first_epi + 4) {
    // epilogue: this CTA's 128 rows of the pair tile, four 128 x 64 boxes,
    // each through a swizzled staging buffer (double-buffered) and one bulk
    // tensor store
    const uint32_t quad = warp & 3u;
    const uint32_t lane_off = (quad * 32u) << 16;
    const uint32_t r = quad * 32 + lane;  // row inside the CTA's 128
    const bool store_thread = warp == first_epi && lane == 0;
    uint32_t lt = 0, box = 0;
    for (int t = pair; t < num_tiles; t += num_pairs, ++lt) {
      int tm, tn;
      tile_coords(t, tiles_m, tiles_n, group_m, tm, tn);
      const uint32_t acc = lt & 1, acc_ph = (lt >> 1) & 1;
      mbar_wait_cluster(&bar->acc_full[acc], acc_ph);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t c = 0; c < kPairN / kEpiBox; ++c, ++box) {
        uint32_t v[64];
        tmem_ld32(tmem + lane_off + acc * kPairN + c * kEpiBox, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld32(tmem + lane_off + acc * kPairN + c * kEpiBox + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_ld_wait();
        if (c == kPairN / kEpiBox - 1) {  // the accumulator is in registers: the next tile may overwrite it
          tc_fence_before();
          warp_arrive_cluster(&bar->acc_empty[acc], 0);
        }
        uint8_t* buf = epi + (box & 1) * kEpiBytes;
        const uint32_t rbase = smem_u32(buf) + r * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)  // 16-byte chunk ch of the row, SW128: chunk ^ (row % 8)
          st_shared_v4(rbase + ((ch ^ (r & 7)) << 4), pack_bf16(__uint_as_float(v[8 * ch + 0]), __uint_as_float(v[8 * ch + 1])),
                       pack_bf16(__uint_as_float(v[8 * ch + 2]), __uint_as_float(v[8 * ch + 3])),
                       pack_bf16(__uint_as_float(v[8 * ch + 4]), __uint_as_float(v[8 * ch + 5])),
                       pack_bf16(__uint_as_float(v[8 * ch + 6]), __uint_as_float(v[8 * ch + 7])));
        fence_proxy_async_shared();
        named_bar_sync(1, 128);
        if (store_thread) {
          tma_store_2d(&tm_c, buf, tn * kPairN + c * kEpiBox, tm * kPairM + static_cast<int>(rank) * kBM);
          bulk_commit();
          bulk_wait_read_1();  // the other staging buffer is free again
        }
        named_bar_sync(1, 128);
      }
    }
    if (store_thread) bulk_wait_all();
  }

  tc_fence_before();
  cluster_sync();  // neither CTA leaves while the pair's MMAs may still touch its memory
  if (warp == static_cast<uint32_t>(plan.mma_warp)) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

size_t gemm_smem_bytes(const TwfaDevicePlan& plan) {
  return 1024 + static_cast<size_t>(plan.k_depth) * kStageBytes + 2 * kEpiBytes + sizeof(GemmBarriers);
}

cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                        const TwfaDevicePlan& plan, const GemmArgs& args, int grid, cudaStream_t stream) {
  const size_t smem = gemm_smem_bytes(plan);
  cudaError_t e =
      cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  gemm_kernel<<<grid, (plan.num_warps + 4) * 32, smem, stream>>>(ta, tb, tc, plan, args);
  return cudaGetLastError();
}

}  // namespace twfa
