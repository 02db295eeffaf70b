// GEMM mainloop on sm_100a under the Twill schedule of the GEMM loop graph
// (BASELINE config 2; graph LDA, LDB -> MMA with a loop-carried accumulator).
// The solver's answer (I = 1, LDA/LDB streamed on the variable-latency warp,
// MMA on its own warp, ring depth = streaming depth) fixes the roles:
//   warp plan.load_warp  TMA producer: A [128 x 64] + B [256 x 64] per k-block
//   warp plan.mma_warp   single-thread tcgen05.mma 128x256x16, TMEM accumulator
//   4 extra warps        epilogue: tcgen05.ld -> bf16 -> global (outside the loop graph)
// Two TMEM accumulators (2 x 256 columns) let the epilogue of one output tile
// overlap the mainloop of the next. Persistent grid, grouped tile order for L2 reuse.
//   C[M, N] = A[M, K] * B[N, K]^T, bf16 in, fp32 accumulate, bf16 out.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fa_fwd.h"
#include "sm100.cuh"

namespace twfa {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KiB
constexpr uint32_t kBBytes = kBN * kBK * 2;  // 32 KiB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kMaxStages = 4;
constexpr int kGroupM = 16;
constexpr uint32_t kIdesc = idesc_bf16_f32(kBM, kBN, 0);

struct __align__(8) GemmBarriers {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = kGroupM * tiles_n;
  const int group = t / per_group;
  const int first_m = group * kGroupM;
  const int gm = min(kGroupM, tiles_m - first_m);
  const int local = t % per_group;
  tm = first_m + local % gm;
  tn = local / gm;
}

}  // namespace

__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const __grid_constant__ TwfaDevicePlan plan, const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = plan.k_depth;
  GemmBarriers* bar = reinterpret_cast<GemmBarriers*>(smem + stages * kStageBytes);
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t first_epi = static_cast<uint32_t>(plan.num_warps);

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&bar->full[s], 1);
      mbar_init(&bar->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bar->acc_full[a], 1);
      mbar_init(&bar->acc_empty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == static_cast<uint32_t>(plan.load_warp) && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
  }
  if (warp == first_epi) tmem_alloc<512>(&bar->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar->tmem_base;

  const int tiles_m = args.M / kBM, tiles_n = args.N / kBN;
  const int num_tiles = tiles_m * tiles_n;
  const int kblocks = args.K / kBK;

  if (warp == static_cast<uint32_t>(plan.load_warp)) {
    // LDA, LDB: streamed loads into the ring (depth = streaming depth).
    // Warp-uniform arithmetic, one elected lane issues (uniform registers).
    const uint64_t pol_a = policy_evict_last();
    const uint64_t pol_b = policy_evict_last();
    uint32_t g = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int tm, tn;
      tile_coords(t, tiles_m, tiles_n, tm, tn);
      for (int kb = 0; kb < kblocks; ++kb, ++g) {
        const uint32_t s = g % stages, ph = (g / stages) & 1;
        mbar_wait(&bar->empty[s], ph ^ 1);
        uint8_t* sa = smem + s * kStageBytes;
        if (elect_one()) {
          mbar_arrive_expect_tx(&bar->full[s], kStageBytes);
          tma_load_2d(sa, &tm_a, &bar->full[s], kb * kBK, tm * kBM, pol_a);
          tma_load_2d(sa + kABytes, &tm_b, &bar->full[s], kb * kBK, tn * kBN, pol_b);
        }
        __syncwarp();
      }
    }
  } else if (warp == static_cast<uint32_t>(plan.mma_warp)) {
    // MMA: D += A B^T, one 128x256x16 instruction per 16-wide k slice.
    // Every lane waits and computes the (uniform) descriptors; one elected
    // lane issues, so the operands stay in uniform registers.
    uint32_t g = 0, lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const uint32_t acc = lt & 1, acc_ph = (lt >> 1) & 1;
      mbar_wait(&bar->acc_empty[acc], acc_ph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb, ++g) {
        const uint32_t s = g % stages, ph = (g / stages) & 1;
        mbar_wait(&bar->full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * kStageBytes);
        // descriptors as base + 16-byte offset (the start-address field of
        // one stage cannot carry; see sdesc_lo)
        const uint32_t da = sdesc_lo(sa, 16), db = sdesc_lo(sa + kABytes, 16);
        constexpr uint32_t hi = sdesc_hi(1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_ss(tmem + acc * kBN, sdesc_join(da + kk * 2, hi), sdesc_join(db + kk * 2, hi), kIdesc,
                   (kb | kk) != 0);
          mma_commit(&bar->empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&bar->acc_full[acc]);
      __syncwarp();
    }
  } else if (warp >= first_epi && warp < first_epi + 4) {
    const uint32_t quad = warp & 3u;
    const uint32_t lane_off = (quad * 32u) << 16;
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int tm, tn;
      tile_coords(t, tiles_m, tiles_n, tm, tn);
      const uint32_t acc = lt & 1, acc_ph = (lt >> 1) & 1;
      mbar_wait(&bar->acc_full[acc], acc_ph);
      tc_fence_after();
      const int row = tm * kBM + quad * 32 + lane;
      __nv_bfloat16* crow = args.c + static_cast<int64_t>(row) * args.N + tn * kBN;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + acc * kBN + c * 32, v);
        tmem_ld_wait();
        uint4* dst = reinterpret_cast<uint4*>(crow + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(v[8 * i + 0]), __uint_as_float(v[8 * i + 1]));
          w.y = pack_bf16(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3]));
          w.z = pack_bf16(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5]));
          w.w = pack_bf16(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7]));
          dst[i] = w;
        }
      }
      tc_fence_before();
      mbar_arrive(&bar->acc_empty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == first_epi) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

size_t gemm_smem_bytes(const TwfaDevicePlan& plan) {
  return 1024 + static_cast<size_t>(plan.k_depth) * kStageBytes + sizeof(GemmBarriers);
}

cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, const TwfaDevicePlan& plan,
                        const GemmArgs& args, int grid, cudaStream_t stream) {
  const size_t smem = gemm_smem_bytes(plan);
  cudaError_t e =
      cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  gemm_kernel<<<grid, (plan.num_warps + 4) * 32, smem, stream>>>(ta, tb, plan, args);
  return cudaGetLastError();
}

}  // namespace twfa
