// Per-op cost of the MMA-issuing warp when it issues a chain of tensor-core
// ops back to back, each op = 8 M=128 N=128 K=16 bf16 MMAs (512 clk of
// tensor-core work) + a commit, the way the FA kernels' MMA warp does:
//   mode 0: MMAs + commit only
//   mode 1: + an mbarrier wait on an already-completed phase before each op
//   mode 2: + tcgen05.fence::after_thread_sync before each op
//   mode 3: 1 + 2 (the kernels' per-op prologue)
//   mode 4: 3 + a global store (a trace stamp) per op
//   mode 5: 3 + a second commit per op (ring-slot release)
// Reported: clocks for kOps ops and the overhead per op over 512 clk.
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;
constexpr int kOps = 32;

__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t done, ready, rel, fin;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    mbar_init(&ready, 1);
    mbar_init(&rel, 1);
    mbar_init(&fin, 1);
    fence_mbar_init();
    mbar_arrive(&ready);  // phase 0 complete before anyone waits
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // modes 12-14: mode 11 with a warp on the MMA warp's sub-partition (warp 5)
  // streaming 12 = MUFU ex2, 13 = tcgen05.ld 32x32b.x32, 14 = st.shared.v4
  if (warp == 5 && mode >= 12) {
    float x = threadIdx.x * 1e-3f;
    uint32_t acc = 0;
    for (int it = 0; it < 4000; ++it) {
      if (mode == 12) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fast_exp2(x) * 0.5f;
      } else if (mode == 13) {
        uint32_t v[32];
        tmem_ld32(((1u * 32u) << 16) + 256u + (it & 3) * 32u, v);  // lanes 32-63 (sub-partition 1)
        tmem_ld_wait();
        acc += v[0] + v[31];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(smem_u32(smem) + 49152 + ((threadIdx.x & 31) * 16 + j * 512) % 16384, it, j, acc, 0);
      }
    }
    if (x == 12345.f || acc == 12345u) out[60] = acc;
  }
  if (warp == 1) {
    constexpr uint32_t hi = sdesc_hi(1024);
    const uint32_t t0 = static_cast<uint32_t>(clock64());
    if (mode >= 10) {
      // one elected lane runs the whole op loop: no per-op elect / __syncwarp
      if (elect_one()) {
        for (int op = 0; op < kOps; ++op) {
          if (mode >= 11) mbar_wait(&ready, 0);
          if (mode >= 11) tc_fence_after();
          const uint32_t a = sdesc_lo(smem_u32(smem) + (op & 1) * 16384, 16), b = sdesc_lo(smem_u32(smem) + 32768, 16);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            mma_ss((op & 1) * 128u, sdesc_join(a + (i & 3) * 2, hi), sdesc_join(b + (i & 3) * 2, hi),
                   idesc_bf16_f32(128, 128, 0), i > 0);
          mma_commit(&done);
          if (op == kOps - 1) mma_commit(&fin);
        }
      }
      __syncwarp();
    }
    for (int op = 0; op < (mode >= 10 ? 0 : kOps); ++op) {
      if (mode == 1 || mode >= 3) mbar_wait(&ready, 0);
      if (mode >= 2) tc_fence_after();
      if (mode == 4 && threadIdx.x == 32) out[8 + op] = static_cast<uint32_t>(clock64());
      const uint32_t a = sdesc_lo(smem_u32(smem) + (op & 1) * 16384, 16), b = sdesc_lo(smem_u32(smem) + 32768, 16);
      if (elect_one()) {
        // modes 6-9 isolate the commit and the accumulator switch:
        // 6 = same D, commit per op; 7 = alternating D, no per-op commit;
        // 8 = same D, accumulate throughout, no per-op commit; 9 = 7 but accumulate=0 only on op 0
        const uint32_t dcol = (mode == 6 || mode == 8) ? 0u : (op & 1) * 128u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          mma_ss(dcol, sdesc_join(a + (i & 3) * 2, hi), sdesc_join(b + (i & 3) * 2, hi), idesc_bf16_f32(128, 128, 0),
                 (mode == 8 || mode == 9) ? (op > 0 || i > 0) : i > 0);
        if (mode != 7 && mode != 8 && mode != 9) mma_commit(&done);
        if (mode == 5) mma_commit(&rel);
        if (op == kOps - 1) mma_commit(&fin);
      }
      __syncwarp();
    }
    const uint32_t t1 = static_cast<uint32_t>(clock64());
    mbar_wait(&fin, 0);
    const uint32_t t2 = static_cast<uint32_t>(clock64());
    if (threadIdx.x == 32) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4 * 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* name[] = {"MMAs + commit", "+ wait (completed)", "+ tcgen05 fence", "+ wait + fence",
                        "+ wait + fence + STG", "+ wait + fence + 2nd commit", "same D, commit per op",
                        "alternating D, no commit", "same D accumulating, no commit", "alt D, acc, no commit",
                        "one lane loops, commit per op", "one lane loops + wait + fence",
                        "11 + MUFU warp on its SMSP", "11 + tcgen05.ld warp on its SMSP", "11 + STS.128 warp on its SMSP"};
  for (int m = 0; m < 15; ++m) {
    uint32_t h[2];
    for (int rep = 0; rep < 3; ++rep) k<<<1, 256, 65536>>>(d, m);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-30s %d ops: issued in %6u clk, complete at %6u clk = %5.0f clk/op (512 of tensor-core work)\n",
           name[m], kOps, h[0], h[1], h[1] / static_cast<double>(kOps));
  }
  return 0;
}
