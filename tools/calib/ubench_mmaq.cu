// tcgen05.mma issue queue depth: one elected thread issues a chain of
// M=128 N=128 K=16 bf16 MMAs back to back and records the clock after each
// issue. Issue returns immediately while the queue has room; once it is full
// each issue waits for one MMA to retire (~64 clk). Prints per-issue deltas.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;
constexpr int kN = 48;
template <int kMode>  // 0: SS K-major, 1: TS (A in TMEM) B MN-major, 2: SS A and B MN-major
__global__ void __launch_bounds__(128, 1) k_mmaq(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t done;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint32_t a = sdesc_lo(smem_u32(smem), 16), b = sdesc_lo(smem_u32(smem) + 32768, 16);
    constexpr uint32_t hi = sdesc_hi(1024);
    uint32_t t[kN + 1];
    if (elect_one()) {
      t[0] = static_cast<uint32_t>(clock64());
#pragma unroll
      for (int i = 0; i < kN; ++i) {
        if constexpr (kMode == 1)  // A (bf16) from tensor memory columns 256.., like PV of the FA kernel
          mma_ts(0, 256 + (i & 7) * 8, sdesc_join(b + (i & 3) * 128, hi), idesc_bf16_f32(128, 128, 1), i > 0);
        else if constexpr (kMode == 2)  // like DQ of the backward: A and B MN-major (LBO = 16 KiB halves)
          mma_ss(0, sdesc_join(sdesc_lo(smem_u32(smem) + (i & 3) * 2048, 16384), hi),
                 sdesc_join(sdesc_lo(smem_u32(smem) + 32768 + (i & 3) * 2048, 16384), hi),
                 idesc_bf16_f32(128, 128, 1) | (1u << 15), i > 0);
        else
          mma_ss(0, sdesc_join(a + (i & 3) * 2, hi), sdesc_join(b + (i & 3) * 2, hi), idesc_bf16_f32(128, 128, 0), i > 0);
        t[i + 1] = static_cast<uint32_t>(clock64());
      }
      mma_commit(&done);
      for (int i = 0; i <= kN; ++i) out[i] = t[i] - t[0];
    }
    __syncwarp();
    mbar_wait(&done, 0);
    if (threadIdx.x == 32) out[kN + 1] = static_cast<uint32_t>(clock64()) - t[0];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tbase); }
}
template <int kTS>
int run(const char* name) {
  uint32_t* d; cudaMalloc(&d, 4 * (kN + 2));
  cudaFuncSetAttribute(k_mmaq<kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 3; ++rep) k_mmaq<kTS><<<1, 128, 65536>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[kN + 2]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s: issue clock after MMA i (M128 N128 K16, 64 clk each at full rate):\n", name);
  for (int i = 1; i <= kN; ++i) printf("%d:%u%s", i, h[i], i % 8 ? " " : "\n");
  printf("all complete: %u clk\n", h[kN + 1]);
  cudaFree(d);
  return 0;
}
int main() { return run<0>("SS") | run<1>("TS (A in TMEM)") | run<2>("SS, A and B MN-major"); }
