// Does an mbarrier wait on the MMA-issuing warp queue behind the tcgen05.mma
// instructions that warp issued just before? One elected thread issues n
// M=128 N=128 K=16 bf16 MMAs (64 clk each at full rate) plus a commit, then
// the warp waits on a barrier whose phase ALREADY completed (arrived at
// init). Recorded: clock after the MMA issues, after the wait returns, and
// when the MMAs' commit barrier fires. If the wait returns only as the MMAs
// drain, every input wait the MMA warp does right after an MMA batch costs
// up to the batch's execution time.
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;

__global__ void __launch_bounds__(128, 1) k(uint32_t* out, int n, int what) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t done, ready, extra;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    mbar_init(&ready, 1);
    mbar_init(&extra, 1);
    fence_mbar_init();
    mbar_arrive(&ready);  // phase 0 of `ready` is complete before anyone waits
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint32_t a = sdesc_lo(smem_u32(smem), 16), b = sdesc_lo(smem_u32(smem) + 32768, 16);
    constexpr uint32_t hi = sdesc_hi(1024);
    uint32_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    t0 = static_cast<uint32_t>(clock64());
    if (elect_one()) {
      for (int i = 0; i < n; ++i)
        mma_ss(0, sdesc_join(a + (i & 3) * 2, hi), sdesc_join(b + (i & 3) * 2, hi), idesc_bf16_f32(128, 128, 0),
               i > 0);
      mma_commit(&done);
    }
    __syncwarp();
    t1 = static_cast<uint32_t>(clock64());
    if (what == 0) {
      mbar_wait(&ready, 0);  // already complete
    } else if (what == 1) {
      if (elect_one()) mbar_arrive(&extra);  // a plain shared-memory arrive
      __syncwarp();
    } else {
      uint32_t v = *reinterpret_cast<volatile uint32_t*>(smem + 4);  // a plain shared load
      if (v == 12345) out[40] = v;
    }
    t2 = static_cast<uint32_t>(clock64());
    mbar_wait(&done, 0);
    t3 = static_cast<uint32_t>(clock64());
    if (threadIdx.x == 32) {
      out[0] = t1 - t0;
      out[1] = t2 - t1;
      out[2] = t3 - t0;
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
  const char* what[] = {"try_wait on a completed barrier", "mbarrier.arrive", "ld.shared"};
  for (int w = 0; w < 3; ++w)
    for (int n : {0, 2, 4, 6, 8, 12, 16}) {
      uint32_t h[3];
      for (int rep = 0; rep < 3; ++rep) k<<<1, 128, 65536>>>(d, n, w);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%-32s after %2d MMAs: issue %5u clk, then the op %5u clk; MMAs complete at %5u clk\n", what[w], n,
             h[0], h[1], h[2]);
    }
  return 0;
}
