// mbarrier handoff latency between warps (ping-pong), the per-edge cost of
// every cross-warp dependence the realized schedule synchronizes.
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;
__global__ void k(long long* out, int mode, int spinners) {
  __shared__ uint64_t b[3];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&b[0], mode ? 1 : 1); mbar_init(&b[1], 1); mbar_init(&b[2], 1); fence_mbar_init(); }
  __syncthreads();
  const int n = 1000;
  long long t0 = clock64();
  if (w == 0) {
    for (int i = 0; i < n; ++i) {
      if (lane == 0) mbar_arrive(&b[0]);
      if (lane == 0) mbar_wait(&b[1], i & 1);
      __syncwarp();
    }
  } else if (w == 1) {
    for (int i = 0; i < n; ++i) {
      if (lane == 0) mbar_wait(&b[0], i & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&b[1]);
    }
  } else if (w - 2 < spinners) {
    // warps spinning on a barrier that never completes until the end
    if (lane == 0) while (!mbar_try_wait(&b[2], 0)) { if (clock64() - t0 > 3000000) break; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}
int main() {
  long long* o; cudaMalloc(&o, 64); long long h;
  for (int sp : {0, 2, 6, 14}) {
    k<<<1, 512>>>(o, 0, sp); k<<<1, 512>>>(o, 0, sp);
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("mbarrier ping-pong round trip: %lld cycles (%d other warps spinning)\n", h, sp);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
