// Cross-warp mbarrier handoff latency on B200, in SM clocks and in ns
// (%globaltimer), under the load the FA-forward kernel puts on an SM: the
// per-edge cost of every cross-warp dependence of the realized schedule.
//
// Warp 0 and warp 1 ping-pong n times over two mbarriers; each side waits
// with `mode`: 0 = mbarrier.try_wait spin (the kernel's mbar_wait),
// 1 = mbarrier.test_wait spin, 2 = try_wait with a 1 us suspend hint.
// `load` warps (2..) run the softmax-like background at the same time:
// tcgen05.ld of 32 columns + ex2 over them, in a loop.
// Prints round-trip cycles, ns and the implied SM clock.
#include <cstdint>
#include <cstdio>

#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t parity, int mode) {
  if (mode == 0) {
    while (!mbar_try_wait(bar, parity)) {
    }
  } else if (mode == 1) {
    while (!test_wait(bar, parity)) {
    }
  } else {
    while (!mbar_try_wait_hint(bar, parity, 1000)) {
    }
  }
}

__global__ void __launch_bounds__(512, 1) k(long long* out, int mode, int load, int n) {
  __shared__ uint64_t b[3];
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&b[0], 1);
    mbar_init(&b[1], 1);
    stop = 0;
    fence_mbar_init();
  }
  if (w == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long c0 = 0, c1 = 0;
  uint64_t g0 = 0, g1 = 0;
  if (w == 0) {
    c0 = clock64();
    g0 = gtimer();
    for (int i = 0; i < n; ++i) {
      if (lane == 0) mbar_arrive(&b[0]);
      wait_mode(&b[1], i & 1, mode);
      __syncwarp();
    }
    c1 = clock64();
    g1 = gtimer();
    stop = 1;
  } else if (w == 1) {
    for (int i = 0; i < n; ++i) {
      wait_mode(&b[0], i & 1, mode);
      __syncwarp();
      if (lane == 0) mbar_arrive(&b[1]);
    }
  } else if (w >= 4 && w - 4 < load) {
    // background: TMEM row reads of this warp's lane quadrant + MUFU ex2
    const uint32_t quad = (w & 3) * 32;
    float acc = 0.f;
    while (!stop) {
      uint32_t r[32];
      tmem_ld32(((quad) << 16) + (w & 3) * 128, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += fast_exp2(__uint_as_float(r[j]) * 1e-3f - 1.f);
    }
    if (acc == 1234.5f) out[7] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) {
    tc_fence_after();
    tmem_dealloc<512>(0);
  }
  if (threadIdx.x == 0) {
    out[0] = (c1 - c0) / n;
    out[1] = static_cast<long long>((g1 - g0) * 1000 / n);  // ps per round trip
    out[2] = (c1 - c0) * 1000 / static_cast<long long>(g1 - g0 > 0 ? g1 - g0 : 1);  // MHz
  }
}

int main() {
  long long* o;
  cudaMalloc(&o, 64);
  long long h[3];
  const char* names[] = {"try_wait spin", "test_wait spin", "try_wait 1us hint"};
  for (int load : {0, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {  // a warm-up launch, then the measured one
        k<<<148, 512>>>(o, mode, load, 20000);
        cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      }
      printf("%-18s load warps %d: round trip %lld clk = %.1f ns (SM %lld MHz) -> one handoff %.0f clk\n",
             names[mode], load, h[0], h[1] / 1000.0, h[2], h[0] / 2.0);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
