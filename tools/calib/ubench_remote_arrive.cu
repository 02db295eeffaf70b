// Cost to the issuing warp of an mbarrier arrive on the peer CTA's barrier
// (shared::cluster, release.cta / release.cluster) against a local arrive, in
// a cluster of two CTAs. One warp per CTA; CTA 1's warp arrives N times on a
// barrier (count 1, so every arrive completes a phase), CTA 0 idles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ubench_remote_arrive.cu -o ubench_remote_arrive
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) k(long long* out, int n) {
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t target = rank ^ (MODE == 0 ? 1u : 0u);  // MODE 0/1: remote, MODE 2: local
  if (MODE == 2) target = rank;
  uint32_t addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(&bar)), "r"(target));
  long long t0 = clock64();
  if (rank == 1 && threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      if (MODE == 1)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
      else
        asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
    }
  }
  long long t1 = clock64();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 1 && threadIdx.x == 0) out[MODE] = (t1 - t0) / n;
}

int main() {
  long long* d;
  cudaMalloc(&d, 4 * sizeof(long long));
  long long h[4] = {0, 0, 0, 0};
  const int n = 1024;
  k<0><<<2, 32>>>(d, n);
  k<1><<<2, 32>>>(d, n);
  k<2><<<2, 32>>>(d, n);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("clk per arrive (back to back, %d): remote release.cta %lld, remote release.cluster %lld, local %lld (%s)\n", n,
         h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
