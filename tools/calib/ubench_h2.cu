// Throughput of the half-precision MUFU exp2 forms against ex2.approx.f32:
// ex2.approx.f16x2 and ex2.approx.ftz.bf16x2 (two results per lane).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(float* out, int n, long long* cyc) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a - 0.25f, d = a + 0.125f;
  uint32_t h0 = 0x3c003c00u ^ threadIdx.x, h1 = h0 ^ 0x1111u, h2 = h0 ^ 0x2222u, h3 = h0 ^ 0x3333u;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    if (MODE == 0) {  // 4 independent f32 ex2
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    } else if (MODE == 1) {  // 4 independent f16x2 ex2 (8 results)
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else {  // 4 independent bf16x2 ex2
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + (float)(h0 ^ h1 ^ h2 ^ h3);
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMallocManaged(&cyc, 148 * 8);
  const int n = 4096;
  const char* names[] = {"ex2.f32 x4", "ex2.f16x2 x4", "ex2.bf16x2 x4"};
  for (int warps : {4, 16}) for (int m = 0; m < 3; ++m) {
    auto fn = m == 0 ? k<0> : m == 1 ? k<1> : k<2>;
    fn<<<148, warps * 32>>>(out, n, cyc); cudaDeviceSynchronize();
    fn<<<148, warps * 32>>>(out, n, cyc); cudaDeviceSynchronize();
    double c = (double)cyc[0] / n / (warps / 4);
    printf("warps/SM=%2d %-14s %.2f cycles per 4 instr per warp-per-SMSP (%.2f per instr)\n", warps, names[m], c, c / 4);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
