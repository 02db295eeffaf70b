// Do MUFU.EX2 and F2FP (bf16x2 pack) share an issue pipe? Time per warp of
// N iterations of {2 ex2}, {1 f2fp}, {2 ex2 + 1 f2fp}, {2 ex2 + poly pair}
// with 4 / 16 warps per SM. Overlapping pipes: mixed ~= max; shared: ~= sum.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;
template <int MODE>
__global__ void k(float* out, int n, long long* cyc) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a - 0.25f, d = a + 0.125f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    if (MODE == 0 || MODE == 2 || MODE == 3) {
      a = fast_exp2(a) - 1.f;
      b = fast_exp2(b) - 1.f;
    }
    if (MODE == 1 || MODE == 2) acc ^= pack_bf16(c, d), c += 1e-7f, d -= 1e-7f;
    if (MODE == 3) {
      float2 p = poly_exp2x2(make_float2(c, d));
      c = p.x - 1.f;
      d = p.y - 1.f;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + acc;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMallocManaged(&cyc, 148 * 8);
  const int n = 4096;
  const char* names[] = {"2x MUFU.EX2", "1x F2FP", "2x EX2 + 1x F2FP", "2x EX2 + poly pair"};
  for (int warps : {4, 8, 16}) for (int m = 0; m < 4; ++m) {
    auto fn = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
    fn<<<148, warps * 32>>>(out, n, cyc); cudaDeviceSynchronize();
    fn<<<148, warps * 32>>>(out, n, cyc); cudaDeviceSynchronize();
    printf("warps/SM=%2d %-22s %.2f cycles/iter/warp-per-SMSP\n", warps, names[m], (double)cyc[0] / n / (warps / 4));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
