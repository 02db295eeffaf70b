// Softmax of one 128 x 128 S tile (row max, exp2, bf16 pack, TMEM store of
// P, row sum) done by one warpgroup (4 warps, 128 columns per thread, the
// production layout) or by two warpgroups that split the columns (8 warps:
// two per SMSP / TMEM lane quadrant, 64 columns per thread, partial row
// maxima exchanged through shared memory on a 64-thread named barrier).
// Clocks per tile, one CTA, the tile alone on the SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ubench_split.cu -o ubench_split
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;

template <int N>
__device__ __forceinline__ float rmax(const uint32_t (&s)[N]) {
  float a[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int i = 0; i < N; i += 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = fmaxf(a[j], __uint_as_float(s[i + j]));
  }
  return fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
}

// exps of N columns starting at s[0], P stored at TMEM column pcol (N/2 packed)
template <int N>
__device__ __forceinline__ float exps(uint32_t (&s)[N], uint32_t pcol, float sl, float m) {
  const float2 sl2 = make_float2(sl, sl), nm2 = make_float2(-m, -m);
#pragma unroll
  for (int c = 0; c < N / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const int e = c * 32 + i;
      const float2 x = ffma2(make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), sl2, nm2);
      float2 p;
      p.x = fast_exp2(x.x);
      p.y = fast_exp2(x.y);
      s[e] = __float_as_uint(p.x);
      s[e + 1] = __float_as_uint(p.y);
      pk[i >> 1] = pack_bf16(p.x, p.y);
    }
    tmem_st16(pcol + c * 16, pk);
  }
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int e = 0; e < N; e += 4) {
    acc[0] = fadd2(acc[0], make_float2(__uint_as_float(s[e]), __uint_as_float(s[e + 1])));
    acc[1] = fadd2(acc[1], make_float2(__uint_as_float(s[e + 2]), __uint_as_float(s[e + 3])));
  }
  tmem_st_wait();
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

__shared__ float g_pmax[2][128];

template <int MODE>  // 0: one warpgroup, 128 columns; 1: two warpgroups, 64 columns each
__global__ void __launch_bounds__(256, 1) k(long long* cyc, float* out, int tiles) {
  __shared__ uint32_t base;
  const uint32_t warp = threadIdx.x >> 5, quad = warp & 3, half = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_off = (quad * 32u) << 16;
  const uint32_t row = quad * 32 + (threadIdx.x & 31);
  uint32_t init[32];
  for (int i = 0; i < 32; ++i) init[i] = __float_as_uint(0.01f * (i + threadIdx.x % 7));
  if (half == 0)
    for (int c = 0; c < 4; ++c) tmem_st32(base + lane_off + c * 32, init);
  tmem_st_wait();
  __syncthreads();
  float acc = 0.f;
  long long t = 0;
  const bool active = MODE == 1 || half == 0;
  for (int it = 0; it < tiles; ++it) {
    __syncthreads();
    const long long c0 = clock64();
    if (active) {
      if constexpr (MODE == 0) {
        uint32_t s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(base + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
        tmem_ld_wait();
        const float m = rmax<128>(s) * 0.127f;
        acc += exps<128>(s, base + lane_off, 0.127f, m);
      } else {
        uint32_t s[64];
        const uint32_t col = half * 64;
        tmem_ld32(base + lane_off + col, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld32(base + lane_off + col + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld_wait();
        g_pmax[half][row] = rmax<64>(s);
        named_bar_sync(1 + quad, 64);  // the two warps of this lane quadrant
        const float m = fmaxf(g_pmax[0][row], g_pmax[1][row]) * 0.127f;
        acc += exps<64>(s, base + lane_off + half * 32, 0.127f, m);
      }
    }
    __syncthreads();
    if (it >= 4) t += clock64() - c0;
    // restore S (P overwrote the first 64 columns)
    if (half == 0)
      for (int c = 0; c < 2; ++c) tmem_st32(base + lane_off + c * 32, init);
    tmem_st_wait();
  }
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[MODE] = t / (tiles - 4);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}

int main() {
  long long* cyc;
  float* out;
  cudaMalloc(&cyc, 64);
  cudaMalloc(&out, 4096 * 4);
  long long h[2];
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 256>>>(cyc, out, 68);
    k<1><<<1, 256>>>(cyc, out, 68);
  }
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("softmax of one 128x128 tile: one warpgroup %lld clk, two warpgroups (column halves) %lld clk (%s)\n", h[0],
         h[1], cudaGetErrorString(cudaDeviceSynchronize()));
}
