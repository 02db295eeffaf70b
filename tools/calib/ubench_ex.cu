// Microbenchmark of the softmax ops of fa_fwd_sm100.cu in isolation:
// MX (load 128-col S row from TMEM + row max) and EX (exp2 + bf16 pack +
// TMEM store) for one 128x128 tile per warpgroup, with 1 or 2 warpgroups
// (2 = both Q sub-tiles concurrently, sharing the four MUFUs).
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2512_18134_b200/csrc/sm100.cuh"
using namespace twfa;
#ifndef POLY_EVERY
#define POLY_EVERY 1000
#endif
constexpr int kPolyEvery = POLY_EVERY;

__device__ __forceinline__ void load_row(uint32_t taddr, uint32_t (&s)[128]) {
  tmem_ld32(taddr + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
  tmem_ld32(taddr + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
  tmem_ld32(taddr + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
  tmem_ld_wait();
}
__device__ __forceinline__ float row_max(const uint32_t (&s)[128]) {
  float a[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int i = 0; i < 128; i += 8) {
    a[(i >> 3) & 3] = fmaxf(a[(i >> 3) & 3], fmaxf(fmaxf(__uint_as_float(s[i]), __uint_as_float(s[i + 1])),
                                                   fmaxf(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]))));
    a[(i >> 3) & 3] = fmaxf(a[(i >> 3) & 3], fmaxf(fmaxf(__uint_as_float(s[i + 4]), __uint_as_float(s[i + 5])),
                                                   fmaxf(__uint_as_float(s[i + 6]), __uint_as_float(s[i + 7]))));
  }
  return fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
}
__device__ __forceinline__ float exp_store_row(const uint32_t (&s)[128], uint32_t taddr, float sl, float m) {
  const float2 sl2 = make_float2(sl, sl), nm2 = make_float2(-m, -m);
  float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(s[c * 32 + i]), __uint_as_float(s[c * 32 + i + 1])), sl2, nm2);
      float2 p;
      if (((i >> 1) % kPolyEvery) == kPolyEvery - 1) { p.x = poly_exp2(x.x); p.y = poly_exp2(x.y); }
      else { p.x = fast_exp2(x.x); p.y = fast_exp2(x.y); }
      acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], p);
      pk[i >> 1] = pack_bf16(p.x, p.y);
    }
    tmem_st16(taddr + c * 16, pk);
  }
  tmem_st_wait();
  return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
}

__global__ void __launch_bounds__(256, 1) k(long long* cyc, float* out, int nwg) {
  __shared__ uint32_t base;
  const uint32_t warp = threadIdx.x >> 5, wg = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t taddr = base + (((warp & 3) * 32u) << 16) + wg * 128;
  // fill S with scores
  uint32_t init[32];
  for (int i = 0; i < 32; ++i) init[i] = __float_as_uint(0.01f * (i + threadIdx.x % 7));
  for (int c = 0; c < 4; ++c) tmem_st32(taddr + c * 32, init);
  tmem_st_wait();
  __syncthreads();
  float acc = 0;
  long long t_mx = 0, t_ex = 0;
  if (nwg == 3 && wg == 1) {  // interference: the other tile's MX (TMEM row loads + max) in a loop
    for (int it = 0; it < 200; ++it) {
      uint32_t s[128];
      load_row(taddr, s);
      acc += row_max(s);
    }
  } else if (wg < (uint32_t)(nwg == 3 ? 1 : nwg)) {
    for (int it = 0; it < 64; ++it) {
      long long c0 = clock64();
      uint32_t s[128];
      load_row(taddr, s);
      float m = row_max(s) * 0.127f;
      long long c1 = clock64();
      acc += exp_store_row(s, taddr, 0.127f, m);
      long long c2 = clock64();
      // restore S (P overwrote the first 64 columns)
      for (int c = 0; c < 2; ++c) tmem_st32(taddr + c * 32, init);
      tmem_st_wait();
      if (it >= 4) { t_mx += c1 - c0; t_ex += c2 - c1; }
    }
  }
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) { cyc[0] = t_mx / 60; cyc[1] = t_ex / 60; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(base); }
}

int main() {
  long long* cyc; float* out;
  cudaMalloc(&cyc, 64); cudaMalloc(&out, 4096 * 4);
  for (int nwg : {1, 2, 3}) {
    long long h[2];
    k<<<1, 256>>>(cyc, out, nwg); k<<<1, 256>>>(cyc, out, nwg);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("poly_every=%d warpgroups=%d: MX (ld row + max) %lld cycles, EX (exp+pack+st) %lld cycles\n", kPolyEvery, nwg, h[0], h[1]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
