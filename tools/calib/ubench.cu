// Cost-model calibration microbenchmarks for the Blackwell FA loop graph
// (SURVEY s8f rank 1): throughput of the softmax building blocks on one SM,
// reported in SM cycles per warp-instruction / per 128x128 tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

#include "../../paper_2512_18134_b200/csrc/sm100.cuh"

using namespace twfa;

constexpr int kIters = 4096;

// each thread: 8 independent chains of op(x) -> x
template <int kOp>
__global__ void k_pipe(float* out, long long* cycles, int active_warps) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  if ((threadIdx.x >> 5) < active_warps) {
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (kOp == 0) x[i] = fast_exp2(x[i]);                       // MUFU.EX2
        if (kOp == 1) x[i] = poly_exp2(x[i]) - 1.0f;                // FMA-pipe exp2
        if (kOp == 2) { acc += pack_bf16(x[i], x[(i + 1) & 7]); x[i] = x[i] * 0.999f; }  // F2FP (+FMUL)
        if (kOp == 3) x[i] = fmaf(x[i], 0.999f, -0.0001f);          // FFMA
        if (kOp == 4) x[i] = x[i] * 0.999f;                          // FMUL
        if (kOp == 5) x[i] = fmaxf(x[i], x[(i + 3) & 7] * 0.5f);     // FMNMX + FMUL
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// TMEM: 32x32b.x32 load (+wait) and x32 store throughput for 4 warps (one per quadrant)
__global__ void k_tmem(long long* cycles, float* out) {
  __shared__ uint32_t base;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = base + (((warp & 3) * 32u) << 16);
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = i;
  float s = 0;
  long long c0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
    tmem_st32(t + (it & 3) * 32, v);
  }
  tmem_st_wait();
  long long c1 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it) {
    tmem_ld32(t + (it & 3) * 32, v);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) s += __uint_as_float(v[i]);
  }
  long long c2 = clock64();
#pragma unroll 1
  for (int it = 0; it < 64; ++it) {  // 4 loads in flight, one wait (128 columns)
    uint32_t a[32], b[32];
    tmem_ld32(t, a);
    tmem_ld32(t + 32, b);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) s = fmaxf(s, fmaxf(__uint_as_float(a[i]), __uint_as_float(b[i])));
    tmem_ld32(t + 64, a);
    tmem_ld32(t + 96, b);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) s = fmaxf(s, fmaxf(__uint_as_float(a[i]), __uint_as_float(b[i])));
  }
  long long c3 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) {
    cycles[0] = c1 - c0;
    cycles[1] = c2 - c1;
    cycles[2] = c3 - c2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}

__global__ void k_tmem_lat(long long* cycles, float* out) {
  __shared__ uint32_t base;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t v[32];
  float s = 0;
  long long c0 = clock64();
  if (warp == 0) {
#pragma unroll 1
    for (int it = 0; it < 256; ++it) {
      tmem_ld32(base + (it & 3) * 32, v);
      tmem_ld_wait();
      s += __uint_as_float(v[0]) + __uint_as_float(v[31]);
    }
  }
  long long c1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[0] = c1 - c0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  const char* names[] = {"MUFU.EX2 (ex2.approx)", "poly_exp2 (FMA pipe)", "F2FP bf16x2 pack (+FMUL)", "FFMA", "FMUL",
                         "FMNMX+FMUL"};
  for (int op = 0; op < 6; ++op) {
    for (int warps : {4, 8, 16}) {
      long long h = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: k_pipe<0><<<1, 512>>>(out, cyc, warps); break;
          case 1: k_pipe<1><<<1, 512>>>(out, cyc, warps); break;
          case 2: k_pipe<2><<<1, 512>>>(out, cyc, warps); break;
          case 3: k_pipe<3><<<1, 512>>>(out, cyc, warps); break;
          case 4: k_pipe<4><<<1, 512>>>(out, cyc, warps); break;
          case 5: k_pipe<5><<<1, 512>>>(out, cyc, warps); break;
        }
        cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      }
      const double warp_instr_per_smsp = double(kIters) * 8 * warps / 4;
      printf("%-28s warps/SM=%2d  %.2f cycles per warp-op per SMSP  (%.1f lanes/clk/SM)\n", names[op], warps,
             double(h) / warp_instr_per_smsp, 32.0 * 4 / (double(h) / warp_instr_per_smsp));
    }
  }
  k_tmem<<<1, 128>>>(cyc, out);
  long long t[3];
  cudaMemcpy(t, cyc, sizeof(t), cudaMemcpyDeviceToHost);
  printf("TMEM st32 (4 warps, 4 KiB per warp-op): %.1f cycles/op -> %.0f B/clk/SM\n", t[0] / 256.0,
         4.0 * 4096 * 256 / t[0]);
  printf("TMEM ld32+wait serialized: %.1f cycles/op -> %.0f B/clk/SM\n", t[1] / 256.0, 4.0 * 4096 * 256 / t[1]);
  printf("TMEM 2x ld32 per wait, 128 cols: %.1f cycles per 128-col row block -> %.0f B/clk/SM\n", t[2] / 64.0,
         4.0 * 16384 * 64 / t[2]);
  k_tmem_lat<<<1, 128>>>(cyc, out);
  cudaMemcpy(t, cyc, sizeof(t[0]), cudaMemcpyDeviceToHost);
  printf("TMEM ld32+wait single warp latency: %.1f cycles\n", t[0] / 256.0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
