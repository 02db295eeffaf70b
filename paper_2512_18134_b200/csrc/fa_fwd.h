// Launch interfaces of the sm_100a kernels (internal to libtwfa).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "plan.h"

namespace twfa {

struct FaArgs {
  // O as a TMA map (d, S, B*H), 64x128 boxes, SWIZZLE_128B: the epilogue
  // stages each 128x64 half-tile in shared memory and stores it with one
  // bulk tensor copy (kernel parameter space keeps the 64-byte alignment)
  alignas(64) CUtensorMap tm_o;
  __nv_bfloat16* o;    // [B, H, S, 128]
  float* lse;          // [B, H, S] natural log-sum-exp, or nullptr
  uint32_t* trace;     // per-warp issue records of CTA 0 (debug), or nullptr
  uint32_t trace_cap;  // records per warp (entry 0 of each warp = count)
  int B, H, S;
  int causal;
  float scale_log2;    // softmax_scale * log2(e)
  // optional per-unit work lists (causal): unit x (a CTA, or a CTA pair)
  // runs work_list[work_off[x] .. work_off[x + 1]) in order; nullptr = the
  // arithmetic round order
  const int* work_list;
  const int* work_off;
};

// CTA-pair realization (cta_group::2, clusters of 2): 128-key K/V tiles,
// unsplit S, two Q sub-tiles per CTA
bool fa_fwd_pair_capable(const TwfaDevicePlan& plan);
size_t fa_fwd_smem_bytes(const TwfaDevicePlan& plan, bool pair);
// Runs the build-time specialized kernel of `plan` when one was generated
// (gen/fa_plans.inc) and allow_specialized is set, else the interpreter;
// `pair`: as CTA pairs (grid even, work lists indexed by pair).
cudaError_t fa_fwd_launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          const TwfaDevicePlan& plan, const FaArgs& args, int grid, cudaStream_t stream,
                          bool allow_specialized, bool pair);
// "specialized:<name>" or "interpreter"
const char* fa_fwd_kernel_name(const TwfaDevicePlan& plan);

struct GemmArgs {
  __nv_bfloat16* c;  // [M, N] row-major (written through the tm_c tensor map)
  int M, N, K;
  int group_m;       // raster: pair-tile rows per group (A panel kept in L2); <= 0: default
  int pol_mode;      // L2 cache policies of the A / B loads (gemm_sm100.cu)
};

size_t gemm_smem_bytes(const TwfaDevicePlan& plan);
cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                        const TwfaDevicePlan& plan, const GemmArgs& args, int grid, cudaStream_t stream);

}  // namespace twfa
