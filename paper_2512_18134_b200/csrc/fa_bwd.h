// Launch interface of the sm_100a FA-backward kernel (internal to libtwfa).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "plan.h"

namespace twfa {

struct FaBwdArgs {
  // bf16 [B*H][S][128] maps with 64 x 128 SW128 boxes (Q, K, V, dO) and the
  // fp32 dQ accumulator map with 32 x 128 SW128 boxes (TMA reduce-add)
  alignas(64) CUtensorMap tm_q;
  alignas(64) CUtensorMap tm_k;
  alignas(64) CUtensorMap tm_v;
  alignas(64) CUtensorMap tm_do;
  alignas(64) CUtensorMap tm_dq;
  // the fp32 dQ accumulator with 64 x 64 unswizzled boxes (the two-sub-tile
  // kernel's reduce-add of a 64-query x 64-dim staging block)
  alignas(64) CUtensorMap tm_dq64;
  const float* lse;   // [B, H, S] natural-log sum-exp of the forward
  float* dvec;        // [B, H, S] workspace: rowsum(dO * O)
  float* dq_acc;      // [B, H, S, 128] workspace: fp32 dQ accumulator
  __nv_bfloat16* dk;  // [B, H, S, 128]
  __nv_bfloat16* dv;
  int B, H, S;
  int causal;
  float scale;        // softmax scale
  float scale_log2;   // scale * log2(e)
  // optional per-CTA work lists (causal): CTA x runs work_list[work_off[x]
  // .. work_off[x + 1]) in order; nullptr = round-robin over the CTAs
  const int* work_list;
  const int* work_off;
  // optional issue trace of CTA 0 (twfa_fa_bwd_traced): per warp, word 0 =
  // record count, then 8-word records {node, iteration, trip, t_issue, 0,
  // t_done, work item ordinal, iterations of that item}
  uint32_t* trace;
  uint32_t trace_cap;
};

size_t fa_bwd_smem_bytes(const TwfaDevicePlan& plan);
size_t fa_bwd_workspace_bytes(int B, int H, int S);
// pre-pass (D), zeroing of the accumulator, the main kernel, post-pass (dQ)
// (num_tiles == 2 plans run the two-sub-tile kernel, fa_bwd_pp_sm100.cu)
cudaError_t fa_bwd_launch(const TwfaDevicePlan& plan, const FaBwdArgs& args, const __nv_bfloat16* o,
                          const __nv_bfloat16* dout, __nv_bfloat16* dq, int grid, cudaStream_t stream);
size_t fa_bwd_pp_smem_bytes(const TwfaDevicePlan& plan);
cudaError_t fa_bwd_pp_main_launch(const TwfaDevicePlan& plan, const FaBwdArgs& args, int grid, cudaStream_t stream);

}  // namespace twfa
