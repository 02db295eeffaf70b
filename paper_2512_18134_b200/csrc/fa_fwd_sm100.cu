// FA-forward on sm_100a: launch dispatch and the runtime interpreter.
// The kernel bodies are in fa_fwd_kernel.cuh; every build-time specialized
// schedule is instantiated in its own generated translation unit
// (gen/fa_spec_<id>.cu, twfa-gen) and reached through gen/fa_spec_launch.h.
#include "fa_fwd_kernel.cuh"
#include <gen/fa_spec_launch.h>

namespace twfa {

bool fa_fwd_pair_capable(const TwfaDevicePlan& plan) {
  return plan.kv_tile == 128 && !plan.s_split && plan.num_tiles == 2;
}

size_t fa_fwd_smem_bytes(const TwfaDevicePlan& plan, bool pair) {
  // dynamic part only: tile buffers (+ alignment slack); FaShared is static.
  // A CTA of a pair stages half of every K / V tile.
  const size_t kv_bytes = static_cast<size_t>(plan.kv_tile) * kHeadDim * 2 / (pair ? 2 : 1);
  // + 16 KiB epilogue staging (one 128 x 64 bf16 SW128 half-tile)
  return 1024 + static_cast<size_t>(plan.num_tiles) * kTileBytes + (plan.k_depth + plan.v_depth) * kv_bytes + 16384;
}

const char* fa_fwd_kernel_name(const TwfaDevicePlan& plan) {
#define TWFA_NAME(id) \
  if (same_plan(plan, gen::PlanOf<id>::value)) return gen::PlanOf<id>::name;
  TWFA_SPECIALIZED_PLANS(TWFA_NAME)
#undef TWFA_NAME
  return "interpreter";
}

cudaError_t fa_fwd_launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          const TwfaDevicePlan& plan, const FaArgs& args, int grid, cudaStream_t stream,
                          bool allow_specialized, bool pair) {
  if (pair && (!fa_fwd_pair_capable(plan) || grid % 2 != 0)) return cudaErrorInvalidValue;
  const size_t smem = fa_fwd_smem_bytes(plan, pair);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;  // deep rings need the CTA-pair realization
  const int threads = plan.num_warps * 32;
  const bool trace = args.trace != nullptr;
  if (allow_specialized) {
#define TWFA_LAUNCH(id) \
  if (same_plan(plan, gen::PlanOf<id>::value)) \
    return gen::launch_spec_##id(tq, tk, tv, args, smem, grid, threads, stream, trace, pair);
    TWFA_SPECIALIZED_PLANS(TWFA_LAUNCH)
#undef TWFA_LAUNCH
  }
  if (plan.kv_tile == 64)
    return trace ? launch(fa_fwd_interp<64, true, false>, smem, grid, threads, stream, 1, tq, tk, tv, plan, args)
                 : launch(fa_fwd_interp<64, false, false>, smem, grid, threads, stream, 1, tq, tk, tv, plan, args);
  if (pair)
    return trace ? launch(fa_fwd_interp<128, true, true>, smem, grid, threads, stream, 2, tq, tk, tv, plan, args)
                 : launch(fa_fwd_interp<128, false, true>, smem, grid, threads, stream, 2, tq, tk, tv, plan, args);
  return trace ? launch(fa_fwd_interp<128, true, false>, smem, grid, threads, stream, 1, tq, tk, tv, plan, args)
               : launch(fa_fwd_interp<128, false, false>, smem, grid, threads, stream, 1, tq, tk, tv, plan, args);
}

}  // namespace twfa
