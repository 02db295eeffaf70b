// twfa-gen: schedule -> compile-time kernel specialization.
//
// The paper compiled the synthesized listing into CUDA by hand
// (PAPER.md:894-899). This tool automates that step: it lowers each
// (problem JSON, solution JSON) pair exactly as twfa_plan_create does
// (lowering.cpp) and emits the resulting TwfaDevicePlan as a C++ constant.
// fa_fwd_sm100.cu instantiates one kernel per constant, with every warp's trip
// program, ring depth and flag known at compile time (no op dispatch, no ring
// division at run time). At launch, a plan equal to a generated one runs its
// specialized kernel; any other plan runs the runtime interpreter. Both realize
// the same schedule through the same op bodies.
//
// usage: twfa-gen <out.inc> <name> <problem.json> <solution.json> [<name> <problem> <solution> ...]
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "lowering.h"

namespace {

std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot read " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

std::string ints(const int32_t* v, int n) {
  std::string s = "{";
  for (int i = 0; i < n; ++i) s += (i ? ", " : "") + std::to_string(v[i]);
  return s + "}";
}

std::string bytes(const uint8_t* v, int n) {
  std::string s = "{";
  for (int i = 0; i < n; ++i) s += (i ? ", " : "") + std::to_string(static_cast<int>(v[i]));
  return s + "}";
}

std::string emit(int id, const std::string& name, const twfa::LoweredSchedule& s, const std::string& src) {
  const TwfaDevicePlan& p = s.plan;
  std::ostringstream o;
  o << "// " << src << ": I=" << s.ii << " L=" << s.length << "\n";
  o << "template <>\nstruct PlanOf<" << id << "> {\n  static constexpr const char* name = \"" << name
    << "\";\n  static constexpr TwfaDevicePlan value = {\n";
  o << "    .family = " << p.family << ", .ii = " << p.ii << ", .length = " << p.length << ", .copies = " << p.copies
    << ", .max_stage = " << p.max_stage << ", .num_nodes = " << p.num_nodes << ",\n";
  o << "    .num_warps = " << p.num_warps << ", .num_tiles = " << p.num_tiles << ", .k_depth = " << p.k_depth
    << ", .v_depth = " << p.v_depth << ", .load_warp = " << p.load_warp << ",\n";
  o << "    .k_prefetch = " << p.k_prefetch << ", .v_prefetch = " << p.v_prefetch << ", .s_depth = " << p.s_depth
    << ", .kv_tile = " << p.kv_tile << ", .s_split = " << p.s_split
    << ", .cr_warp = " << ints(p.cr_warp, TWFA_MAX_TILES) << ", .sm_warp = " << ints(p.sm_warp, TWFA_MAX_TILES)
    << ", .mma_warp = " << p.mma_warp << ",\n";
  o << "    .heavy_wg_mask = " << p.heavy_wg_mask << ", .q_warp = " << p.q_warp << ", .ex_ring_len = " << p.ex_ring_len
    << ", .ex_ring = " << bytes(p.ex_ring, TWFA_MAX_TILES) << ",\n";
  o << "    .ops = {\n";
  for (int v = 0; v < TWFA_MAX_NODES; ++v) {
    const TwfaPlanOp& op = p.ops[v];
    o << "        {" << int(op.node) << ", " << int(op.kind) << ", " << int(op.tile) << ", " << int(op.stage) << ", "
      << int(op.slot) << ", " << int(op.warp_start) << ", " << int(op.warp_count) << ", " << int(op.order) << ", "
      << int(op.flags) << ", {0, 0, 0, 0, 0, 0, 0}},";
    if (v < p.num_nodes) o << "  // " << s.nodes[static_cast<size_t>(v)].id;
    o << "\n";
  }
  o << "    },\n    .prog = {\n";
  for (int w = 0; w < TWFA_MAX_WARPS; ++w) {
    o << "        " << bytes(p.prog[w], TWFA_MAX_NODES) << ",";
    if (p.prog_len[w]) {
      o << "  // warp " << w << ":";
      for (int i = 0; i < p.prog_len[w]; ++i) o << " " << s.nodes[p.prog[w][i]].id;
    }
    o << "\n";
  }
  o << "    },\n    .prog_len = " << bytes(p.prog_len, TWFA_MAX_WARPS) << ",\n  };\n";
  // role[w]: the first warp with w's trip program and register class. Warps
  // of one role share one instantiation of the role's code (instruction
  // cache: a specialized copy per warp would not fit).
  int role[TWFA_MAX_WARPS];
  for (int w = 0; w < TWFA_MAX_WARPS; ++w) {
    role[w] = w;
    for (int u = 0; u < w; ++u) {
      const bool same_class = ((p.heavy_wg_mask >> (u / 4)) & 1) == ((p.heavy_wg_mask >> (w / 4)) & 1) &&
                              (u == p.load_warp) == (w == p.load_warp);
      bool same = same_class && p.prog_len[u] == p.prog_len[w];
      for (int i = 0; same && i < p.prog_len[w]; ++i) same = p.prog[u][i] == p.prog[w][i];
      if (same) {
        role[w] = u;
        break;
      }
    }
  }
  o << "  static constexpr int role[" << TWFA_MAX_WARPS << "] = " << ints(role, TWFA_MAX_WARPS) << ";\n};\n\n";
  return o.str();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5 || (argc - 2) % 3 != 0) {
    std::fprintf(stderr, "usage: twfa-gen <out.inc> <name> <problem.json> <solution.json> [...]\n");
    return 2;
  }
  std::string body, list;
  std::vector<bool> pair_capable;  // 128-key K/V tiles, unsplit S, two Q sub-tiles (fa_fwd_pair_capable)
  int id = 0;
  try {
    for (int i = 2; i + 2 < argc; i += 3) {
      const std::string name = argv[i];
      const twfa::LoweredSchedule s = twfa::lower(slurp(argv[i + 1]), slurp(argv[i + 2]));
      if (s.plan.family != TWFA_FAMILY_FA_FWD) continue;  // the GEMM kernel has a single fixed role layout
      body += emit(id, name, s, std::string(argv[i + 2]).substr(std::string(argv[i + 2]).rfind('/') + 1));
      pair_capable.push_back(s.plan.kv_tile == 128 && !s.plan.s_split && s.plan.num_tiles == 2);
      list += " X(" + std::to_string(id++) + ")";
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  // one translation unit per specialization (compiled in parallel) and the
  // declarations of their launchers
  const std::string inc_path = argv[1];
  const std::string dir = inc_path.substr(0, inc_path.rfind('/') + 1);
  std::ofstream decl(dir + "fa_spec_launch.h");
  decl << "// GENERATED by twfa-gen: launchers of the specialized FA kernels.\n#pragma once\n"
          "#include <cuda.h>\n#include <cuda_runtime.h>\n#include <fa_fwd.h>\n\nnamespace twfa {\nnamespace gen {\n";
  for (int i = 0; i < id; ++i) {
    decl << "cudaError_t launch_spec_" << i
         << "(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FaArgs& args, size_t smem,\n"
            "                          int grid, int threads, cudaStream_t stream, bool trace, bool pair);\n";
    std::ofstream tu(dir + "fa_spec_" + std::to_string(i) + ".cu");
    tu << "// GENERATED by twfa-gen: kernel specialization " << i << " (gen::PlanOf<" << i << ">).\n"
          "#include <fa_fwd_kernel.cuh>\n#include <gen/fa_spec_launch.h>\n\nnamespace twfa {\nnamespace gen {\n"
          "cudaError_t launch_spec_" << i
       << "(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FaArgs& args, size_t smem,\n"
          "                          int grid, int threads, cudaStream_t stream, bool trace, bool pair) {\n";
    if (pair_capable[i])
      tu << "  if (pair)\n"
            "    return trace ? launch(fa_fwd_spec<" << i << ", true, true>, smem, grid, threads, stream, 2, tq, tk, tv, args)\n"
            "                 : launch(fa_fwd_spec<" << i << ", false, true>, smem, grid, threads, stream, 2, tq, tk, tv, args);\n";
    else
      tu << "  if (pair) return cudaErrorInvalidValue;  // no CTA-pair realization of this plan\n";
    tu << "  return trace ? launch(fa_fwd_spec<" << i << ", true, false>, smem, grid, threads, stream, 1, tq, tk, tv, args)\n"
          "               : launch(fa_fwd_spec<" << i << ", false, false>, smem, grid, threads, stream, 1, tq, tk, tv, args);\n"
          "}\n}  // namespace gen\n}  // namespace twfa\n";
  }
  decl << "}  // namespace gen\n}  // namespace twfa\n";
  std::ofstream out(argv[1]);
  out << "// GENERATED by twfa-gen (csrc/gen_main.cpp) from the committed solution JSON.\n"
         "// Do not edit: rebuilt by paper_2512_18134_b200/_build.py.\n"
         "#pragma once\n#include \"plan.h\"\n\nnamespace twfa {\nnamespace gen {\n\ntemplate <int I>\nstruct PlanOf;\n\n"
      << body << "}  // namespace gen\n}  // namespace twfa\n\n#define TWFA_SPECIALIZED_PLANS(X)" << list << "\n";
  return out ? 0 : 1;
}
