// Schedule -> kernel lowering. See lowering.h for the contract.
#include "lowering.h"

#include <algorithm>
#include <cstring>
#include <set>
#include <tuple>

#include "json.hpp"

namespace twfa {
namespace {

using json = nlohmann::json;

void require_keys(const json& obj, const char* what, std::initializer_list<const char*> allowed) {
  for (auto it = obj.begin(); it != obj.end(); ++it) {
    bool ok = false;
    for (const char* k : allowed) ok = ok || it.key() == k;
    if (!ok) throw DomainError(std::string(what) + " has unknown key \"" + it.key() + "\"");
  }
}

int64_t get_int(const json& obj, const char* what, const char* key, bool required, int64_t dflt) {
  auto it = obj.find(key);
  if (it == obj.end()) {
    if (required) throw DomainError(std::string(what) + " requires \"" + key + "\"");
    return dflt;
  }
  if (!it->is_number_integer()) throw DomainError(std::string(what) + " key \"" + key + "\" must be an integer");
  return it->get<int64_t>();
}

// ---- problem: parse_problem (ir.cpp:93-229), same keys, checks and messages
void parse_problem(const std::string& text, LoweredSchedule& s) {
  json root;
  try {
    root = json::parse(text);
  } catch (const json::exception& e) {
    throw DomainError(std::string("problem is not valid JSON: ") + e.what());
  }
  if (!root.is_object()) throw DomainError("problem top level must be an object");
  require_keys(root, "problem", {"machine", "graph"});
  if (!root.contains("machine") || !root.contains("graph"))
    throw DomainError("problem requires \"machine\" and \"graph\"");
  const json& mj = root["machine"];
  if (!mj.is_object()) throw DomainError("\"machine\" must be an object");
  require_keys(mj, "machine", {"units", "memories", "num_warps", "reg_limit", "vl_warp"});
  if (!mj.contains("units") || !mj["units"].is_array()) throw DomainError("machine requires a \"units\" array");
  auto get_name = [](const json& o, const char* what) {
    if (!o.contains("name") || !o["name"].is_string())
      throw DomainError(std::string(what) + " requires a string \"name\"");
    return o["name"].get<std::string>();
  };
  auto index_of = [](const std::vector<LResource>& v, const std::string& name) {
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i].name == name) return static_cast<int>(i);
    return -1;
  };
  for (const json& uj : mj["units"]) {
    if (!uj.is_object()) throw DomainError("unit entries must be objects");
    require_keys(uj, "unit", {"name", "capacity"});
    LResource u{get_name(uj, "unit"), get_int(uj, "unit", "capacity", true, 0)};
    if (u.capacity <= 0) throw DomainError("unit \"" + u.name + "\" capacity must be positive");
    if (index_of(s.units, u.name) >= 0) throw DomainError("duplicate unit \"" + u.name + "\"");
    s.units.push_back(u);
  }
  if (mj.contains("memories")) {
    if (!mj["memories"].is_array()) throw DomainError("\"memories\" must be an array");
    for (const json& memj : mj["memories"]) {
      if (!memj.is_object()) throw DomainError("memory entries must be objects");
      require_keys(memj, "memory", {"name", "capacity"});
      LResource m{get_name(memj, "memory"), get_int(memj, "memory", "capacity", true, 0)};
      if (m.capacity < 0) throw DomainError("memory \"" + m.name + "\" capacity must be >= 0");
      if (index_of(s.memories, m.name) >= 0) throw DomainError("duplicate memory \"" + m.name + "\"");
      s.memories.push_back(m);
    }
  }
  s.num_warps = static_cast<int>(get_int(mj, "machine", "num_warps", true, 1));
  if (s.num_warps <= 0) throw DomainError("num_warps must be positive");
  s.reg_limit = get_int(mj, "machine", "reg_limit", true, 0);
  if (s.reg_limit < 0) throw DomainError("reg_limit must be >= 0");
  s.vl_warp = static_cast<int>(get_int(mj, "machine", "vl_warp", true, 0));
  if (s.vl_warp < 0 || s.vl_warp >= s.num_warps) throw DomainError("vl_warp must lie in [0, num_warps)");

  const json& gj = root["graph"];
  if (!gj.is_object()) throw DomainError("\"graph\" must be an object");
  require_keys(gj, "graph", {"nodes", "edges"});
  if (!gj.contains("nodes") || !gj["nodes"].is_array()) throw DomainError("graph requires a \"nodes\" array");
  if (gj["nodes"].empty()) throw DomainError("graph has no nodes");
  std::map<std::string, int> index;
  for (const json& nj : gj["nodes"]) {
    if (!nj.is_object()) throw DomainError("node entries must be objects");
    require_keys(nj, "node", {"id", "rrt", "cycles", "regs", "footprint", "spill_cost",
                              "variable_latency", "warps_required"});
    LNode n;
    if (!nj.contains("id") || !nj["id"].is_string()) throw DomainError("node requires a string \"id\"");
    n.id = nj["id"].get<std::string>();
    if (n.id.empty()) throw DomainError("node id must be nonempty");
    if (index.count(n.id)) throw DomainError("duplicate node \"" + n.id + "\"");
    n.cycles = get_int(nj, "node", "cycles", true, 1);
    if (n.cycles < 1) throw DomainError("node \"" + n.id + "\" cycles must be >= 1");
    n.rrt.assign(s.units.size(), std::vector<int64_t>(static_cast<size_t>(n.cycles), 0));
    if (nj.contains("rrt")) {
      if (!nj["rrt"].is_object()) throw DomainError("node \"" + n.id + "\" rrt must be an object");
      for (auto it = nj["rrt"].begin(); it != nj["rrt"].end(); ++it) {
        const int f = index_of(s.units, it.key());
        if (f < 0) throw DomainError("node \"" + n.id + "\" uses undeclared unit \"" + it.key() + "\"");
        if (!it->is_array()) throw DomainError("rrt rows must be arrays");
        if (static_cast<int64_t>(it->size()) > n.cycles)
          throw DomainError("node \"" + n.id + "\" rrt row for \"" + it.key() + "\" is longer than cycles");
        for (size_t c = 0; c < it->size(); ++c) {
          const json& cell = (*it)[c];
          if (!cell.is_number_integer()) throw DomainError("rrt entries must be integers");
          const int64_t v = cell.get<int64_t>();
          if (v < 0) throw DomainError("rrt entries must be >= 0");
          n.rrt[static_cast<size_t>(f)][c] = v;
        }
      }
    }
    n.regs = get_int(nj, "node", "regs", false, 0);
    if (n.regs < 0) throw DomainError("node \"" + n.id + "\" regs must be >= 0");
    n.footprint.assign(s.memories.size(), 0);
    if (nj.contains("footprint")) {
      if (!nj["footprint"].is_object()) throw DomainError("node \"" + n.id + "\" footprint must be an object");
      for (auto it = nj["footprint"].begin(); it != nj["footprint"].end(); ++it) {
        const int mi = index_of(s.memories, it.key());
        if (mi < 0)
          throw DomainError("node \"" + n.id + "\" footprint names undeclared memory \"" + it.key() + "\"");
        if (!it->is_number_integer()) throw DomainError("footprint entries must be integers");
        const int64_t v = it->get<int64_t>();
        if (v < 0) throw DomainError("footprint entries must be >= 0");
        n.footprint[static_cast<size_t>(mi)] = v;
      }
    }
    n.spill_cost = get_int(nj, "node", "spill_cost", false, 0);
    if (n.spill_cost < 0) throw DomainError("spill_cost must be >= 0");
    if (nj.contains("variable_latency")) {
      if (!nj["variable_latency"].is_boolean()) throw DomainError("variable_latency must be a boolean");
      n.variable_latency = nj["variable_latency"].get<bool>();
    }
    n.warps_required = static_cast<int>(get_int(nj, "node", "warps_required", false, 1));
    if (n.warps_required < 1) throw DomainError("warps_required must be >= 1");
    index[n.id] = static_cast<int>(s.nodes.size());
    s.nodes.push_back(n);
  }
  if (gj.contains("edges")) {
    if (!gj["edges"].is_array()) throw DomainError("\"edges\" must be an array");
    for (const json& ej : gj["edges"]) {
      if (!ej.is_object()) throw DomainError("edge entries must be objects");
      require_keys(ej, "edge", {"src", "dst", "d", "delta", "blocking"});
      LEdge e;
      if (!ej.contains("src") || !ej["src"].is_string() || !ej.contains("dst") || !ej["dst"].is_string())
        throw DomainError("edge requires string \"src\" and \"dst\"");
      auto si = index.find(ej["src"].get<std::string>());
      auto di = index.find(ej["dst"].get<std::string>());
      if (si == index.end())
        throw DomainError("edge references undeclared node \"" + ej["src"].get<std::string>() + "\"");
      if (di == index.end())
        throw DomainError("edge references undeclared node \"" + ej["dst"].get<std::string>() + "\"");
      e.src = si->second;
      e.dst = di->second;
      e.d = get_int(ej, "edge", "d", true, 0);
      if (e.d < 0) throw DomainError("edge d must be >= 0");
      e.delta = static_cast<int>(get_int(ej, "edge", "delta", false, 0));
      if (e.delta < 0) throw DomainError("edge delta must be >= 0");
      if (ej.contains("blocking")) {
        if (!ej["blocking"].is_boolean()) throw DomainError("edge \"blocking\" must be a boolean");
        e.blocking = ej["blocking"].get<bool>();
      }
      s.edges.push_back(e);
    }
  }
  const std::vector<Violation> diags = validate_graph(s);
  if (!diags.empty()) throw DomainError("invalid loop graph (" + diags[0].family + "): " + diags[0].message);
}

// ---- solution: solution_from_json (cli.cpp:96-155) + reconstruct (:161-168)
void parse_solution(const std::string& text, LoweredSchedule& s) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw DomainError(std::string("invalid solution JSON: ") + e.what());
  }
  if (!j.is_object()) throw DomainError("solution JSON must be an object");
  for (auto it = j.begin(); it != j.end(); ++it) {
    const std::string& k = it.key();
    if (k != "I" && k != "L" && k != "M" && k != "A" && k != "streaming_depths" && k != "search_report")
      throw DomainError("unknown solution key: " + k);
  }
  if (!j.contains("I") || !j["I"].is_number_integer() || j["I"].get<int64_t>() < 1)
    throw DomainError("solution needs a positive integer I");
  if (!j.contains("L") || !j["L"].is_number_integer() || j["L"].get<int64_t>() < 1)
    throw DomainError("solution needs a positive integer L");
  if (!j.contains("M") || !j["M"].is_object()) throw DomainError("solution needs an M object");
  s.ii = j["I"].get<int64_t>();
  s.length = j["L"].get<int64_t>();
  const size_t n = s.nodes.size();
  s.m.assign(n, 0);
  s.a.assign(n, 0);
  auto node_of = [&](const std::string& id) {
    for (size_t v = 0; v < n; ++v)
      if (s.nodes[v].id == id) return static_cast<int>(v);
    return -1;
  };
  for (auto it = j["M"].begin(); it != j["M"].end(); ++it) {
    int v = node_of(it.key());
    if (v < 0) throw DomainError("M names unknown node " + it.key());
    if (!it.value().is_number_integer()) throw DomainError("M[" + it.key() + "] must be an integer");
    s.m[static_cast<size_t>(v)] = it.value().get<int64_t>();
  }
  if (j["M"].size() != n) throw DomainError("M must cover every node exactly once");
  // fit in L against the graph as parsed (before the streaming rewrite), as
  // solution_from_json does (cli.cpp:130-137)
  for (size_t v = 0; v < n; ++v) {
    const int64_t eff = std::max<int64_t>(1, s.nodes[v].cycles);
    if (s.m[v] < 0 || s.m[v] > s.length - eff)
      throw DomainError("M[" + s.nodes[v].id + "] = " + std::to_string(s.m[v]) + " does not fit in L");
  }
  if (j.contains("A")) {
    if (!j["A"].is_object()) throw DomainError("A must be an object");
    for (auto it = j["A"].begin(); it != j["A"].end(); ++it) {
      int v = node_of(it.key());
      if (v < 0) throw DomainError("A names unknown node " + it.key());
      if (!it.value().is_number_integer()) throw DomainError("A[" + it.key() + "] must be an integer");
      s.a[static_cast<size_t>(v)] = it.value().get<int>();
    }
  }
  if (j.contains("streaming_depths")) {
    if (!j["streaming_depths"].is_object()) throw DomainError("streaming_depths must be an object");
    for (auto it = j["streaming_depths"].begin(); it != j["streaming_depths"].end(); ++it) {
      if (!it.value().is_number_integer()) throw DomainError("streaming_depths entries must be integers");
      s.streaming_depths[it.key()] = it.value().get<int64_t>();
    }
  }
  // The graph the tables expand against is the streamed one whenever depths
  // were recorded: variable-latency ops without predecessors issue in zero
  // cycles (jointsolve.cpp:511-524).
  if (!s.streaming_depths.empty()) {
    std::vector<int> indeg(n, 0);
    for (const LEdge& e : s.edges) ++indeg[static_cast<size_t>(e.dst)];
    for (size_t v = 0; v < n; ++v)
      if (s.nodes[v].variable_latency && indeg[v] == 0) {
        s.nodes[v].cycles = 0;
        for (auto& row : s.nodes[v].rrt) row.clear();
      }
  }
  // A's alignment and range are checked with the other families by
  // validate_schedule (warp_uniqueness), which runs before anything indexes A
  s.copies = (s.length + s.ii - 1) / s.ii;
}

// Node id -> executor op. The ids are the names the FA / GEMM loop problems
// use (tools/make_problems.py); anything else cannot be realized.
bool classify(const std::string& id, uint8_t& kind, uint8_t& tile) {
  struct Pfx { const char* p; uint8_t k; };
  static const Pfx fixed[] = {{"LDK", TWFA_OP_LDK}, {"LDV", TWFA_OP_LDV}, {"LDA", TWFA_OP_LDA},
                              {"LDB", TWFA_OP_LDB}, {"MMA", TWFA_OP_MMA}, {"LDQ", TWFA_OP_LDQ},
                              {"LDO", TWFA_OP_LDO}, {"ST", TWFA_OP_ST},   {"DP", TWFA_OP_DP},
                              {"EXB", TWFA_OP_EXB}, {"DS", TWFA_OP_DS},   {"DV", TWFA_OP_DV},
                              {"DK", TWFA_OP_DK},   {"DQ", TWFA_OP_DQ},   {"RD", TWFA_OP_RD}};
  for (const Pfx& f : fixed)
    if (id == f.p) { kind = f.k; tile = 0; return true; }
  static const Pfx tiled[] = {{"MX", TWFA_OP_MX},   {"EX", TWFA_OP_EX},  {"CR", TWFA_OP_CR},  {"PV", TWFA_OP_PV},
                              {"SA", TWFA_OP_SA},   {"SB", TWFA_OP_SB},  {"S", TWFA_OP_S},    {"ST", TWFA_OP_ST},
                              {"DP", TWFA_OP_DP},   {"EXB", TWFA_OP_EXB}, {"DS", TWFA_OP_DS}, {"DV", TWFA_OP_DV},
                              {"DK", TWFA_OP_DK},   {"DQ", TWFA_OP_DQ},  {"RD", TWFA_OP_RD}};
  for (const Pfx& f : tiled) {
    const size_t l = std::strlen(f.p);
    if (id.size() == l + 1 && id.compare(0, l, f.p) == 0 && id[l] >= '0' && id[l] < '0' + TWFA_MAX_TILES) {
      kind = f.k;
      tile = static_cast<uint8_t>(id[l] - '0');
      return true;
    }
  }
  return false;
}

// FA backward (family FA_BWD): the roles of the realized kernel are the
// solver's warp assignment. Tensor-core ops issue from one thread (their
// in-order execution realizes the DV -> DQ and DK -> DP aliasing edges);
// EXB and DS share a warpgroup and the DS after EXB carries P in registers;
// RD runs on a warpgroup; LDQ / LDO stream from one TMA warp.
template <class NodeId, class DepthOf, class PrefetchOf>
void derive_bwd(LoweredSchedule& s, NodeId&& node_id, DepthOf&& depth_of, PrefetchOf&& prefetch_of) {
  TwfaDevicePlan& p = s.plan;
  p.family = TWFA_FAMILY_FA_BWD;
  p.num_tiles = 1;
  static const char* ids[] = {"LDQ", "LDO", "ST", "DP", "EXB", "DS", "DV", "DK", "DQ", "RD"};
  for (const char* id : ids)
    if (node_id(id) < 0) throw DomainError(std::string("FA-backward loop is missing ") + id);
  if (s.nodes.size() != 10) throw DomainError("FA-backward loop has unexpected extra nodes");
  const TwfaPlanOp &ldq = p.ops[node_id("LDQ")], &ldo = p.ops[node_id("LDO")];
  if (ldq.warp_start != ldo.warp_start || ldq.warp_count != 1)
    throw DomainError("LDQ and LDO must be issued by one TMA warp");
  p.load_warp = ldq.warp_start;
  p.k_depth = depth_of("LDQ");
  p.v_depth = depth_of("LDO");
  p.k_prefetch = prefetch_of(node_id("LDQ"), p.k_depth);
  p.v_prefetch = prefetch_of(node_id("LDO"), p.v_depth);
  if (p.k_depth > 2 || p.v_depth > 2) throw DomainError("Q / dO rings deeper than 2 exceed shared memory");
  const int mma = p.ops[node_id("ST")].warp_start;
  for (const char* id : {"ST", "DP", "DV", "DK", "DQ"}) {
    const TwfaPlanOp& o = p.ops[node_id(id)];
    if (o.warp_count != 1 || o.warp_start != mma)
      throw DomainError("tensor-core ops of the backward loop must issue from one warp");
  }
  p.mma_warp = mma;
  const TwfaPlanOp &exb = p.ops[node_id("EXB")], &ds = p.ops[node_id("DS")], &rd = p.ops[node_id("RD")];
  for (const TwfaPlanOp* o : {&exb, &ds, &rd})
    if (o->warp_count != 4 || o->warp_start % 4 != 0)
      throw DomainError("EXB, DS and RD are row-wise over 128 TMEM lanes: they need a warpgroup");
  for (int w : {p.load_warp, p.mma_warp})
    for (const TwfaPlanOp* o : {&exb, &ds, &rd})
      if (w >= o->warp_start && w < o->warp_start + 4)
        throw DomainError("the TMA / MMA warp cannot be inside the EXB, DS or RD warpgroup");
  if (rd.warp_start == exb.warp_start || rd.warp_start == ds.warp_start)
    throw DomainError("RD needs its own warpgroup (register budget of the dQ staging)");
  const int exi = node_id("EXB"), dsi = node_id("DS"), sti = node_id("ST");
  if (exb.warp_start == ds.warp_start) {
    // one warpgroup: P^T (128 fp32 registers) lives from EXB to DS, so DS
    // must be the next op of every warp of the group, in the same iteration
    for (int w = exb.warp_start; w < exb.warp_start + 4; ++w) {
      const std::vector<int>& prog = s.warp_prog[static_cast<size_t>(w)];
      auto it = std::find(prog.begin(), prog.end(), exi);
      if (it == prog.end() || it + 1 == prog.end() || *(it + 1) != dsi ||
          s.stage[static_cast<size_t>(exi)] != s.stage[static_cast<size_t>(dsi)])
        throw DomainError("DS must directly follow EXB on a shared warpgroup (P is carried in registers)");
    }
    p.ops[exi].flags |= TWFA_OPF_FUSE_NEXT;
    p.ops[dsi].flags |= TWFA_OPF_FUSED;
  } else {
    // two warpgroups: DS reads P^T (bf16) back from the S^T columns, which
    // S^T(i+1) overwrites; the graph must order that read (DS -> ST, delta >= 1)
    bool ordered = false;
    for (const LEdge& e : s.edges)
      ordered = ordered || (e.src == dsi && e.dst == sti && e.delta >= 1);
    if (!ordered) throw DomainError("EXB and DS on different warpgroups need a DS -> ST (delta 1) edge");
    p.ops[sti].flags |= TWFA_OPF_WAIT_PREAD;
  }
  p.sm_warp[0] = exb.warp_start;
  p.sm_warp[1] = ds.warp_start;
  p.cr_warp[0] = rd.warp_start;  // RD warpgroup (also writes dK, dV)
  p.heavy_wg_mask = (1 << (exb.warp_start / 4)) | (1 << (ds.warp_start / 4));
  auto later = [&](const char* a, const char* b) {
    const int x = node_id(a), y = node_id(b);
    return std::make_pair(s.m[static_cast<size_t>(x)], p.ops[x].order) >
                   std::make_pair(s.m[static_cast<size_t>(y)], p.ops[y].order)
               ? x
               : y;
  };
  // dQ staging buffer: the graph says where RD stages dQ_i -- an LDQ -> RD
  // edge puts it in Q_i's ring slot (RD then releases that slot, and DQ's
  // commit frees the dS buffer); otherwise the dS buffer (RD frees it)
  bool q_staging = false;
  for (const LEdge& e : s.edges) q_staging = q_staging || (e.src == node_id("LDQ") && e.dst == node_id("RD"));
  p.s_split = q_staging ? 1 : 0;  // FA backward: RD stages dQ in the Q ring slot
  if (q_staging) {
    p.ops[node_id("RD")].flags |= TWFA_OPF_RELEASE;
    p.ops[node_id("DQ")].flags |= TWFA_OPF_RELEASE;  // DQ's commit frees the dS buffer
    p.ops[later("DP", "DV")].flags |= TWFA_OPF_RELEASE;
    return;
  }
  // the later tensor-core reader of Q_i (ST, DK) and of dO_i (DP, DV)
  // releases the ring slot with its commit
  p.ops[later("ST", "DK")].flags |= TWFA_OPF_RELEASE;
  p.ops[later("DP", "DV")].flags |= TWFA_OPF_RELEASE;
}

// FA backward with two 64-query sub-tiles per iteration (family FA_BWD,
// num_tiles 2; tools/make_problems.py:fa_backward_pp_problem, realized by
// fa_bwd_pp_sm100.cu): per sub-tile k the nodes ST_k, DP_k, EXB_k, DS_k,
// DV_k, DK_k, DQ_k, RD_k, plus the streamed LDQ / LDO of the 128-row tiles.
// All tensor-core ops issue from one thread (the in-order aliasing edges
// DV_k -> DQ_k and DK_k -> DP_k); EXB_k and DS_k share a warpgroup with DS_k
// right after EXB_k (P^T_k in registers); RD_k runs on a warpgroup of its own
// register class. The later tensor-core reader of Q_i (dO_i) in issue order
// releases its ring slot.
template <class NodeId, class DepthOf, class PrefetchOf>
void derive_bwd_pp(LoweredSchedule& s, NodeId&& node_id, DepthOf&& depth_of, PrefetchOf&& prefetch_of) {
  TwfaDevicePlan& p = s.plan;
  p.family = TWFA_FAMILY_FA_BWD;
  p.num_tiles = 2;
  static const char* per_tile[] = {"ST", "DP", "EXB", "DS", "DV", "DK", "DQ", "RD"};
  for (const char* id : {"LDQ", "LDO"})
    if (node_id(id) < 0) throw DomainError(std::string("FA-backward loop is missing ") + id);
  for (int k = 0; k < 2; ++k)
    for (const char* id : per_tile)
      if (node_id(id + std::to_string(k)) < 0)
        throw DomainError(std::string("two-sub-tile FA-backward loop is missing ") + id + std::to_string(k));
  if (s.nodes.size() != 18) throw DomainError("two-sub-tile FA-backward loop has unexpected extra nodes");
  const TwfaPlanOp &ldq = p.ops[node_id("LDQ")], &ldo = p.ops[node_id("LDO")];
  if (ldq.warp_start != ldo.warp_start || ldq.warp_count != 1)
    throw DomainError("LDQ and LDO must be issued by one TMA warp");
  p.load_warp = ldq.warp_start;
  p.k_depth = depth_of("LDQ");
  p.v_depth = depth_of("LDO");
  p.k_prefetch = prefetch_of(node_id("LDQ"), p.k_depth);
  p.v_prefetch = prefetch_of(node_id("LDO"), p.v_depth);
  if (p.k_depth > 2 || p.v_depth > 2) throw DomainError("Q / dO rings deeper than 2 exceed shared memory");
  auto op = [&](const char* id, int k) -> TwfaPlanOp& { return p.ops[node_id(id + std::to_string(k))]; };
  const int mma = op("ST", 0).warp_start;
  for (int k = 0; k < 2; ++k)
    for (const char* id : {"ST", "DP", "DV", "DK", "DQ"}) {
      const TwfaPlanOp& o = op(id, k);
      if (o.warp_count != 1 || o.warp_start != mma)
        throw DomainError("tensor-core ops of the backward loop must issue from one warp");
    }
  p.mma_warp = mma;
  int heavy = 0;
  for (int k = 0; k < 2; ++k) {
    const TwfaPlanOp &exb = op("EXB", k), &ds = op("DS", k), &rd = op("RD", k);
    for (const TwfaPlanOp* o : {&exb, &ds, &rd})
      if (o->warp_count != 4 || o->warp_start % 4 != 0)
        throw DomainError("EXB, DS and RD are row-wise over 128 TMEM lanes: they need a warpgroup");
    for (int w : {p.load_warp, p.mma_warp})
      for (const TwfaPlanOp* o : {&exb, &ds, &rd})
        if (w >= o->warp_start && w < o->warp_start + 4)
          throw DomainError("the TMA / MMA warp cannot be inside an EXB, DS or RD warpgroup");
    if (exb.warp_start != ds.warp_start)
      throw DomainError("EXB_k and DS_k must share a warpgroup (P^T_k is carried in registers)");
    const int exi = node_id("EXB" + std::to_string(k)), dsi = node_id("DS" + std::to_string(k));
    for (int w = exb.warp_start; w < exb.warp_start + 4; ++w) {
      const std::vector<int>& prog = s.warp_prog[static_cast<size_t>(w)];
      auto it = std::find(prog.begin(), prog.end(), exi);
      if (it == prog.end() || it + 1 == prog.end() || *(it + 1) != dsi ||
          s.stage[static_cast<size_t>(exi)] != s.stage[static_cast<size_t>(dsi)])
        throw DomainError("DS_k must directly follow EXB_k on its warpgroup (P is carried in registers)");
    }
    p.ops[exi].flags |= TWFA_OPF_FUSE_NEXT;
    p.ops[dsi].flags |= TWFA_OPF_FUSED;
    p.sm_warp[k] = exb.warp_start;
    p.cr_warp[k] = rd.warp_start;
    heavy |= 1 << (exb.warp_start / 4);
  }
  for (int k = 0; k < 2; ++k)
    if (p.cr_warp[k] == p.sm_warp[0] || p.cr_warp[k] == p.sm_warp[1])
      throw DomainError("RD needs a warpgroup of its own (register budget of the dQ staging)");
  p.heavy_wg_mask = heavy;
  // the graph's aliasing edges the kernel realizes by issue order on the MMA
  // thread or by its barriers
  auto has_edge = [&](const std::string& a, const std::string& b, int delta) {
    for (const LEdge& e : s.edges)
      if (e.src == node_id(a) && e.dst == node_id(b) && e.delta == delta) return true;
    return false;
  };
  for (int k = 0; k < 2; ++k) {
    const std::string K = std::to_string(k);
    if (!has_edge("DV" + K, "DQ" + K, 0) || !has_edge("DK" + K, "DP" + K, 1) || !has_edge("RD" + K, "ST" + K, 1) ||
        !has_edge("DQ" + K, "DS" + K, 1) || !has_edge("RD" + K, "DS" + K, 1))
      throw DomainError("two-sub-tile FA-backward loop lacks a tensor-memory / shared-memory aliasing edge");
  }
  // ring slots: the last tensor-core reader of Q_i (of dO_i) in issue order
  auto last = [&](std::initializer_list<std::string> ids) {
    int best = -1;
    for (const std::string& id : ids) {
      const int v = node_id(id);
      if (best < 0 || std::make_pair(s.stage[static_cast<size_t>(v)], p.ops[v].order) >
                          std::make_pair(s.stage[static_cast<size_t>(best)], p.ops[best].order))
        best = v;
    }
    return best;
  };
  p.ops[last({"ST0", "ST1", "DK0", "DK1"})].flags |= TWFA_OPF_RELEASE;
  p.ops[last({"DP0", "DP1", "DV0", "DV1"})].flags |= TWFA_OPF_RELEASE;
}

void derive(LoweredSchedule& s) {
  const size_t n = s.nodes.size();
  if (n > TWFA_MAX_NODES) throw DomainError("graph has more nodes than the executor supports");
  if (s.num_warps > TWFA_MAX_WARPS) throw DomainError("machine has more warps than a CTA of the executor");
  TwfaDevicePlan& p = s.plan;
  std::memset(&p, 0, sizeof(p));
  p.ii = static_cast<int32_t>(s.ii);
  p.length = static_cast<int32_t>(s.length);
  p.copies = static_cast<int32_t>(s.copies);
  p.num_nodes = static_cast<int32_t>(n);
  p.num_warps = s.num_warps;
  s.stage.assign(n, 0);
  s.slot.assign(n, 0);
  std::set<int> kinds;
  int max_stage = 0;
  for (size_t v = 0; v < n; ++v) {
    TwfaPlanOp& op = p.ops[v];
    uint8_t kind = 0, tile = 0;
    if (!classify(s.nodes[v].id, kind, tile))
      throw DomainError("node \"" + s.nodes[v].id + "\" has no sm_100a realization");
    s.stage[v] = s.m[v] / s.ii;
    s.slot[v] = s.m[v] % s.ii;
    if (s.stage[v] > 250) throw DomainError("schedule too deep");
    max_stage = std::max<int>(max_stage, static_cast<int>(s.stage[v]));
    op.node = static_cast<uint8_t>(v);
    op.kind = kind;
    op.tile = tile;
    op.stage = static_cast<uint8_t>(s.stage[v]);
    op.slot = static_cast<uint8_t>(s.slot[v]);
    op.warp_start = static_cast<uint8_t>(s.a[v]);
    op.warp_count = static_cast<uint8_t>(std::max(1, s.nodes[v].warps_required));
    kinds.insert(kind);
  }
  p.max_stage = max_stage;

  // per-warp trip programs: ops covering the warp, ordered by their cycle in
  // the trip and then by declaration order -- the key the reference's
  // program synthesis sorts a region by (codegen.cpp:179-183) -- except that
  // streamed loads (zero cycles and no unit reservation after the streaming
  // rewrite, jointsolve.cpp:511-524) issue after the timed ops of their
  // cycle: a zero-duration op occupies no part of the cycle, so either side
  // realizes the same modulo schedule, and the ring prefetch (prefetch_of)
  // already serves its consumers from an earlier trip.
  auto streamed = [&](int v) { return s.nodes[static_cast<size_t>(v)].cycles == 0; };
  // streamed loads moved to the end of their trip program (see below)
  std::vector<bool> late(n, false);
  auto order_key = [&](int v) {
    const bool l = late[static_cast<size_t>(v)];
    return std::make_tuple(l ? s.ii : s.slot[static_cast<size_t>(v)], streamed(v) ? 1 : 0, v);
  };
  auto build_programs = [&] {
    s.warp_prog.assign(static_cast<size_t>(s.num_warps), {});
    for (int w = 0; w < s.num_warps; ++w) {
      std::vector<int>& prog = s.warp_prog[static_cast<size_t>(w)];
      for (size_t v = 0; v < n; ++v)
        if (p.ops[v].warp_start <= w && w < p.ops[v].warp_start + p.ops[v].warp_count)
          prog.push_back(static_cast<int>(v));
      std::stable_sort(prog.begin(), prog.end(), [&](int x, int y) { return order_key(x) < order_key(y); });
      p.prog_len[w] = static_cast<uint8_t>(prog.size());
      for (size_t i = 0; i < prog.size(); ++i) {
        p.prog[w][i] = static_cast<uint8_t>(prog[i]);
        if (w == p.ops[prog[i]].warp_start) p.ops[prog[i]].order = static_cast<uint8_t>(i);
      }
    }
    // Realizability of the order: a consumer that issues in the same cycle as
    // its producer on a shared warp must come after it in the trip program,
    // otherwise the warp would wait on itself.
    for (const LEdge& e : s.edges) {
      if (e.src == e.dst) continue;
      const TwfaPlanOp& u = p.ops[e.src];
      const TwfaPlanOp& v = p.ops[e.dst];
      const int64_t gap = s.m[static_cast<size_t>(e.dst)] + e.delta * s.ii - s.m[static_cast<size_t>(e.src)];
      if (gap < e.d)
        throw DomainError("schedule violates dependence " + s.nodes[e.src].id + " -> " + s.nodes[e.dst].id);
      const bool share = u.warp_start < v.warp_start + v.warp_count && v.warp_start < u.warp_start + u.warp_count;
      if (gap == 0 && share && !streamed(e.src) && order_key(e.dst) < order_key(e.src))
        throw DomainError("same-cycle dependence " + s.nodes[e.src].id + " -> " + s.nodes[e.dst].id +
                          " is ordered consumer-first on a shared warp");
    }
  };
  build_programs();

  auto depth_of = [&](const char* id) -> int32_t {
    auto it = s.streaming_depths.find(id);
    return it == s.streaming_depths.end() ? 0 : static_cast<int32_t>(it->second);
  };
  auto node_id = [&](const std::string& id) {
    for (size_t v = 0; v < n; ++v)
      if (s.nodes[v].id == id) return static_cast<int>(v);
    return -1;
  };
  // streamed loads: ring depth must cover the stage lag to every consumer
  // Streamed load of depth D: iteration j is loaded in trip j + stage - p
  // (prefetch distance p) into slot j % D, after the consumers of iteration
  // j - D released that slot. p = D - 1 unless a consumer on the load's own
  // warp would release the slot only later in program order.
  auto prefetch_of = [&](int ld, int32_t depth) -> int32_t {
    if (depth < 1) throw DomainError("streamed load " + s.nodes[ld].id + " has no ring depth");
    const TwfaPlanOp& L = p.ops[ld];
    int64_t pf = depth - 1;
    for (const LEdge& e : s.edges) {
      if (e.src != ld) continue;
      const TwfaPlanOp& C = p.ops[e.dst];
      const int64_t lag = s.stage[static_cast<size_t>(e.dst)] + e.delta - s.stage[static_cast<size_t>(ld)];
      if (lag >= depth)
        throw DomainError("ring depth " + std::to_string(depth) + " of " + s.nodes[ld].id +
                          " is shallower than its consumer lag");
      const bool share = L.warp_start < C.warp_start + C.warp_count && C.warp_start < L.warp_start + L.warp_count;
      if (!share) continue;
      const bool before = order_key(e.dst) < order_key(ld);
      pf = std::min<int64_t>(pf, depth - lag - (before ? 0 : 1));
    }
    if (pf < 0)
      throw DomainError("ring depth " + std::to_string(depth) + " of " + s.nodes[ld].id +
                        " cannot cover a consumer on its own warp");
    return static_cast<int32_t>(pf);
  };

  // A streamed load whose ring slot is released by a consumer later in its
  // own warp's trip program cannot run ahead from its slot position
  // (prefetch 0): the iteration it loads is then consumed in the same trip,
  // and a consumer ordered before it would wait on it. Such a load issues at
  // the end of its trip program instead -- after every same-warp consumer --
  // which lets it run one iteration ahead. Zero-cycle streamed ops occupy no
  // part of the cycle, so the modulo schedule is unchanged.
  bool moved = false;
  for (size_t v = 0; v < n; ++v) {
    if (!streamed(static_cast<int>(v))) continue;
    auto it = s.streaming_depths.find(s.nodes[v].id);
    if (it == s.streaming_depths.end() || it->second < 2) continue;
    if (prefetch_of(static_cast<int>(v), static_cast<int32_t>(it->second)) > 0) continue;
    late[v] = true;
    moved = true;
  }
  if (moved) build_programs();
  for (size_t v = 0; v < n; ++v) {  // no consumer may wait on a later load of its own warp
    if (!streamed(static_cast<int>(v))) continue;
    auto it = s.streaming_depths.find(s.nodes[v].id);
    if (it == s.streaming_depths.end()) continue;
    if (prefetch_of(static_cast<int>(v), static_cast<int32_t>(it->second)) > 0) continue;
    for (const LEdge& e : s.edges) {
      if (static_cast<size_t>(e.src) != v) continue;
      const TwfaPlanOp &L = p.ops[v], &C = p.ops[e.dst];
      const bool share = L.warp_start < C.warp_start + C.warp_count && C.warp_start < L.warp_start + L.warp_count;
      const int64_t lag = s.stage[static_cast<size_t>(e.dst)] + e.delta - s.stage[v];
      if (share && lag == 0 && order_key(e.dst) < order_key(static_cast<int>(v)))
        throw DomainError("streamed load " + s.nodes[v].id + " cannot run ahead of " + s.nodes[e.dst].id +
                          " on their shared warp");
    }
  }

  const bool is_fa = (kinds.count(TWFA_OP_S) || (kinds.count(TWFA_OP_SA) && kinds.count(TWFA_OP_SB))) &&
                     kinds.count(TWFA_OP_PV);
  const bool is_gemm = kinds.count(TWFA_OP_MMA) && kinds.count(TWFA_OP_LDA) && kinds.count(TWFA_OP_LDB);
  const bool is_bwd = kinds.count(TWFA_OP_ST) && kinds.count(TWFA_OP_DQ);
  if (is_fa + is_gemm + is_bwd != 1) throw DomainError("graph is neither the FA-forward, FA-backward nor GEMM loop");
  if (is_bwd) {
    if (node_id("ST0") >= 0)
      derive_bwd_pp(s, node_id, depth_of, prefetch_of);
    else
      derive_bwd(s, node_id, depth_of, prefetch_of);
    return;
  }
  if (is_gemm) {
    p.family = TWFA_FAMILY_GEMM;
    const int lda = node_id("LDA"), ldb = node_id("LDB"), mma = node_id("MMA");
    if (n != 3) throw DomainError("GEMM loop must have exactly LDA, LDB, MMA");
    if (p.ops[lda].warp_start != p.ops[ldb].warp_start)
      throw DomainError("LDA and LDB must share the TMA warp");
    if (p.ops[mma].warp_count != 1) throw DomainError("MMA issue is single-warp");
    if (p.ops[mma].warp_start == p.ops[lda].warp_start)
      throw DomainError("MMA issue cannot share the TMA warp");
    p.load_warp = p.ops[lda].warp_start;
    p.mma_warp = p.ops[mma].warp_start;
    p.k_depth = depth_of("LDA");
    p.v_depth = depth_of("LDB");
    if (p.k_depth != p.v_depth) throw DomainError("LDA and LDB must stream with one ring depth");
    p.k_prefetch = prefetch_of(lda, p.k_depth);
    p.v_prefetch = prefetch_of(ldb, p.v_depth);
    if (s.ii != 1 || max_stage != 0)
      throw DomainError("GEMM mainloop realization expects the I = 1 single-stage schedule");
    return;
  }

  p.family = TWFA_FAMILY_FA_FWD;
  // S_k as one GEMM, or split into SA_k + SB_k
  const bool split = node_id("SA0") >= 0;
  const char* s_last = split ? "SB" : "S";  // the GEMM that overwrites P_k's columns
  p.s_split = split ? 1 : 0;
  int tiles = 0;
  while (tiles < TWFA_MAX_TILES && node_id((split ? "SA" : "S") + std::to_string(tiles)) >= 0) ++tiles;
  if (tiles < 1) throw DomainError("FA loop needs S0 (or SA0, SB0)");
  p.num_tiles = tiles;
  const int ldk = node_id("LDK"), ldv = node_id("LDV");
  if (ldk < 0 || ldv < 0) throw DomainError("FA loop needs LDK and LDV");
  for (int k = 0; k < tiles; ++k)
    for (const char* pre : {"S", "SA", "SB", "MX", "EX", "CR", "PV"})
      if ((split ? std::string(pre) != "S" : (std::string(pre) != "SA" && std::string(pre) != "SB")) &&
          node_id(pre + std::to_string(k)) < 0)
        throw DomainError(std::string("FA loop is missing ") + pre + std::to_string(k));
  if (static_cast<int>(n) != 2 + (split ? 6 : 5) * tiles) throw DomainError("FA loop has unexpected extra nodes");
  if (p.ops[ldk].warp_start != p.ops[ldv].warp_start || p.ops[ldk].warp_count != 1)
    throw DomainError("LDK and LDV must be issued by one TMA warp");
  p.load_warp = p.ops[ldk].warp_start;
  p.k_depth = depth_of("LDK");
  p.v_depth = depth_of("LDV");
  p.k_prefetch = prefetch_of(ldk, p.k_depth);
  p.v_prefetch = prefetch_of(ldv, p.v_depth);
  for (int k = 0; k < tiles; ++k) {
    const TwfaPlanOp& mx = p.ops[node_id("MX" + std::to_string(k))];
    const TwfaPlanOp& ex = p.ops[node_id("EX" + std::to_string(k))];
    const TwfaPlanOp& cr = p.ops[node_id("CR" + std::to_string(k))];
    const TwfaPlanOp& sk = p.ops[node_id(s_last + std::to_string(k))];
    if (split && p.ops[node_id("SA" + std::to_string(k))].warp_count != 1)
      throw DomainError("MMA issue ops are single-warp");
    const TwfaPlanOp& pv = p.ops[node_id("PV" + std::to_string(k))];
    // TMEM lane quadrants: a 128-row tile is touched by 4 warps, one per
    // quadrant (warp % 4), so row-wise ops need an aligned warpgroup.
    for (const TwfaPlanOp* o : {&mx, &ex, &cr})
      if (o->warp_count != 4 || o->warp_start % 4 != 0)
        throw DomainError("softmax/correction ops of tile " + std::to_string(k) + " must run on a warpgroup");
    // running max and row sum are carried in registers of one warpgroup
    if (mx.warp_start != ex.warp_start)
      throw DomainError("MX" + std::to_string(k) + " and EX" + std::to_string(k) + " must share a warpgroup");
    if (sk.warp_count != 1 || pv.warp_count != 1) throw DomainError("MMA issue ops are single-warp");
    p.sm_warp[k] = mx.warp_start;
    p.cr_warp[k] = cr.warp_start;
    p.heavy_wg_mask |= 1 << (mx.warp_start / 4);
    // fuse MX_k -> EX_k when EX_k is the next op of every warp of the group
    const int mxi = node_id("MX" + std::to_string(k)), exi = node_id("EX" + std::to_string(k));
    bool adjacent = s.stage[static_cast<size_t>(mxi)] == s.stage[static_cast<size_t>(exi)];
    for (int w = mx.warp_start; w < mx.warp_start + 4 && adjacent; ++w) {
      const std::vector<int>& prog = s.warp_prog[static_cast<size_t>(w)];
      auto it = std::find(prog.begin(), prog.end(), mxi);
      adjacent = it != prog.end() && it + 1 != prog.end() && *(it + 1) == exi;
    }
    if (adjacent) {
      p.ops[mxi].flags |= TWFA_OPF_FUSE_NEXT;
      p.ops[exi].flags |= TWFA_OPF_FUSED;
    } else if (split) {
      // SA_k(i+1) may overwrite S columns 0-63 once MX_k(i) has read them:
      // only a register-resident row (fused MX_k; EX_k) never re-reads S
      throw DomainError("split S needs MX" + std::to_string(k) + " and EX" + std::to_string(k) +
                        " back to back on their warpgroup");
    }
    // same issuing warp for S_k and PV_k: the realizability check above
    // guarantees PV_k(i-1) precedes S_k(i) in that warp's program order
    if (sk.warp_start == pv.warp_start) p.ops[node_id(s_last + std::to_string(k))].flags |= TWFA_OPF_INORDER;
  }
  if (__builtin_popcount(static_cast<unsigned>(p.heavy_wg_mask)) > 2)
    throw DomainError("softmax of more than two warpgroups exceeds the register file");
  // MUFU reservation order of the EX ops (all EX share the unit; realized as a
  // token ring when they share a stage so every trip holds each of them once)
  {
    std::vector<int> ex;
    for (int k = 0; k < tiles; ++k) ex.push_back(node_id("EX" + std::to_string(k)));
    bool same_stage = true;
    for (int v : ex) same_stage = same_stage && s.stage[static_cast<size_t>(v)] == s.stage[static_cast<size_t>(ex[0])];
    if (same_stage && ex.size() >= 2) {
      std::stable_sort(ex.begin(), ex.end(), [&](int x, int y) {
        return std::make_pair(s.slot[static_cast<size_t>(x)], x) < std::make_pair(s.slot[static_cast<size_t>(y)], y);
      });
      p.ex_ring_len = static_cast<int32_t>(ex.size());
      for (size_t i = 0; i < ex.size(); ++i) p.ex_ring[i] = p.ops[ex[i]].tile;
    }
  }
  // S ring in tensor memory: the delta of PV_k -> S_k (S_k(i + delta)
  // overwrites the P_k(i) aliased over S_k(i)); 1 = one 128-key S tile per
  // sub-tile, 2 = two 64-key tiles in the same 128 columns
  p.s_depth = 0;
  for (const LEdge& e : s.edges)
    for (int k = 0; k < tiles; ++k)
      if (e.src == node_id("PV" + std::to_string(k)) && e.dst == node_id(s_last + std::to_string(k))) {
        if (p.s_depth != 0 && p.s_depth != e.delta) throw DomainError("sub-tiles disagree on the S ring depth");
        p.s_depth = e.delta;
      }
  if (p.s_depth != 1 && p.s_depth != 2)
    throw DomainError("PV_k -> S_k must carry delta 1 or 2 (S ring depth in tensor memory)");
  p.kv_tile = 128 / p.s_depth;
  if (split && p.s_depth != 1) throw DomainError("split S is realized with a single 128-key S tile (delta 1)");
  // smem: Q (tiles x 32 KiB) + K ring + V ring of kv_tile-key slots
  const int64_t kv_bytes = static_cast<int64_t>(p.kv_tile) * 256;
  // + 16 KiB epilogue staging; 227 KiB per CTA minus the static state
  // (barriers, row statistics, trip programs ~10 KiB) and alignment slack
  // A plan the CTA-pair realization can run (128-key tiles, unsplit S, two
  // sub-tiles) stages half of every K / V tile per CTA, so deeper rings fit
  // there (the launch then requires pairs, capi.cpp use_pairs)
  const bool pair_capable = p.kv_tile == 128 && !split && tiles == 2;
  const int64_t smem = 32768LL * tiles + kv_bytes / (pair_capable ? 2 : 1) * (p.k_depth + p.v_depth) + 16384;
  if (p.k_depth > 4 || p.v_depth > 4) throw DomainError("ring depth above 4");
  if (smem > 216 * 1024) throw DomainError("ring depths exceed shared memory");
  // Q tiles are loaded once per work tile, outside the loop body: an idle
  // warp (no op of the schedule, outside the softmax and correction
  // warpgroups) waits for the last S_k of a tile and loads the next tile's
  // Q_k while the pipeline drains, so the load warp never blocks on it
  p.q_warp = -1;
  for (int w = 0; w < s.num_warps && p.q_warp < 0; ++w) {
    if (p.prog_len[w] != 0 || w == p.load_warp || ((p.heavy_wg_mask >> (w / 4)) & 1)) continue;
    bool cr = false;
    for (int k = 0; k < tiles; ++k) cr = cr || (w / 4) * 4 == p.cr_warp[k];
    if (!cr) p.q_warp = w;
  }
  // one epilogue staging buffer: the sub-tiles' corrections (and with them
  // the epilogues) must run on one warpgroup
  for (int k = 1; k < tiles; ++k)
    if (p.cr_warp[k] != p.cr_warp[0])
      throw DomainError("CR ops of all Q sub-tiles must share a warpgroup (one epilogue staging buffer)");
}

}  // namespace

LoweredSchedule parse(const std::string& problem_json, const std::string& solution_json) {
  LoweredSchedule s;
  parse_problem(problem_json, s);
  parse_solution(solution_json, s);
  return s;
}

std::string violations_json(const std::vector<Violation>& v) {
  json arr = json::array();
  for (const Violation& x : v) arr.push_back(json::array({x.family, x.message}));
  return arr.dump();
}

LoweredSchedule lower(const std::string& problem_json, const std::string& solution_json) {
  LoweredSchedule s;
  parse_problem(problem_json, s);
  parse_solution(solution_json, s);
  const std::vector<Violation> bad = validate_schedule(s);
  if (!bad.empty()) {
    std::string fams;
    for (const Violation& v : bad)
      if (fams.find(v.family) == std::string::npos) fams += (fams.empty() ? "" : ", ") + v.family;
    throw DomainError("schedule rejected by validate_program (" + std::to_string(bad.size()) + " violation" +
                      (bad.size() > 1 ? "s" : "") + " in " + fams + "; first: " + bad[0].family + ": " +
                      bad[0].message + ")");
  }
  derive(s);
  return s;
}

std::vector<Violation> validate_graph(const LoweredSchedule& s) {
  std::vector<Violation> out;
  const int n = static_cast<int>(s.nodes.size());
  // the delta = 0 subgraph must be a DAG (iterative DFS, 0 new / 1 open / 2 done)
  std::vector<std::vector<int>> adj(static_cast<size_t>(n));
  for (const LEdge& e : s.edges)
    if (e.delta == 0) adj[static_cast<size_t>(e.src)].push_back(e.dst);
  std::vector<int> state(static_cast<size_t>(n), 0);
  bool cycle = false;
  for (int root = 0; root < n && !cycle; ++root) {
    if (state[static_cast<size_t>(root)]) continue;
    std::vector<std::pair<int, size_t>> stack{{root, 0}};
    state[static_cast<size_t>(root)] = 1;
    while (!stack.empty() && !cycle) {
      auto& [v, i] = stack.back();
      if (i < adj[static_cast<size_t>(v)].size()) {
        const int w = adj[static_cast<size_t>(v)][i++];
        if (state[static_cast<size_t>(w)] == 1) cycle = true;
        else if (state[static_cast<size_t>(w)] == 0) {
          state[static_cast<size_t>(w)] = 1;
          stack.push_back({w, 0});
        }
      } else {
        state[static_cast<size_t>(v)] = 2;
        stack.pop_back();
      }
    }
  }
  if (cycle) out.push_back({"zero-delta-cycle", "dependence cycle with zero total iteration distance"});
  for (const LNode& node : s.nodes) {
    for (size_t f = 0; f < node.rrt.size(); ++f)
      for (size_t c = 0; c < node.rrt[f].size(); ++c)
        if (node.rrt[f][c] > s.units[f].capacity)
          out.push_back({"rrt-exceeds-capacity", "node \"" + node.id + "\" reserves " +
                                                     std::to_string(node.rrt[f][c]) + " of unit \"" + s.units[f].name +
                                                     "\" (capacity " + std::to_string(s.units[f].capacity) + ")"});
    if (node.warps_required > s.num_warps)
      out.push_back({"warps-required-too-large", "node \"" + node.id + "\" requires " +
                                                     std::to_string(node.warps_required) +
                                                     " warps but the machine has " + std::to_string(s.num_warps)});
  }
  return out;
}

std::vector<Violation> validate_schedule(const LoweredSchedule& s) {
  std::vector<Violation> out;
  const size_t n = s.nodes.size();
  const int64_t ii = s.ii, len = s.length;
  const int64_t copies = std::max<int64_t>(1, (len + ii - 1) / ii);
  const int64_t horizon = (copies - 1) * ii + len;
  auto fmt = [](int64_t x) { return std::to_string(x); };
  auto eff = [&](size_t v) { return std::max<int64_t>(1, s.nodes[v].cycles); };
  auto wreq = [&](size_t v) { return std::max(1, s.nodes[v].warps_required); };
  // expand_solution (sim.cpp:57-77): copy c of v issues at M(v) + c I
  std::vector<std::vector<int64_t>> issue(n, std::vector<int64_t>(static_cast<size_t>(copies), -1));
  std::vector<std::vector<std::vector<char>>> op(n);
  for (size_t v = 0; v < n; ++v) {
    op[v].assign(static_cast<size_t>(copies), std::vector<char>(static_cast<size_t>(horizon), 0));
    for (int64_t c = 0; c < copies; ++c) {
      const int64_t t = s.m[v] + c * ii;
      if (t >= 0 && t < horizon) {
        op[v][static_cast<size_t>(c)][static_cast<size_t>(t)] = 1;
        issue[v][static_cast<size_t>(c)] = t;
      }
    }
  }
  // compute_live_tables (sim.cpp:29-55): backward fixed point
  std::vector<std::vector<std::vector<char>>> live(n);
  for (size_t v = 0; v < n; ++v) {
    bool carries = false;
    for (const LEdge& e : s.edges)
      if (e.src == static_cast<int>(v) && e.delta > 0) carries = true;
    live[v].assign(static_cast<size_t>(copies), std::vector<char>(static_cast<size_t>(horizon) + 1, 0));
    for (int64_t c = 0; c < copies; ++c) {
      auto& lv = live[v][static_cast<size_t>(c)];
      lv[static_cast<size_t>(horizon)] = carries && c == copies - 1;
      for (int64_t t = horizon; t >= 1; --t) {
        const bool op_t = t < horizon && op[v][static_cast<size_t>(c)][static_cast<size_t>(t)];
        bool use_t = false;
        if (t < horizon)
          for (const LEdge& e : s.edges) {
            if (e.src != static_cast<int>(v)) continue;
            const int64_t cc = c + e.delta;
            if (cc < copies && op[static_cast<size_t>(e.dst)][static_cast<size_t>(cc)][static_cast<size_t>(t)])
              use_t = true;
          }
        lv[static_cast<size_t>(t) - 1] = lv[static_cast<size_t>(t)] ? !op_t : use_t;
      }
    }
  }
  for (size_t v = 0; v < n; ++v)
    for (int64_t c = 0; c < copies; ++c) {
      const int64_t t = issue[v][static_cast<size_t>(c)];
      if (t < 0) {
        out.push_back({"uniqueness", "node " + s.nodes[v].id + " copy " + fmt(c) + " issues 0 times"});
        continue;
      }
      const int64_t lo = c * ii, hi = c * ii + len - eff(v);
      if (t < lo || t > hi)
        out.push_back({"completion", "node " + s.nodes[v].id + " copy " + fmt(c) + " issues at " + fmt(t) +
                                         " outside [" + fmt(lo) + ", " + fmt(hi) + "]"});
    }
  for (const LEdge& e : s.edges)
    for (int64_t c = 0; c + e.delta < copies; ++c) {
      const int64_t tu = issue[static_cast<size_t>(e.src)][static_cast<size_t>(c)];
      const int64_t tv = issue[static_cast<size_t>(e.dst)][static_cast<size_t>(c + e.delta)];
      if (tu < 0 || tv < 0) continue;
      if (tv < tu + e.d)
        out.push_back({"dependence", "edge " + s.nodes[static_cast<size_t>(e.src)].id + "->" +
                                         s.nodes[static_cast<size_t>(e.dst)].id + ": consumer copy " +
                                         fmt(c + e.delta) + " at " + fmt(tv) + " before " + fmt(tu) + "+" + fmt(e.d)});
    }
  // unit capacity over the whole horizon
  std::vector<std::vector<int64_t>> occ(static_cast<size_t>(horizon), std::vector<int64_t>(s.units.size(), 0));
  for (size_t v = 0; v < n; ++v)
    for (int64_t c = 0; c < copies; ++c) {
      const int64_t t = issue[v][static_cast<size_t>(c)];
      if (t < 0) continue;
      for (size_t f = 0; f < s.nodes[v].rrt.size() && f < s.units.size(); ++f)
        for (size_t cyc = 0; cyc < s.nodes[v].rrt[f].size(); ++cyc)
          if (t + static_cast<int64_t>(cyc) < horizon) occ[static_cast<size_t>(t) + cyc][f] += s.nodes[v].rrt[f][cyc];
    }
  for (int64_t t = 0; t < horizon; ++t)
    for (size_t f = 0; f < s.units.size(); ++f)
      if (occ[static_cast<size_t>(t)][f] > s.units[f].capacity)
        out.push_back({"capacity", "unit " + s.units[f].name + " oversubscribed at cycle " + fmt(t) + ": " +
                                       fmt(occ[static_cast<size_t>(t)][f]) + " > " + fmt(s.units[f].capacity)});
  // memory footprints of live values
  for (size_t mem = 0; mem < s.memories.size(); ++mem)
    for (int64_t t = 0; t <= horizon; ++t) {
      int64_t used = 0;
      for (size_t v = 0; v < n; ++v) {
        if (mem >= s.nodes[v].footprint.size()) continue;
        for (int64_t c = 0; c < copies; ++c)
          if (live[v][static_cast<size_t>(c)][static_cast<size_t>(t)]) used += s.nodes[v].footprint[mem];
      }
      if (used > s.memories[mem].capacity)
        out.push_back({"memory", "memory " + s.memories[mem].name + " oversubscribed at cycle " + fmt(t) + ": " +
                                     fmt(used) + " > " + fmt(s.memories[mem].capacity)});
    }
  // warp slots and the variable-latency warp
  bool any_vl = false;
  for (const LNode& nd : s.nodes) any_vl = any_vl || nd.variable_latency;
  for (size_t v = 0; v < n; ++v) {
    const int st = s.a[v], wr = wreq(v);
    if (st < 0 || st % wr != 0 || st + wr > s.num_warps) {
      out.push_back({"warp_uniqueness", "node " + s.nodes[v].id + " warp start " + fmt(st) +
                                            " is not an aligned slot of width " + fmt(wr)});
      continue;
    }
    if (!any_vl) continue;
    const bool covers_vl = st <= s.vl_warp && s.vl_warp < st + wr;
    if (s.nodes[v].variable_latency && st != s.vl_warp)
      out.push_back({"variable_latency", "node " + s.nodes[v].id + " must issue from warp " + fmt(s.vl_warp)});
    if (!s.nodes[v].variable_latency && covers_vl)
      out.push_back({"variable_latency", "node " + s.nodes[v].id + " overlaps the reserved warp " + fmt(s.vl_warp)});
  }
  // per-warp register limit over live values
  if (s.reg_limit > 0)
    for (int w = 0; w < s.num_warps; ++w)
      for (int64_t t = 0; t <= horizon; ++t) {
        int64_t used = 0;
        for (size_t v = 0; v < n; ++v) {
          if (s.nodes[v].regs <= 0 || !(s.a[v] <= w && w < s.a[v] + wreq(v))) continue;
          for (int64_t c = 0; c < copies; ++c)
            if (live[v][static_cast<size_t>(c)][static_cast<size_t>(t)]) used += s.nodes[v].regs;
        }
        if (used > s.reg_limit)
          out.push_back({"register_limit", "warp " + fmt(w) + " over the register limit at cycle " + fmt(t) + ": " +
                                               fmt(used) + " > " + fmt(s.reg_limit)});
      }
  // cross-warp transfers and blocking waits: nothing else may occupy the
  // consumer's warps at the receive / wait point
  auto overlap = [](int a, int wa, int b, int wb) { return a < b + wb && b < a + wa; };
  auto isolated = [&](size_t v, int64_t at, const std::string& family, const std::string& why) {
    for (size_t o = 0; o < n; ++o) {
      if (o == v || s.nodes[o].cycles <= 0) continue;
      if (!overlap(s.a[v], wreq(v), s.a[o], wreq(o))) continue;
      const int64_t lo = std::max<int64_t>(0, at - s.nodes[o].cycles + 1), hi = std::min(at, horizon - 1);
      for (int64_t c = 0; c < copies; ++c) {
        const int64_t to = issue[o][static_cast<size_t>(c)];
        if (to >= lo && to <= hi)
          out.push_back({family, "node " + s.nodes[o].id + " occupies the warps of " + s.nodes[v].id + " at cycle " +
                                     fmt(at) + " " + why});
      }
    }
  };
  for (const LEdge& e : s.edges) {
    if (e.src == e.dst) continue;
    const size_t u = static_cast<size_t>(e.src), v = static_cast<size_t>(e.dst);
    const bool cross = s.a[u] != s.a[v] || wreq(u) != wreq(v);
    const int64_t spill = s.nodes[u].spill_cost;
    if (cross && spill > 0) {
      for (int64_t c = 0; c + e.delta < copies; ++c) {
        const int64_t tu = issue[u][static_cast<size_t>(c)], tv = issue[v][static_cast<size_t>(c + e.delta)];
        if (tu < 0 || tv < 0) continue;
        if (tv >= tu + e.d && tv < tu + e.d + spill)
          out.push_back({"spill", "edge " + s.nodes[u].id + "->" + s.nodes[v].id + ": consumer copy " +
                                      fmt(c + e.delta) + " at " + fmt(tv) + " inside the transfer window [" +
                                      fmt(tu + e.d) + ", " + fmt(tu + e.d + spill) + ")"});
      }
      for (int64_t c = 0; c + e.delta < copies; ++c) {
        const int64_t tu = issue[u][static_cast<size_t>(c)];
        if (tu < 0) continue;
        const int64_t recv = tu + e.d + spill - 1;
        if (recv >= horizon) continue;
        isolated(v, recv, "spill_sync", "(transfer receive point)");
      }
    }
    if (e.blocking)
      for (int64_t c = 0; c + e.delta < copies; ++c) {
        const int64_t tv = issue[v][static_cast<size_t>(c + e.delta)];
        if (tv < 0) continue;
        isolated(v, tv, "concurrency", "(blocked on " + s.nodes[u].id + ")");
      }
  }
  return out;
}

std::string describe(const LoweredSchedule& s) {
  json j;
  const TwfaDevicePlan& p = s.plan;
  j["family"] = p.family == TWFA_FAMILY_FA_FWD ? "fa_fwd" : p.family == TWFA_FAMILY_FA_BWD ? "fa_bwd" : "gemm";
  j["I"] = s.ii;
  j["L"] = s.length;
  j["copies"] = s.copies;
  j["max_stage"] = p.max_stage;
  j["num_warps"] = s.num_warps;
  j["load_warp"] = p.load_warp;
  json nodes = json::object();
  for (size_t v = 0; v < s.nodes.size(); ++v) {
    json o;
    o["M"] = s.m[v];
    o["stage"] = s.stage[v];
    o["slot"] = s.slot[v];
    o["warp_start"] = s.a[v];
    o["warp_count"] = std::max(1, s.nodes[v].warps_required);
    nodes[s.nodes[v].id] = o;
  }
  j["nodes"] = nodes;
  json progs = json::object();
  for (size_t w = 0; w < s.warp_prog.size(); ++w) {
    if (s.warp_prog[w].empty()) continue;
    json arr = json::array();
    for (int v : s.warp_prog[w]) arr.push_back(s.nodes[static_cast<size_t>(v)].id);
    progs[std::to_string(w)] = arr;
  }
  j["warp_programs"] = progs;
  json rings = json::object();
  if (p.family == TWFA_FAMILY_FA_FWD) {
    rings["K"] = p.k_depth;
    rings["S"] = p.s_depth;
    j["kv_tile"] = p.kv_tile;
    j["s_split"] = p.s_split;
    rings["V"] = p.v_depth;
    j["prefetch"] = {{"LDK", p.k_prefetch}, {"LDV", p.v_prefetch}};
    j["num_tiles"] = p.num_tiles;
    json roles = json::object();
    for (int k = 0; k < p.num_tiles; ++k) {
      roles["softmax" + std::to_string(k)] = p.sm_warp[k];
      roles["correction" + std::to_string(k)] = p.cr_warp[k];
    }
    j["warpgroups"] = roles;
    json inorder = json::array();
    for (int v = 0; v < p.num_nodes; ++v)
      if (p.ops[v].flags & TWFA_OPF_INORDER) inorder.push_back(s.nodes[static_cast<size_t>(v)].id);
    j["inorder_tc_issue"] = inorder;
    json fused = json::array();
    for (int v = 0; v < p.num_nodes; ++v)
      if (p.ops[v].flags & TWFA_OPF_FUSE_NEXT) fused.push_back(s.nodes[static_cast<size_t>(v)].id);
    j["register_resident_softmax"] = fused;
    json ring = json::array();
    for (int i = 0; i < p.ex_ring_len; ++i) ring.push_back("EX" + std::to_string(p.ex_ring[i]));
    j["mufu_order"] = ring;
    j["q_warp"] = p.q_warp;
  } else if (p.family == TWFA_FAMILY_FA_BWD) {
    rings["Q"] = p.k_depth;
    rings["dO"] = p.v_depth;
    j["prefetch"] = {{"LDQ", p.k_prefetch}, {"LDO", p.v_prefetch}};
    j["mma_warp"] = p.mma_warp;
    j["num_tiles"] = p.num_tiles;
    if (p.num_tiles == 2) {  // two 64-query sub-tiles (fa_bwd_pp_sm100.cu)
      j["warpgroups"] = {{"exp_ds0", p.sm_warp[0]}, {"exp_ds1", p.sm_warp[1]},
                         {"dq_reduce0", p.cr_warp[0]}, {"dq_reduce1", p.cr_warp[1]}};
      j["p_transfer"] = "registers (EXB_k and DS_k fused)";
    } else {
      j["warpgroups"] = {{"exp", p.sm_warp[0]}, {"ds", p.sm_warp[1]}, {"dq_reduce", p.cr_warp[0]}};
      j["p_transfer"] =
          p.sm_warp[0] == p.sm_warp[1] ? "registers (EXB and DS fused)" : "tensor memory (bf16 P^T re-read)";
    }
    json rel = json::array();
    for (int v = 0; v < p.num_nodes; ++v)
      if (p.ops[v].flags & TWFA_OPF_RELEASE) rel.push_back(s.nodes[static_cast<size_t>(v)].id);
    j["ring_release"] = rel;
    if (p.num_tiles == 2) {
      j["dq_staging"] = "dS_k buffer, transposed, two 64-dim passes";
      j["tmem_columns"] = {{"dK", 0},           {"dV", 128},           {"S^T_0/P^T_0/dQ^T_0", 256},
                           {"dP^T_0/dS^T_0", 320}, {"S^T_1/P^T_1/dQ^T_1", 384}, {"dP^T_1/dS^T_1", 448}};
    } else {
      j["dq_staging"] = p.s_split ? "Q ring slot" : "dS buffer";
      j["tmem_columns"] = {{"dK", 0}, {"dV", 128}, {"S^T/P^T/dQ", 256}, {"dP^T/dS^T", 384}};
    }
  } else {
    rings["AB"] = p.k_depth;
    j["mma_warp"] = p.mma_warp;
  }
  j["rings"] = rings;
  return j.dump();
}

}  // namespace twfa
