// Schedule -> kernel lowering (host side).
//
// Input: the two documents the reference exchanges on disk -- the problem
// JSON (/root/reference/proj/src/ir.cpp:93-229) and the solution JSON
// written by `weftsched joint` (solution_to_json, cli.cpp:68-94). Output: a
// TwfaDevicePlan the sm_100a kernels execute.
//
// The reference's own consumer of a solution is `synthesize`
// (codegen.cpp:43-189) which renders text; this lowering is the B200
// consumer in the same position. It reproduces the reference's reading of a
// solution file exactly (solution_from_json + reconstruct, cli.cpp:96-168:
// unknown keys rejected, M must cover every node and fit in [0, L - eff],
// the streaming rewrite re-applied when streaming depths are present,
// jointsolve.cpp:511-524) and then derives the per-warp trip programs.
#pragma once
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "plan.h"

namespace twfa {

// Error classes mirror the reference's exit-code map (cli.hpp:11-13,
// cli.cpp:462-471): DomainError -> 1 (bad document / unrealizable
// schedule), UsageError -> 2 (bad call arguments).
struct DomainError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct LNode {
  std::string id;
  int64_t cycles = 1;        // after the streaming rewrite (0 for streamed loads)
  int warps_required = 1;
  bool variable_latency = false;
  int64_t spill_cost = 0;
  int64_t regs = 0;
  std::vector<std::vector<int64_t>> rrt;  // [unit][cycle], dense (empty rows once streamed)
  std::vector<int64_t> footprint;         // by memory index, dense
};

struct LResource {
  std::string name;
  int64_t capacity = 0;
};

struct LEdge {
  int src = 0, dst = 0;
  int64_t d = 0;
  int delta = 0;
  bool blocking = false;
};

struct LoweredSchedule {
  // problem
  std::vector<LNode> nodes;
  std::vector<LEdge> edges;
  std::vector<LResource> units, memories;
  int num_warps = 1;
  int vl_warp = 0;
  int64_t reg_limit = 0;
  // solution
  int64_t ii = 1, length = 1, copies = 1;
  std::vector<int64_t> m;      // M by node
  std::vector<int> a;          // A by node
  std::map<std::string, int64_t> streaming_depths;
  // derived
  std::vector<int64_t> stage;  // M div I
  std::vector<int64_t> slot;   // M mod I
  std::vector<std::vector<int>> warp_prog;  // [warp] -> node indices in trip order
  TwfaDevicePlan plan{};
};

// One violated constraint family of the reference's checker.
struct Violation {
  std::string family, message;
};

// validate_graph (ir.cpp:231-276) restated: zero-delta cycles, RRT rows over
// a unit's capacity, warps_required over the machine.
std::vector<Violation> validate_graph(const LoweredSchedule& s);

// validate_program (sim.cpp:79-311) restated over the tables the solution
// expands to (expand_solution, sim.cpp:57-77): completion window,
// dependence, unit capacity, memory footprint of live values, aligned warp
// slots, the variable-latency warp, the per-warp register limit, spill
// windows, spill receive isolation and blocking isolation. Empty = valid.
std::vector<Violation> validate_schedule(const LoweredSchedule& s);

// Parses and lowers. Throws DomainError on malformed documents, on any
// violation validate_graph / validate_schedule report (the reference's
// checker must accept the schedule), and on schedules the B200 executor
// cannot realize.
LoweredSchedule lower(const std::string& problem_json, const std::string& solution_json);

// Parses both documents (the problem through validate_graph, the solution
// through solution_from_json + reconstruct) without validating the schedule
// or lowering it.
LoweredSchedule parse(const std::string& problem_json, const std::string& solution_json);

// validate_schedule as the JSON list [[family, message], ...] the
// reference's Python binding returns (bindings/module.cpp:176-184).
std::string violations_json(const std::vector<Violation>& v);

// JSON description of the plan: I, L, copies, per-node stage/slot/warp,
// per-warp programs, ring depths.
std::string describe(const LoweredSchedule& s);

}  // namespace twfa
