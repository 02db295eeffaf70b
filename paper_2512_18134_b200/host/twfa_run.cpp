// twfa-run: C++ host driver over the C ABI (include/twfa.h).
//
// This is the "existing C++ host" side of the boundary: a CPU
// program that takes the two documents `weftsched joint` exchanges (problem
// JSON, solution JSON; cli.cpp:68-94) and runs the schedule on the GPU
// through libtwfa, with host buffers. It mirrors the reference CLI's
// conventions (cli.cpp:376-473): subcommands, errors on stderr, exit code
// 0 ok / 1 domain error / 2 usage error (+3 CUDA error, the executor's own).
//
//   twfa-run describe <problem.json> <solution.json>
//   twfa-run fa <problem.json> <solution.json> [--B n] [--H n] [--S n]
//            [--causal] [--iters n] [--seed n]
//
// `fa` fills Q, K, V with a seeded N(0,1) (rounded to bf16), runs
// twfa_fa_fwd_host (host -> device copies, kernel, device -> host) `iters`
// times and prints one JSON line with the wall time per call, the TFLOP/s of
// that end-to-end call and an O checksum.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "twfa.h"

namespace {

int usage(const char* msg) {
  std::fprintf(stderr,
               "error: %s\nusage: twfa-run describe <problem.json> <solution.json>\n"
               "       twfa-run fa <problem.json> <solution.json> [--B n] [--H n] [--S n] [--causal] "
               "[--iters n] [--seed n]\n",
               msg);
  return TWFA_EUSAGE;
}

bool slurp(const char* path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::stringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return true;
}

uint16_t to_bf16(float x) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

float from_bf16(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

int fail(int rc) {
  std::fprintf(stderr, "error: %s\n", twfa_last_error());
  return rc;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) return usage("missing arguments");
  const std::string cmd = argv[1];
  if (cmd != "describe" && cmd != "fa") return usage("unknown subcommand");
  std::string prob, sol;
  if (!slurp(argv[2], prob)) return usage("cannot read problem file");
  if (!slurp(argv[3], sol)) return usage("cannot read solution file");
  int B = 1, H = 2, S = 512, iters = 3, causal = 0;
  unsigned seed = 7;
  for (int i = 4; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&](int& dst) {
      if (i + 1 >= argc) return false;
      char* end = nullptr;
      long v = std::strtol(argv[++i], &end, 10);
      if (*end != '\0' || v < 1 || v > (1L << 30)) return false;
      dst = static_cast<int>(v);
      return true;
    };
    int tmp = 0;
    if (a == "--B") { if (!next(B)) return usage("--B needs a positive integer"); }
    else if (a == "--H") { if (!next(H)) return usage("--H needs a positive integer"); }
    else if (a == "--S") { if (!next(S)) return usage("--S needs a positive integer"); }
    else if (a == "--iters") { if (!next(iters)) return usage("--iters needs a positive integer"); }
    else if (a == "--seed") { if (!next(tmp)) return usage("--seed needs a positive integer"); seed = tmp; }
    else if (a == "--causal") causal = 1;
    else return usage(("unknown option " + a).c_str());
  }

  twfa_plan* plan = nullptr;
  int rc = twfa_plan_create(prob.c_str(), sol.c_str(), &plan);
  if (rc != TWFA_OK) return fail(rc);
  if (cmd == "describe") {
    size_t need = 0;
    twfa_plan_describe(plan, nullptr, 0, &need);
    std::vector<char> buf(need);
    rc = twfa_plan_describe(plan, buf.data(), buf.size(), &need);
    if (rc != TWFA_OK) return fail(rc);
    std::printf("%s\n", buf.data());
    twfa_plan_destroy(plan);
    return TWFA_OK;
  }

  const int D = 128;
  const size_t n = static_cast<size_t>(B) * H * S * D;
  std::vector<uint16_t> q(n), k(n), v(n), o(n);
  std::vector<float> lse(static_cast<size_t>(B) * H * S);
  std::mt19937 gen(seed);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (auto* t : {&q, &k, &v})
    for (auto& x : *t) x = to_bf16(nd(gen));
  const float scale = 1.0f / std::sqrt(static_cast<float>(D));
  double best = 1e30;
  for (int it = 0; it < iters; ++it) {
    auto t0 = std::chrono::steady_clock::now();
    rc = twfa_fa_fwd_host(plan, q.data(), k.data(), v.data(), o.data(), lse.data(), B, H, S, D, causal, scale);
    auto t1 = std::chrono::steady_clock::now();
    if (rc != TWFA_OK) {
      twfa_plan_destroy(plan);
      return fail(rc);
    }
    if (it > 0 || iters == 1) best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
  }
  double sum = 0.0, lsum = 0.0;
  for (uint16_t x : o) sum += from_bf16(x);
  for (float x : lse) lsum += x;
  const double flops = 4.0 * B * H * static_cast<double>(S) * S * D / (causal ? 2.0 : 1.0);
  std::printf("{\"B\": %d, \"H\": %d, \"S\": %d, \"d\": %d, \"causal\": %d, \"seconds_per_call\": %.6f, "
              "\"e2e_tflops\": %.3f, \"o_sum\": %.6f, \"lse_sum\": %.6f}\n",
              B, H, S, D, causal, best, flops / best / 1e12, sum, lsum);
  twfa_plan_destroy(plan);
  return TWFA_OK;
}
