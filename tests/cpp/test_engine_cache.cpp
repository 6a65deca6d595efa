// kronred::run_reduction's per-thread engine cache (capi.cpp): a second call
// on the same network reuses the resident engine and must give the same bits
// as the first; a call with other values of the same structure (the scenario
// library permuted) must give exactly what an uncached engine gives; a
// different network must not hit the cache. Prints cold / warm call times.
//
// usage: test_engine_cache net.json scen.csv other_net.json other_scen.csv e_bar
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "kronred_b200.hpp"

using namespace kronred;

static bool same(const ReductionResult& a, const ReductionResult& b) {
  if (a.trace.size() != b.trace.size()) return false;
  for (size_t i = 0; i < a.trace.size(); ++i) {
    const TraceRow &x = a.trace[i], &y = b.trace[i];
    if (x.s != y.s || x.r != y.r || std::memcmp(&x.smice, &y.smice, 8) != 0 || x.max_err != y.max_err) return false;
  }
  return reduced_json_string(a.model) == reduced_json_string(b.model);
}

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const Network net = read_network_json(argv[1]);
  const ScenarioLibrary lib = load_library(net, argv[2]);
  const Network net2 = read_network_json(argv[3]);
  const ScenarioLibrary lib2 = load_library(net2, argv[4]);
  ReductionConfig cfg;
  cfg.e_bar = std::strtod(argv[5], nullptr);
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  release_engine_cache();
  auto t0 = clk::now();
  const ReductionResult a = run_reduction(net, lib, cfg);
  const double cold = ms(t0);
  t0 = clk::now();
  const ReductionResult b = run_reduction(net, lib, cfg);
  const double warm = ms(t0);
  int bad = 0;
  if (!same(a, b)) {
    std::printf("FAIL: cached second call differs\n");
    ++bad;
  }
  // same structure, other values: scenarios in reverse order
  ScenarioLibrary rev = lib;
  std::reverse(rev.scenarios.begin(), rev.scenarios.end());
  const ReductionResult c = run_reduction(net, rev, cfg);
  setenv("KRONRED_ENGINE_CACHE", "0", 1);
  const ReductionResult d = run_reduction(net, rev, cfg);
  unsetenv("KRONRED_ENGINE_CACHE");
  if (!same(c, d)) {
    std::printf("FAIL: cached engine with new values differs from a fresh engine\n");
    ++bad;
  }
  // another network (different structure), then back
  const ReductionResult e = run_reduction(net2, lib2, cfg);
  setenv("KRONRED_ENGINE_CACHE", "0", 1);
  const ReductionResult f = run_reduction(net2, lib2, cfg);
  unsetenv("KRONRED_ENGINE_CACHE");
  if (!same(e, f)) {
    std::printf("FAIL: structure change\n");
    ++bad;
  }
  const ReductionResult g = run_reduction(net, lib, cfg);
  if (!same(a, g)) {
    std::printf("FAIL: back to the first network\n");
    ++bad;
  }
  release_engine_cache();
  std::printf("cold_call_ms %.2f warm_call_ms %.2f iterations %zu failures %d\n", cold, warm, a.trace.size(), bad);
  return bad == 0 ? 0 : 1;
}
