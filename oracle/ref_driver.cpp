// Test-infrastructure driver for the reference build (oracle/_ref). It links the
// UNMODIFIED reference library (libkronred_ref.a, built by oracle/Makefile from
// /root/reference/proj/src) and calls only its public API. It never enters the
// product path: it generates golden inputs/outputs for tests/golden and times
// the reference CPU arm for bench.py --impl reference.
//
// Subcommands
//   gen    --n N --seed S --L L [--preset acceptance|default] [--branching b]
//          [--frac2 x] [--frac1 y] --net out.json --scen out.csv [--pq out_pq.csv]
//          Writes the network JSON (reference writer, io.cpp:138-166) and a
//          constant-current scenario CSV (17 significant digits) whose reload
//          reproduces the generated library bit-for-bit (scenario.cpp:39-50).
//   reduce --net f --scen f [--e-bar E] [--objective mag|complex] [--target T]
//          [--workers W] [--radialize] [--reduced out.json] [--trace out.csv]
//          [--trace-hex out.txt] [--validate report.csv [--bins k]]
//          Runs kronred::run_reduction (reduce.cpp:349-451) and prints one JSON
//          summary line (wall, iterations, candidates, cand/s).
//   scores --net f --scen f [--e-bar E] [--objective ...] --iters K --out f
//          Per-candidate delta-path scores of the first K iterations
//          (reduce.cpp:194-244), bit patterns in hex.
//   solve  --net f --scen f --out f     v0, every unit-injection column, V-hat.
//   kron   --net f --reduce list.txt --out f   kron_reduce (kron.cpp:34-46).
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "kronred/feeder_gen.hpp"
#include "kronred/grid_model.hpp"
#include "kronred/io.hpp"
#include "kronred/kron.hpp"
#include "kronred/radialize.hpp"
#include "kronred/reduce.hpp"
#include "kronred/solver.hpp"

using namespace kronred;

namespace {

std::map<std::string, std::string> parse_args(int argc, char** argv, int first) {
  std::map<std::string, std::string> a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) continue;
    k = k.substr(2);
    if (i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0)
      a[k] = argv[++i];
    else
      a[k] = "1";
  }
  return a;
}

std::string hx(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  char buf[20];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, u);
  return buf;
}

double getd(const std::map<std::string, std::string>& a, const char* k, double d) {
  auto it = a.find(k);
  return it == a.end() ? d : std::strtod(it->second.c_str(), nullptr);
}
long getl(const std::map<std::string, std::string>& a, const char* k, long d) {
  auto it = a.find(k);
  return it == a.end() ? d : std::strtol(it->second.c_str(), nullptr, 10);
}
std::string gets(const std::map<std::string, std::string>& a, const char* k,
                 const std::string& d) {
  auto it = a.find(k);
  return it == a.end() ? d : it->second;
}

void write_current_csv(const std::string& path, const ScenarioLibrary& lib) {
  std::ofstream out(path);
  out << "scenario_id,node_id,phase,i_re,i_im\n";
  for (const Scenario& sc : lib.scenarios) {
    for (size_t k = 0; k < sc.injections.size(); ++k) {
      const cx z = sc.injections[k];
      if (z == cx{}) continue;
      out << sc.id << "," << k / 3 << "," << char('a' + int(k % 3)) << ","
          << format_double(z.real()) << "," << format_double(z.imag()) << "\n";
    }
  }
}

int cmd_gen(const std::map<std::string, std::string>& a) {
  GenParams p;
  if (gets(a, "preset", "default") == "acceptance") {
    // acceptance_main.cpp:56-66 (thousand_node_params)
    p.branching = 0.3;
    p.self_r_min = 0.0016;
    p.self_r_max = 0.0120;
    p.load_p_min = 0.15e-3;
    p.load_p_max = 1.00e-3;
  }
  p.n = int(getl(a, "n", 100));
  p.seed = std::uint64_t(getl(a, "seed", 1));
  p.scenario_count = int(getl(a, "L", 2));
  if (a.count("branching")) p.branching = getd(a, "branching", p.branching);
  if (a.count("frac2")) p.frac_two_phase = getd(a, "frac2", p.frac_two_phase);
  if (a.count("frac1")) p.frac_single_phase = getd(a, "frac1", p.frac_single_phase);
  if (a.count("spread")) p.scenario_spread = getd(a, "spread", p.scenario_spread);
  GeneratedLoads loads;
  auto [net, lib] = generate(p, loads);
  write_network_json(net, gets(a, "net", "net.json"));
  write_current_csv(gets(a, "scen", "scen.csv"), lib);
  if (a.count("pq")) write_scenario_csv(gets(a, "pq", ""), loads);
  // round-trip check: reload and compare V-hat bitwise
  const Network net2 = read_network_json(gets(a, "net", "net.json"));
  const ScenarioLibrary lib2 = load_library(net2, gets(a, "scen", "scen.csv"));
  bool same = lib2.scenarios.size() == lib.scenarios.size();
  for (size_t l = 0; same && l < lib.scenarios.size(); ++l)
    same = std::memcmp(lib.scenarios[l].voltages.data(), lib2.scenarios[l].voltages.data(),
                       lib.scenarios[l].voltages.size() * sizeof(cx)) == 0;
  std::printf("{\"n\": %d, \"L\": %d, \"roundtrip_bitwise\": %s}\n", net.size(),
              p.scenario_count, same ? "true" : "false");
  return same ? 0 : 1;
}

ReductionConfig make_cfg(const std::map<std::string, std::string>& a) {
  ReductionConfig cfg;
  cfg.e_bar = getd(a, "e-bar", 1e-3);
  cfg.objective = gets(a, "objective", "mag") == "complex" ? Objective::complex_error
                                                            : Objective::magnitude;
  if (a.count("target")) cfg.target_reduction = getd(a, "target", 1.0);
  if (a.count("use-delta")) cfg.use_delta = getl(a, "use-delta", 1) != 0;  // 0: eval_full_solve path
  long w = getl(a, "workers", 1);
  if (w <= 0) w = long(std::thread::hardware_concurrency());
  cfg.workers = int(w);
  return cfg;
}

int cmd_reduce(const std::map<std::string, std::string>& a) {
  const Network net = read_network_json(gets(a, "net", ""));
  const ScenarioLibrary lib = load_library(net, gets(a, "scen", ""));
  const ReductionConfig cfg = make_cfg(a);
  long long cands = 0;
  // --trace-hex rows are streamed from the observer (one flushed line per
  // commit, reduce.cpp:423) so a long golden run leaves a usable prefix even
  // if it is stopped; the `final` line is appended after the run.
  std::ofstream hexout;
  if (a.count("trace-hex")) hexout.open(gets(a, "trace-hex", ""));
  const auto t0 = std::chrono::steady_clock::now();
  ReductionResult res = run_reduction(net, lib, cfg, [&](const AssignmentState&, const TraceRow& r) {
    cands += r.candidate_count;
    if (hexout.is_open()) {
      hexout << r.iteration << " " << r.s << " " << r.r << " " << hx(r.smice);
      for (double e : r.max_err) hexout << " " << hx(e);
      hexout << " " << r.supernode_count << " " << r.candidate_count << "\n";
      hexout.flush();
    }
  });
  const auto t1 = std::chrono::steady_clock::now();
  ReducedModel model = std::move(res.model);
  if (a.count("radialize")) {
    const BlockAdmittance y = assemble_admittance(net);
    model = radialize(model, net, y, &lib);
  }
  const double wall = std::chrono::duration<double>(t1 - t0).count();
  if (a.count("reduced")) write_reduced_json(model, gets(a, "reduced", ""));
  if (a.count("validate"))  // io.cpp:385-416 on the model just reduced
    write_validate_report(make_validate_report(model, net, lib, int(getl(a, "bins", 20))), gets(a, "validate", ""));
  if (a.count("trace")) {
    // wall_ms is nondeterministic; zero it so the file is a stable golden
    std::vector<TraceRow> tr = res.trace;
    for (TraceRow& r : tr) r.wall_ms = 0;
    write_trace_csv(gets(a, "trace", ""), tr, model.scenario_ids, model.final_max_err);
  }
  if (hexout.is_open()) {
    hexout << "final";
    for (double e : model.final_max_err) hexout << " " << hx(e);
    hexout << "\n";
  }
  std::printf(
      "{\"wall_s\": %.6f, \"iterations\": %zu, \"candidates\": %lld, \"cand_per_s\": %.3f, "
      "\"kept\": %zu, \"n\": %d, \"workers\": %d}\n",
      wall, res.trace.size(), cands, wall > 0 ? double(cands) / wall : 0.0,
      model.kept_ids.size(), net.size(), cfg.workers);
  return 0;
}

int cmd_scores(const std::map<std::string, std::string>& a) {
  const Network net = read_network_json(gets(a, "net", ""));
  const ScenarioLibrary lib = load_library(net, gets(a, "scen", ""));
  const ReductionConfig cfg = make_cfg(a);
  const int iters = int(getl(a, "iters", 1));
  const BlockAdmittance y = assemble_admittance(net);
  const auto masks = phase_masks(net);
  const AnchoredSolver solver(y, masks, net.slack_id(),
                              net.nodes[size_t(net.slack_id())].slack_voltage);
  AssignmentState st = init_state(net, lib);
  DeltaCache cache(lib, solver);
  cache.refresh_base(st);
  std::ofstream out(gets(a, "out", "scores.txt"));
  for (int it = 1; it <= iters; ++it) {
    const auto cands = enumerate_candidates(st, net);
    if (cands.empty()) break;
    for (const Candidate& c : cands) {
      cache.ensure_columns(c.s);
      cache.ensure_columns(c.r);
    }
    int best = -1;
    std::vector<CandidateScore> sc(cands.size());
    for (size_t i = 0; i < cands.size(); ++i) {
      sc[i] = evaluate_candidate_delta(st, cands[i], cache, cfg);
      out << it << " " << cands[i].s << " " << cands[i].r << " " << (sc[i].feasible ? 1 : 0)
          << " " << hx(sc[i].smice);
      for (double e : sc[i].max_err) out << " " << hx(e);
      out << "\n";
      if (sc[i].feasible && (best < 0 || sc[i].smice < sc[size_t(best)].smice)) best = int(i);
    }
    if (best < 0) break;
    commit(st, cands[size_t(best)]);
    cache.evict_columns(cands[size_t(best)].r);
    cache.refresh_base(st);
  }
  return 0;
}

int cmd_solve(const std::map<std::string, std::string>& a) {
  const Network net = read_network_json(gets(a, "net", ""));
  const ScenarioLibrary lib = load_library(net, gets(a, "scen", ""));
  const BlockAdmittance y = assemble_admittance(net);
  const auto masks = phase_masks(net);
  const AnchoredSolver solver(y, masks, net.slack_id(),
                              net.nodes[size_t(net.slack_id())].slack_voltage);
  std::ofstream out(gets(a, "out", "solve.txt"));
  auto dump = [&](const std::string& tag, const std::vector<cx>& v) {
    out << tag;
    for (const cx& z : v) out << " " << hx(z.real()) << " " << hx(z.imag());
    out << "\n";
  };
  dump("v0", solver.zero_injection_solution());
  for (size_t l = 0; l < lib.scenarios.size(); ++l) dump("vhat" + std::to_string(l), lib.scenarios[l].voltages);
  const int n = net.size();
  std::vector<cx> unit(size_t(3 * n), cx{});
  for (int k = 0; k < n; ++k)
    for (int p = 0; p < 3; ++p) {
      if (!masks[size_t(k)].has(p)) continue;
      unit[size_t(3 * k + p)] = cx{1.0, 0.0};
      dump("e" + std::to_string(3 * k + p), solver.solve(unit));
      unit[size_t(3 * k + p)] = cx{};
    }
  return 0;
}

int cmd_kron(const std::map<std::string, std::string>& a) {
  const Network net = read_network_json(gets(a, "net", ""));
  const BlockAdmittance y = assemble_admittance(net);
  const auto masks = phase_masks(net);
  std::ifstream in(gets(a, "reduce", ""));
  Partition part;
  std::set<int> red;
  int v;
  while (in >> v) red.insert(v);
  part.reduce.assign(red.begin(), red.end());
  for (int i = 0; i < net.size(); ++i)
    if (!red.count(i)) part.keep.push_back(i);
  const KronResult kr = kron_reduce(y, masks, part);
  std::ofstream out(gets(a, "out", "kron.txt"));
  for (int i = 0; i < kr.y_kron.n(); ++i)
    for (const auto& [j, blk] : kr.y_kron.row(i)) {
      out << kr.kept_ids[size_t(i)] << " " << kr.kept_ids[size_t(j)];
      for (const cx& z : blk.m) out << " " << hx(z.real()) << " " << hx(z.imag());
      out << "\n";
    }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: kronred_ref gen|reduce|scores|solve|kron [--flags]\n");
    return 2;
  }
  const std::string cmd = argv[1];
  const auto a = parse_args(argc, argv, 2);
  try {
    if (cmd == "gen") return cmd_gen(a);
    if (cmd == "reduce") return cmd_reduce(a);
    if (cmd == "scores") return cmd_scores(a);
    if (cmd == "solve") return cmd_solve(a);
    if (cmd == "kron") return cmd_kron(a);
  } catch (const SolverError& e) {
    std::fprintf(stderr, "SolverError: %s\n", e.what());
    return 3;
  } catch (const ValidationError& e) {
    std::fprintf(stderr, "ValidationError: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
