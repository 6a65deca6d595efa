// C ABI (include/kronred_b200.h) and the C++ drop-in entry points
// (include/kronred_b200.hpp): input parsing, problem construction and result
// marshalling around the device Engine. Exceptions map to status codes the way
// the reference CLI maps them to exit codes (main.cpp:234-246).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>

#include "kr_internal.hpp"

using namespace kronred;
using namespace kronred::b200;

namespace kronred {
Network parse_network_text(const std::string& text);
}

namespace {

thread_local std::string g_err;
thread_local double g_pivot = 0.0;
thread_local int g_node = -1;

}  // namespace

namespace kronred::b200 {

void set_error(const std::string& msg, double pivot, int node) {
  g_err = msg;
  g_pivot = pivot;
  g_node = node;
}

int status_from_current_exception() {
  try {
    throw;
  } catch (const SolverError& e) {
    set_error(e.what(), e.smallest_pivot, e.node);
    return KRG_E_SOLVER;
  } catch (const ValidationError& e) {
    set_error(e.what());
    return KRG_E_VALIDATION;
  } catch (const CudaError& e) {
    set_error(e.what());
    return KRG_E_CUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return KRG_E_INTERNAL;
  } catch (...) {
    set_error("unknown error");
    return KRG_E_INTERNAL;
  }
}

}  // namespace kronred::b200

// ---------------------------------------------------------------------------
// scenario CSV (scenario.cpp:100-212)

struct krg_host_problem {
  Network net;
  bool pq = false;
  std::vector<std::string> ids;
  std::vector<std::vector<std::pair<int, cx>>> pq_loads;
  std::vector<double> inj;  // current mode, [L][3n][2]
  // flat views
  std::vector<std::uint8_t> phases;
  std::vector<int32_t> from, to;
  std::vector<double> ys, sf, st, slackv;
  std::vector<double> pq_flat;  // [L][3n][2] summed PQ (view only)
};

struct krg_ctx {
  std::unique_ptr<Engine> eng;
};

struct krg_result {
  ResultData d;
};

namespace {

std::vector<std::string> split_fields(const std::string& line) {
  std::vector<std::string> out(1);
  for (char c : line) {
    if (c == ',')
      out.emplace_back();
    else if (c != '\r')
      out.back() += c;
  }
  for (std::string& f : out) {
    const auto b = f.find_first_not_of(" \t");
    const auto e = f.find_last_not_of(" \t");
    f = b == std::string::npos ? std::string() : f.substr(b, e - b + 1);
  }
  return out;
}

double parse_number(const std::string& s, const std::string& ctx) {
  try {
    size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw ValidationError(ctx + ": bad number '" + s + "'");
  }
}

void parse_scenarios(krg_host_problem& hp, const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open scenario file '" + path + "'");
  std::string line, header;
  int lineno = 0;
  bool have = false;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    header = line;
    have = true;
    break;
  }
  if (!have) return;  // empty library; rejected when a run starts
  const auto hf = split_fields(header);
  if (hf == std::vector<std::string>{"scenario_id", "node_id", "phase", "p_pu", "q_pu"})
    hp.pq = true;
  else if (hf == std::vector<std::string>{"scenario_id", "node_id", "phase", "i_re", "i_im"})
    hp.pq = false;
  else
    throw ValidationError("scenario file '" + path + "': unrecognized header '" + header + "'");
  const int n = hp.net.size();
  std::map<std::string, size_t> group;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty() || line[0] == '#') continue;
    const std::string ctx = path + ":" + std::to_string(lineno);
    const auto f = split_fields(line);
    if (f.size() != 5) throw ValidationError(ctx + ": expected 5 columns, got " + std::to_string(f.size()));
    auto [it, fresh] = group.try_emplace(f[0], hp.ids.size());
    if (fresh) {
      hp.ids.push_back(f[0]);
      hp.pq_loads.emplace_back();
      hp.inj.resize(hp.inj.size() + size_t(6 * n), 0.0);
    }
    const size_t g = it->second;
    const int node = int(parse_number(f[1], ctx));
    int phase = -1;
    if (f[2] == "a") phase = 0;
    if (f[2] == "b") phase = 1;
    if (f[2] == "c") phase = 2;
    if (phase < 0) throw ValidationError(ctx + ": bad phase '" + f[2] + "' (want a|b|c)");
    if (node < 0 || node >= n) throw ValidationError(ctx + ": unknown node " + f[1]);
    if (!hp.net.nodes[size_t(node)].phases.has(phase))
      throw ValidationError(ctx + ": phase " + f[2] + " absent at node " + f[1]);
    const double x0 = parse_number(f[3], ctx), x1 = parse_number(f[4], ctx);
    if (hp.pq) {
      hp.pq_loads[g].push_back({3 * node + phase, cx{x0, x1}});
    } else {
      double* z = &hp.inj[g * size_t(6 * n) + size_t(3 * node + phase) * 2];
      const cx sum = cx{z[0], z[1]} + cx{x0, x1};
      z[0] = sum.real();
      z[1] = sum.imag();
    }
  }
}

void fill_views(krg_host_problem& hp) {
  const Network& net = hp.net;
  hp.phases.clear();
  for (const Node& nd : net.nodes) hp.phases.push_back(nd.phases.bits);
  hp.slackv.assign(6, 0.0);
  const int sl = net.slack_id();
  if (sl >= 0)
    for (int p = 0; p < 3; ++p) {
      hp.slackv[size_t(2 * p)] = net.nodes[size_t(sl)].slack_voltage[p].real();
      hp.slackv[size_t(2 * p + 1)] = net.nodes[size_t(sl)].slack_voltage[p].imag();
    }
  for (const Branch& b : net.branches) {
    hp.from.push_back(b.from);
    hp.to.push_back(b.to);
    for (int k = 0; k < 9; ++k) {
      hp.ys.push_back(b.y_series.m[size_t(k)].real());
      hp.ys.push_back(b.y_series.m[size_t(k)].imag());
      hp.sf.push_back(b.shunt_from.m[size_t(k)].real());
      hp.sf.push_back(b.shunt_from.m[size_t(k)].imag());
      hp.st.push_back(b.shunt_to.m[size_t(k)].real());
      hp.st.push_back(b.shunt_to.m[size_t(k)].imag());
    }
  }
  if (hp.pq) {
    const int n = net.size();
    hp.pq_flat.assign(hp.ids.size() * size_t(6 * n), 0.0);
    for (size_t g = 0; g < hp.ids.size(); ++g)
      for (const auto& ld : hp.pq_loads[g]) {
        double* z = &hp.pq_flat[g * size_t(6 * n) + size_t(ld.first) * 2];
        const cx sum = cx{z[0], z[1]} + ld.second;
        z[0] = sum.real();
        z[1] = sum.imag();
      }
  }
}

Problem base_problem(const Network& net) {
  const bool tr = std::getenv("KRONRED_RELOAD_TRACE") != nullptr;  // tuning aid: phase times
  const auto t0 = std::chrono::steady_clock::now();
  validate_or_throw(net);
  const auto t1 = std::chrono::steady_clock::now();
  Problem p;
  p.net = net;
  for (const Node& nd : net.nodes) p.mask.push_back(nd.phases.bits);
  p.slack = net.slack_id();
  const auto t2 = std::chrono::steady_clock::now();
  const BlockAdmittance y = assemble_admittance(net);
  const auto t3 = std::chrono::steady_clock::now();
  p.y = FlatBlocks::from(y);
  if (tr) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "assembly: validate %.3f ms, copy %.3f ms, admittance %.3f ms, flatten %.3f ms\n", ms(t0, t1),
                 ms(t1, t2), ms(t2, t3), ms(t3, std::chrono::steady_clock::now()));
  }
  return p;
}

// scenario_from_currents (scenario.cpp:39-50): zero slack / absent entries
void zero_invalid(const Network& net, std::vector<double>& inj, int L) {
  const int n = net.size();
  for (int l = 0; l < L; ++l)
    for (const Node& nd : net.nodes)
      for (int p = 0; p < 3; ++p)
        if (nd.is_slack || !nd.phases.has(p)) {
          inj[(size_t(l) * 3 * n + size_t(3 * nd.id + p)) * 2] = 0.0;
          inj[(size_t(l) * 3 * n + size_t(3 * nd.id + p)) * 2 + 1] = 0.0;
        }
}

// A small pool of host worker threads, created on first use and kept for the
// process (a reload's per-scenario checks would otherwise pay a thread start
// per worker on every call). parallel_for(n, fn) runs fn(0..n-1) and returns
// when all are done; the caller works too. Concurrent callers (one host
// thread per device) take turns.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  void parallel_for(size_t n, const std::function<void(size_t)>& fn) {
    if (n == 0) return;
    std::lock_guard<std::mutex> turn(call_m_);
    if (workers_.empty() || n == 1) {
      for (size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> lk(m_);
    fn_ = &fn;
    n_ = n;
    next_ = 0;
    busy_ = workers_.size();
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    run_tasks();
    lk.lock();
    done_cv_.wait(lk, [&] { return busy_ == 0; });
    fn_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nw = std::min(15u, hw > 1 ? hw - 1 : 0u);
    for (unsigned i = 0; i < nw; ++i) workers_.emplace_back([this] { loop(); });
  }
  void run_tasks() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= n_) break;
      (*fn_)(i);
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      lk.unlock();
      run_tasks();
      lk.lock();
      if (--busy_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_m_, m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0};
  size_t busy_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// scenario_consistent (scenario.cpp:26-31): residual of Y V = I on non-slack
// present-phase rows, relative to max(1, |I|_inf). Scenarios are independent:
// they are checked on up to 16 host threads, and the first failing one (in
// library order) is reported, as the sequential loop would.
void check_residual(const Problem& p, const std::vector<double>& inj, const std::vector<double>& volt,
                    const std::vector<std::string>& ids) {
  const int n = p.y.n;
  const size_t L = ids.size();
  // std::complex product without the C99 Annex G call for finite operands
  // (same bits; NaN results take the library path)
  auto mul = [](cx a, cx b) {
    const double re = a.real() * b.real() - a.imag() * b.imag(), im = a.real() * b.imag() + a.imag() * b.real();
    return (std::isnan(re) && std::isnan(im)) ? a * b : cx{re, im};
  };
  std::vector<char> ok(L, 1);
  auto check = [&](size_t l0, size_t l1) {
    thread_local std::vector<cx> yv;
    yv.resize(size_t(3 * n));
    for (size_t l = l0; l < l1; ++l) {
      const double* V = volt.data() + l * size_t(6 * n);
      const double* I = inj.data() + l * size_t(6 * n);
      std::fill(yv.begin(), yv.end(), cx{});
      for (size_t b = 0; b < p.y.row.size(); ++b) {
        const int i = p.y.row[b], j = p.y.col[b];
        const double* blk = p.y.val.data() + b * 18;
        for (int r = 0; r < 3; ++r) {
          cx acc{};
          for (int c = 0; c < 3; ++c)
            acc += mul(cx{blk[6 * r + 2 * c], blk[6 * r + 2 * c + 1]}, cx{V[(3 * j + c) * 2], V[(3 * j + c) * 2 + 1]});
          yv[size_t(3 * i + r)] += acc;
        }
      }
      double res = 0, inorm = 0;
      for (int k = 0; k < 3 * n; ++k) inorm = std::max(inorm, std::abs(cx{I[2 * k], I[2 * k + 1]}));
      for (int i = 0; i < n; ++i) {
        if (i == p.slack) continue;
        for (int q = 0; q < 3; ++q)
          if ((p.mask[size_t(i)] >> q) & 1)
            res = std::max(res, std::abs(yv[size_t(3 * i + q)] - cx{I[(3 * i + q) * 2], I[(3 * i + q) * 2 + 1]}));
      }
      ok[l] = res <= 1e-10 * std::max(1.0, inorm) ? 1 : 0;
    }
  };
  if (size_t(n) * L < 4096)
    check(0, L);
  else
    HostPool::get().parallel_for(L, [&](size_t l) { check(l, l + 1); });
  for (size_t l = 0; l < L; ++l)
    if (!ok[l]) throw SolverError("scenario '" + ids[l] + "' failed the residual check");
}

// Engine over a host problem: current mode solves V-hat, PQ mode runs the
// constant-current fixed point on the device (load_library, scenario.cpp:141-220).
void load_scenarios_from_host(Engine* eng, const Problem& p, const krg_host_problem& hp);

std::unique_ptr<Engine> engine_from_host(const krg_host_problem& hp, int device) {
  Problem p = base_problem(hp.net);
  auto eng = std::make_unique<Engine>(p, device);
  load_scenarios_from_host(eng.get(), p, hp);
  return eng;
}

void load_scenarios_from_host(Engine* eng, const Problem& p, const krg_host_problem& hp) {
  const int L = int(hp.ids.size());
  if (L == 0) return;
  // per-thread scratch, reused across calls (MB-sized fresh vectors cost
  // their page faults on every reload)
  thread_local std::vector<double> inj, volt;
  if (hp.pq) {
    for (size_t g = 0; g < hp.ids.size(); ++g)
      for (const auto& ld : hp.pq_loads[g])
        if (ld.first / 3 == p.slack)
          throw ValidationError("scenario '" + hp.ids[g] + "': load placed at the slack node");
    // placeholder library (ids for messages); voltages given so no solve runs
    eng->set_scenarios(hp.ids, std::vector<double>(size_t(L) * 6 * size_t(hp.net.size()), 0.0),
                       std::vector<double>(size_t(L) * 6 * size_t(hp.net.size()), 0.0));
    eng->pq_to_currents(hp.pq_loads, inj, volt);
  } else {
    // current mode: V-hat = solve(I-hat) on the device (the engine keeps both)
    inj.assign(hp.inj.begin(), hp.inj.end());
    zero_invalid(hp.net, inj, L);
    eng->set_scenarios(hp.ids, inj, {});
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<double>& vh = eng->vhat();
    const auto t1 = std::chrono::steady_clock::now();
    check_residual(p, inj, vh, hp.ids);
    if (std::getenv("KRONRED_RELOAD_TRACE")) {
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "scenarios: V-hat %.3f ms, residual %.3f ms\n", ms(t0, t1),
                   ms(t1, std::chrono::steady_clock::now()));
    }
    return;
  }
  check_residual(p, inj, volt, hp.ids);
  eng->set_scenarios(hp.ids, inj, volt);
}

Problem problem_from(const Network& net, const ScenarioLibrary* lib) {
  Problem p = base_problem(net);
  if (lib != nullptr) {
    if (lib->scenarios.empty()) throw ValidationError("scenario library is empty");
    if (lib->n != net.size()) throw ValidationError("scenario library was built for a different network size");
    const int n = net.size();
    p.L = lib->size();
    for (const Scenario& sc : lib->scenarios) {
      p.scenario_ids.push_back(sc.id);
      if (int(sc.injections.size()) != 3 * n || int(sc.voltages.size()) != 3 * n)
        throw ValidationError("scenario '" + sc.id + "': vectors must have 3n entries");
      for (const cx& z : sc.injections) {
        p.injections.push_back(z.real());
        p.injections.push_back(z.imag());
      }
      for (const cx& z : sc.voltages) {
        p.voltages.push_back(z.real());
        p.voltages.push_back(z.imag());
      }
    }
  }
  return p;
}

ReductionConfig cfg_from_c(const krg_config* c) {
  ReductionConfig cfg;
  if (c == nullptr) return cfg;
  cfg.e_bar = c->e_bar;
  cfg.objective = c->objective == KRG_OBJ_COMPLEX ? Objective::complex_error : Objective::magnitude;
  if (c->has_target) cfg.target_reduction = c->target_reduction;
  cfg.use_delta = c->use_delta != 0;
  cfg.workers = c->workers;
  return cfg;
}

int device_from_env() {
  if (const char* e = std::getenv("KRONRED_DEVICE")) return std::atoi(e);
  return -1;  // current device of the calling thread
}

// KRONRED_DEVICES="0,1,..." : run_reduction on several GPUs of this process
// (the reference's worker split, parallel.cpp:11-34, across devices)
std::vector<int> devices_from_env() {
  std::vector<int> d;
  if (const char* e = std::getenv("KRONRED_DEVICES")) {
    std::string s(e);
    size_t i = 0;
    while (i < s.size()) {
      const size_t j = s.find(',', i);
      const std::string tok = s.substr(i, j == std::string::npos ? std::string::npos : j - i);
      if (!tok.empty()) d.push_back(std::atoi(tok.c_str()));
      if (j == std::string::npos) break;
      i = j + 1;
    }
  }
  return d;
}

// One engine and host thread per device, joined in one NCCL communicator;
// every rank runs the device loop on its candidate range and the in-graph
// exchange keeps them in lock step. Rank 0's result (identical on every
// rank) is returned; the observer runs on rank 0's thread.
void run_multi_device(const Problem& p, const std::vector<int>& devs, const ReductionConfig& cfg,
                      const Engine::Observer& obs, ResultData& out) {
  const int W = int(devs.size());
  std::vector<std::unique_ptr<Engine>> engs(static_cast<size_t>(W));
  std::vector<ResultData> res(static_cast<size_t>(W));
  std::vector<std::string> err(static_cast<size_t>(W));
  std::uint8_t id[KRG_NCCL_ID_BYTES];
  if (krg_nccl_unique_id(id) != KRG_OK) throw Error("ncclGetUniqueId failed");
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      try {
        engs[size_t(r)] = std::make_unique<Engine>(p, devs[size_t(r)]);
        engs[size_t(r)]->set_comm(r, W, id);  // collective over the W threads
        engs[size_t(r)]->run(cfg, r == 0 ? obs : Engine::Observer{}, res[size_t(r)]);
      } catch (const std::exception& e) {
        err[size_t(r)] = e.what();
      }
    });
  for (std::thread& t : th) t.join();
  for (int r = 0; r < W; ++r)
    if (!err[size_t(r)].empty()) throw Error("rank " + std::to_string(r) + ": " + err[size_t(r)]);
  out = std::move(res[0]);
}

// Engine cache of the C++ drop-in entry points (one per calling thread): the
// reference signature builds its solver per call (reduce.cpp:359); here a call
// on a network of the same STRUCTURE (node phases, slack, branch endpoints,
// block pattern, scenario count, device) reuses the resident engine -- its
// elimination schedule, device allocations and instantiated loop graph -- and
// only re-uploads the values (Engine::reload + set_scenarios: H2D copies and
// the refactorization every run performs anyway). KRONRED_ENGINE_CACHE=0
// disables it; kronred::release_engine_cache() frees it.
struct EngineCache {
  std::string key;
  std::unique_ptr<Engine> eng;
};
thread_local EngineCache t_engine_cache;

std::string structure_key(const Problem& p, int device) {
  std::string k;
  auto put = [&](const void* d, size_t n) { k.append(static_cast<const char*>(d), n); };
  const int hdr[4] = {p.y.n, p.slack, p.L, device};
  put(hdr, sizeof hdr);
  put(p.mask.data(), p.mask.size());
  put(p.y.row.data(), p.y.row.size() * sizeof(int));
  put(p.y.col.data(), p.y.col.size() * sizeof(int));
  for (const Branch& b : p.net.branches) {
    const int e[2] = {b.from, b.to};
    put(e, sizeof e);
  }
  return k;
}

// the engine for `p`: the cached one with new values, or a new one
Engine& cached_engine(const Problem& p) {
  const int dev = device_from_env();
  const char* e = std::getenv("KRONRED_ENGINE_CACHE");
  const bool on = !(e && std::string(e) == "0");
  std::string key = structure_key(p, dev);
  EngineCache& c = t_engine_cache;
  if (on && c.eng && c.key == key) {
    c.eng->reload(p);
    c.eng->set_scenarios(p.scenario_ids, p.injections, p.voltages);
    return *c.eng;
  }
  c.eng.reset();  // release the old device memory before allocating
  c.eng = std::make_unique<Engine>(p, dev);
  c.key = on ? std::move(key) : std::string();
  return *c.eng;
}

}  // namespace

// ---------------------------------------------------------------------------
// C++ drop-in API

namespace kronred {

ScenarioLibrary load_library(const Network& net, const std::string& path) {
  krg_host_problem hp;
  hp.net = net;
  parse_scenarios(hp, path);
  ScenarioLibrary lib;
  lib.n = net.size();
  if (hp.ids.empty()) return lib;
  auto eng = engine_from_host(hp, device_from_env());
  const int n = net.size();
  const Problem& p = eng->problem();
  const std::vector<double>& vh = eng->vhat();
  for (size_t l = 0; l < hp.ids.size(); ++l) {
    Scenario sc;
    sc.id = hp.ids[l];
    for (int k = 0; k < 3 * n; ++k) {
      sc.injections.push_back(cx{p.injections[(l * 3 * n + size_t(k)) * 2], p.injections[(l * 3 * n + size_t(k)) * 2 + 1]});
      sc.voltages.push_back(cx{vh[(l * 3 * n + size_t(k)) * 2], vh[(l * 3 * n + size_t(k)) * 2 + 1]});
    }
    lib.scenarios.push_back(std::move(sc));
  }
  return lib;
}

ReductionResult run_reduction(const Network& net, const ScenarioLibrary& lib, const ReductionConfig& cfg,
                              const IterationObserver& observer) {
  validate_or_throw(net);
  if (!(cfg.e_bar >= 0)) throw ConfigError("e_bar must be non-negative");
  if (cfg.target_reduction && !(*cfg.target_reduction >= 0 && *cfg.target_reduction <= 1))
    throw ConfigError("target_reduction must lie in [0,1]");
  ResultData rd;
  Engine::Observer obs;
  if (observer) obs = [&](const HostState& hs, const TraceRow& row) { observer(hs, row); };
  const std::vector<int> devs = devices_from_env();
  if (devs.size() > 1) {
    run_multi_device(problem_from(net, &lib), devs, cfg, obs, rd);
  } else {
    Engine& eng = cached_engine(problem_from(net, &lib));
    eng.run(cfg, obs, rd);
  }
  ReductionResult res;
  res.model = std::move(rd.model);
  res.trace = std::move(rd.trace);
  res.state = static_cast<AssignmentState&&>(std::move(rd.state));
  return res;
}

KronResult kron_reduce(const BlockMatrix& y, const std::vector<PhaseMask>& phases, const Partition& part) {
  Problem p;
  p.y = FlatBlocks::from(y);
  for (const PhaseMask& m : phases) p.mask.push_back(m.bits);
  p.slack = -1;
  Engine eng(p, device_from_env());
  ReducedModel m;
  eng.kron(part.reduce, m);
  std::vector<int> keep = part.keep;
  std::sort(keep.begin(), keep.end());
  if (keep != m.kept_ids) throw ValidationError("partition: keep set does not cover the non-reduced nodes");
  KronResult kr;
  kr.y_kron = std::move(m.y_kron);
  kr.kept_ids = std::move(m.kept_ids);
  kr.kept_phases = std::move(m.kept_phases);
  return kr;
}

std::vector<double> model_max_errors(const ReducedModel& model, const Network& net, const ScenarioLibrary& lib) {
  return cached_engine(problem_from(net, &lib)).model_errors(model);
}

ValidateReport make_validate_report(const ReducedModel& model, const Network& net, const ScenarioLibrary& lib,
                                    int bins) {
  return validate_report(lib.ids(), model_max_errors(model, net, lib), bins);
}

void write_validate_report(const ValidateReport& rep, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Error("cannot write " + path);
  f << validate_csv(rep);
}

void release_engine_cache() {
  t_engine_cache.eng.reset();
  t_engine_cache.key.clear();
}

ReducedModel radialize(const ReducedModel& model, const Network& original, const BlockMatrix& y,
                       const ScenarioLibrary* lib) {
  Problem p = problem_from(original, lib);
  p.y = FlatBlocks::from(y);
  Engine eng(p, device_from_env());
  ReducedModel out = model;
  eng.radialize(out, lib != nullptr);
  return out;
}

}  // namespace kronred

// ---------------------------------------------------------------------------
// C ABI

#define KRG_TRY try {
#define KRG_CATCH \
  }               \
  catch (...) { return status_from_current_exception(); }

extern "C" {

const char* krg_last_error(void) { return g_err.c_str(); }
double krg_last_error_pivot(void) { return g_pivot; }
int32_t krg_last_error_node(void) { return g_node; }
const char* krg_version(void) { return "kronred-b200 0.1.0 (sm_100a)"; }

int krg_host_load(const char* net_path, const char* scen_path, krg_host_problem** out) {
  KRG_TRY
  auto hp = std::make_unique<krg_host_problem>();
  std::ifstream f(net_path, std::ios::binary);
  if (!f) throw ValidationError(std::string("cannot open '") + net_path + "'");
  std::ostringstream ss;
  ss << f.rdbuf();
  hp->net = parse_network_text(ss.str());
  if (scen_path != nullptr && scen_path[0] != 0) parse_scenarios(*hp, scen_path);
  fill_views(*hp);
  *out = hp.release();
  return KRG_OK;
  KRG_CATCH
}

int krg_host_view(const krg_host_problem* p, krg_network* net, int32_t* L, int32_t* pq_mode,
                  const double** data) {
  if (p == nullptr) return KRG_E_INTERNAL;
  net->n_nodes = p->net.size();
  net->phases = p->phases.data();
  net->slack = p->net.slack_id();
  net->slack_voltage = p->slackv.data();
  net->n_branches = int32_t(p->net.branches.size());
  net->br_from = p->from.data();
  net->br_to = p->to.data();
  net->y_series = p->ys.data();
  net->shunt_from = p->sf.data();
  net->shunt_to = p->st.data();
  if (L) *L = int32_t(p->ids.size());
  if (pq_mode) *pq_mode = p->pq ? 1 : 0;
  if (data) *data = p->pq ? p->pq_flat.data() : p->inj.data();
  return KRG_OK;
}

const char* krg_host_scenario_id(const krg_host_problem* p, int32_t l) {
  return (p && l >= 0 && size_t(l) < p->ids.size()) ? p->ids[size_t(l)].c_str() : nullptr;
}

void krg_host_free(krg_host_problem* p) { delete p; }

int krg_validate(const krg_network* cn) {
  KRG_TRY
  validate_or_throw(network_from_c(cn));
  return KRG_OK;
  KRG_CATCH
}

int64_t krg_enumerate_after(const krg_network* cn, const int32_t* ts, const int32_t* tr, int32_t nc,
                            int32_t* cs, int32_t* cr, int64_t cap) {
  try {
    const Network net = network_from_c(cn);
    validate_or_throw(net);
    HostState hs;
    hs.init(net);
    for (int i = 0; i < nc; ++i) hs.commit(ts[i], tr[i]);
    std::vector<int> a, b;
    hs.enumerate(a, b);
    for (size_t i = 0; i < a.size() && int64_t(i) < cap; ++i) {
      cs[i] = a[i];
      cr[i] = b[i];
    }
    return int64_t(a.size());
  } catch (...) {
    return -int64_t(status_from_current_exception());
  }
}

void krg_shard_range(int64_t count, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
  // contiguous split, the first (count % world) ranks take one extra
  // (parallel.cpp:21-29)
  if (world < 1) world = 1;
  const int64_t base = count / world, extra = count % world;
  const int64_t b = rank * base + std::min<int64_t>(rank, extra);
  *begin = b;
  *end = b + base + (rank < extra ? 1 : 0);
}

int32_t krg_merge_best(const double* smice, const int64_t* index, int32_t world) {
  int32_t best = -1;
  for (int32_t w = 0; w < world; ++w) {
    if (index[w] < 0) continue;
    if (best < 0 || smice[w] < smice[best] || (smice[w] == smice[best] && index[w] < index[best])) best = w;
  }
  return best;
}

int krg_create(const krg_network* cn, const krg_scenarios* scen, int32_t device, krg_ctx** out) {
  KRG_TRY
  const Network net = network_from_c(cn);
  Problem p = base_problem(net);
  auto ctx = std::make_unique<krg_ctx>();
  ctx->eng = std::make_unique<Engine>(p, device);
  if (scen != nullptr && scen->n_scenarios > 0) {
    const int n = net.size(), L = scen->n_scenarios;
    std::vector<double> inj(scen->injections, scen->injections + size_t(L) * 6 * n);
    std::vector<double> volt;
    std::vector<std::string> ids;
    for (int l = 0; l < L; ++l) ids.push_back("s" + std::to_string(l));
    if (scen->voltages != nullptr) {
      volt.assign(scen->voltages, scen->voltages + size_t(L) * 6 * n);
    } else {
      zero_invalid(net, inj, L);
    }
    ctx->eng->set_scenarios(ids, inj, volt);
  }
  *out = ctx.release();
  return KRG_OK;
  KRG_CATCH
}

int krg_create_from_host(const krg_host_problem* hp, int32_t device, krg_ctx** out) {
  KRG_TRY
  auto ctx = std::make_unique<krg_ctx>();
  ctx->eng = engine_from_host(*hp, device);
  *out = ctx.release();
  return KRG_OK;
  KRG_CATCH
}

int krg_reload_from_host(krg_ctx* ctx, const krg_host_problem* hp) {
  KRG_TRY
  const bool tr = std::getenv("KRONRED_RELOAD_TRACE") != nullptr;  // tuning aid: phase times
  const auto t0 = std::chrono::steady_clock::now();
  Problem p = base_problem(hp->net);
  const auto t1 = std::chrono::steady_clock::now();
  ctx->eng->reload(p);
  const auto t2 = std::chrono::steady_clock::now();
  load_scenarios_from_host(ctx->eng.get(), p, *hp);
  const auto t3 = std::chrono::steady_clock::now();
  if (tr) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "reload: assembly %.2f ms, refactorize %.2f ms, scenarios %.2f ms\n", ms(t0, t1), ms(t1, t2),
                 ms(t2, t3));
  }
  return KRG_OK;
  KRG_CATCH
}

void krg_destroy(krg_ctx* ctx) { delete ctx; }

int krg_set_exchange(krg_ctx* ctx, int32_t rank, int32_t world, krg_exchange_fn fn, void* user) {
  KRG_TRY
  ctx->eng->set_exchange(rank, world, fn, user);
  return KRG_OK;
  KRG_CATCH
}

int krg_set_comm(krg_ctx* ctx, int32_t rank, int32_t world, const uint8_t* unique_id) {
  KRG_TRY
  ctx->eng->set_comm(rank, world, unique_id);
  return KRG_OK;
  KRG_CATCH
}

int64_t krg_launch_count(const krg_ctx* ctx) { return ctx ? ctx->eng->launches() : 0; }
int32_t krg_last_run_device_loop(const krg_ctx* ctx) { return ctx && ctx->eng->last_run_device_loop() ? 1 : 0; }

int krg_set_profile(krg_ctx* ctx, int32_t on) {
  KRG_TRY
  ctx->eng->set_profile(on != 0);
  return KRG_OK;
  KRG_CATCH
}

int krg_kernel_stats(const krg_ctx* ctx, int32_t which, int64_t* launches, double* ms, double* flops,
                     double* bytes) {
  const KernelStats k = ctx->eng->stats(which);
  *launches = k.launches;
  *ms = k.ms;
  *flops = k.flops;
  *bytes = k.bytes;
  return KRG_OK;
}

double krg_result_device_ms(const krg_result* r) { return r->d.device_ms; }

int krg_scenario_voltages(krg_ctx* ctx, double* out) {
  KRG_TRY
  ctx->eng->scenario_voltages(out);
  return KRG_OK;
  KRG_CATCH
}

int krg_run_reduction(krg_ctx* ctx, const krg_config* c, krg_observer_fn obs, void* user, krg_result** out) {
  KRG_TRY
  auto res = std::make_unique<krg_result>();
  Engine::Observer o;
  if (obs)
    o = [&](const HostState&, const TraceRow& r) {
      obs(user, r.iteration, r.s, r.r, r.smice, r.max_err.data(), r.supernode_count, r.candidate_count, r.wall_ms);
    };
  ctx->eng->run(cfg_from_c(c), o, res->d);
  *out = res.release();
  return KRG_OK;
  KRG_CATCH
}

int krg_solve(krg_ctx* ctx, const double* inj, int32_t nrhs, double* out) {
  KRG_TRY
  ctx->eng->solve(inj, nrhs, out);
  return KRG_OK;
  KRG_CATCH
}

int krg_debug_base_refresh(krg_ctx* ctx, int32_t reps, double* ms, long long* clocks) {
  KRG_TRY
  ctx->eng->debug_base_refresh(reps, ms, clocks);
  return KRG_OK;
  KRG_CATCH
}

int krg_loop_begin(krg_ctx* ctx, const krg_config* c) {
  KRG_TRY
  ctx->eng->loop_begin(cfg_from_c(c));
  return KRG_OK;
  KRG_CATCH
}

int64_t krg_loop_candidates(krg_ctx* ctx, int32_t* cs, int32_t* cr, int64_t cap) {
  try {
    std::vector<int> a, b;
    const int64_t C = ctx->eng->loop_candidates(a, b);
    for (int64_t i = 0; i < C && i < cap; ++i) {
      cs[i] = a[size_t(i)];
      cr[i] = b[size_t(i)];
    }
    return C;
  } catch (...) {
    return -int64_t(status_from_current_exception());
  }
}

int krg_loop_score_all(krg_ctx* ctx, double* smice, uint8_t* feasible, double* max_err) {
  KRG_TRY
  ctx->eng->loop_score_all(smice, feasible, max_err);
  return KRG_OK;
  KRG_CATCH
}

int krg_loop_best(krg_ctx* ctx, krg_best* out, double* max_err) {
  KRG_TRY
  ctx->eng->loop_best(out, max_err);
  return KRG_OK;
  KRG_CATCH
}

int krg_loop_commit(krg_ctx* ctx, int32_t s, int32_t r) {
  KRG_TRY
  ctx->eng->loop_commit(s, r);
  return KRG_OK;
  KRG_CATCH
}

int krg_zcols(krg_ctx* ctx, double* out, int64_t cap) {
  KRG_TRY
  ctx->eng->zcols(out, cap);
  return KRG_OK;
  KRG_CATCH
}

int krg_loop_base(krg_ctx* ctx, double* out) {
  KRG_TRY
  ctx->eng->loop_base(out);
  return KRG_OK;
  KRG_CATCH
}

int krg_kron_reduce(krg_ctx* ctx, const int32_t* reduce, int32_t m, krg_result** out) {
  KRG_TRY
  auto res = std::make_unique<krg_result>();
  std::vector<int> red(reduce, reduce + m);
  ctx->eng->kron(red, res->d.model);
  *out = res.release();
  return KRG_OK;
  KRG_CATCH
}

int krg_radialize(krg_ctx* ctx, krg_result* res, int32_t with_errors) {
  KRG_TRY
  ctx->eng->radialize(res->d.model, with_errors != 0);
  return KRG_OK;
  KRG_CATCH
}

int32_t krg_result_iterations(const krg_result* r) { return int32_t(r->d.trace.size()); }
int32_t krg_result_n_scenarios(const krg_result* r) { return int32_t(r->d.model.scenario_ids.size()); }

int krg_result_trace(const krg_result* res, int32_t* s, int32_t* r, double* smice, double* max_err,
                     int32_t* snc, int32_t* cc, double* wall) {
  const auto& tr = res->d.trace;
  for (size_t i = 0; i < tr.size(); ++i) {
    if (s) s[i] = tr[i].s;
    if (r) r[i] = tr[i].r;
    if (smice) smice[i] = tr[i].smice;
    if (max_err)
      std::copy(tr[i].max_err.begin(), tr[i].max_err.end(), max_err + i * tr[i].max_err.size());
    if (snc) snc[i] = tr[i].supernode_count;
    if (cc) cc[i] = tr[i].candidate_count;
    if (wall) wall[i] = tr[i].wall_ms;
  }
  return KRG_OK;
}

int32_t krg_result_n_kept(const krg_result* r) { return int32_t(r->d.model.kept_ids.size()); }

int krg_result_kept(const krg_result* r, int32_t* ids, uint8_t* phases) {
  for (size_t i = 0; i < r->d.model.kept_ids.size(); ++i) {
    if (ids) ids[i] = r->d.model.kept_ids[i];
    if (phases) phases[i] = r->d.model.kept_phases[i].bits;
  }
  return KRG_OK;
}

int64_t krg_result_n_blocks(const krg_result* r) { return r->d.model.y_kron.block_count(); }

int krg_result_blocks(const krg_result* r, int32_t* bi, int32_t* bj, double* vals) {
  const auto& m = r->d.model;
  size_t k = 0;
  for (int i = 0; i < m.y_kron.n(); ++i)
    for (const auto& [j, blk] : m.y_kron.row(i)) {
      if (bi) bi[k] = m.kept_ids[size_t(i)];
      if (bj) bj[k] = m.kept_ids[size_t(j)];
      if (vals)
        for (int e = 0; e < 9; ++e) {
          vals[k * 18 + size_t(2 * e)] = blk.m[size_t(e)].real();
          vals[k * 18 + size_t(2 * e + 1)] = blk.m[size_t(e)].imag();
        }
      ++k;
    }
  return KRG_OK;
}

int krg_result_final_max_err(const krg_result* r, double* out) {
  std::copy(r->d.model.final_max_err.begin(), r->d.model.final_max_err.end(), out);
  return KRG_OK;
}

int32_t krg_result_n_clusters(const krg_result* r) { return int32_t(r->d.model.clusters.size()); }

int krg_result_clusters(const krg_result* r, int32_t* sup, int32_t* off, int32_t* members) {
  size_t k = 0, m = 0;
  if (off) off[0] = 0;
  for (const auto& [s, mem] : r->d.model.clusters) {
    if (sup) sup[k] = s;
    for (int j : mem) {
      if (members) members[m] = j;
      ++m;
    }
    ++k;
    if (off) off[k] = int32_t(m);
  }
  return KRG_OK;
}

int32_t krg_result_n_reinserted(const krg_result* r) { return int32_t(r->d.model.reinserted.size()); }

int krg_result_reinserted(const krg_result* r, int32_t* ids) {
  std::copy(r->d.model.reinserted.begin(), r->d.model.reinserted.end(), ids);
  return KRG_OK;
}

int64_t krg_result_total_candidates(const krg_result* r) { return r->d.total_candidates; }

int krg_result_write_reduced_json(const krg_result* r, const char* path) {
  KRG_TRY
  write_reduced_json(r->d.model, path);
  return KRG_OK;
  KRG_CATCH
}

int64_t krg_validate_report(krg_ctx* ctx, const krg_result* res, int32_t bins, char* out, int64_t cap) {
  try {
    const std::string csv =
        validate_csv(validate_report(res->d.model.scenario_ids, ctx->eng->model_errors(res->d.model), bins));
    if (out && cap > 0) {
      const size_t k = std::min(size_t(cap - 1), csv.size());
      std::memcpy(out, csv.data(), k);
      out[k] = '\0';
    }
    return int64_t(csv.size());
  } catch (...) {
    return -int64_t(status_from_current_exception());
  }
}

int krg_result_write_trace_csv(const krg_result* r, const char* path, int32_t zero_wall) {
  KRG_TRY
  std::vector<TraceRow> tr = r->d.trace;
  if (zero_wall)
    for (TraceRow& t : tr) t.wall_ms = 0;
  write_trace_csv(path, tr, r->d.model.scenario_ids, r->d.model.final_max_err);
  return KRG_OK;
  KRG_CATCH
}

void krg_result_free(krg_result* r) { delete r; }

}  // extern "C"
