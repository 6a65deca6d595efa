// Reference-side shim: kronred::run_reduction of the REFERENCE's own headers
// (proj/include/kronred/reduce.hpp:168-170) implemented by forwarding to the
// B200 library's C ABI (include/kronred_b200.h). A reference build keeps all of
// its sources and headers, adds this translation unit, and drops (or weakens)
// the CPU definition in reduce.cpp:349-451; every caller -- the CLI's
// cmd_reduce, the acceptance binary, user code -- then reduces on the GPU.
//
// What crosses the boundary is plain data: the Network's nodes and branches
// (Mat3c = 9 row-major std::complex<double> = 18 doubles), the library's
// injections and voltages, the config. The result comes back through the
// krg_result_* accessors. The per-iteration AssignmentState the observer sees,
// and the final one, are rebuilt with the reference's own init_state/commit
// (reduce.cpp:39-61, 299-344) from the committed (s, r) pairs, so an observer
// gets exactly the reference's state objects, live (krg observer callback).
//
// Built and checked by oracle/Makefile (target `shim`) and
// tests/test_gpu_parity.py::test_reference_shim_relinks_reference_binary.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronred/errors.hpp"
#include "kronred/reduce.hpp"
#include "kronred_b200.h"

namespace kronred {
namespace {

void throw_status(int st) {
  const std::string msg = krg_last_error() ? krg_last_error() : "kronred_b200 error";
  if (st == KRG_E_VALIDATION) throw ValidationError(msg);
  if (st == KRG_E_SOLVER) throw SolverError(msg, krg_last_error_pivot(), krg_last_error_node());
  throw Error(msg);
}
void ck(int st) {
  if (st != KRG_OK) throw_status(st);
}

struct ObserverState {
  const IterationObserver* obs;
  AssignmentState* st;
  std::vector<TraceRow>* rows;
};

void observer_trampoline(void* user, int32_t it, int32_t s, int32_t r, double smice, const double* me, int32_t snc,
                         int32_t cc, double wall_ms) {
  auto* o = static_cast<ObserverState*>(user);
  commit(*o->st, Candidate{s, r});
  TraceRow row;
  row.iteration = it;
  row.s = s;
  row.r = r;
  row.smice = smice;
  row.max_err.assign(me, me + o->st->i_agg.size());
  row.supernode_count = snc;
  row.candidate_count = cc;
  row.wall_ms = wall_ms;
  if (*o->obs) (*o->obs)(*o->st, row);
  o->rows->push_back(std::move(row));
}

}  // namespace

ReductionResult run_reduction(const Network& net, const ScenarioLibrary& lib, const ReductionConfig& cfg,
                              const IterationObserver& observer) {
  const int n = net.size(), L = lib.size();
  // network -> krg_network (plain arrays)
  std::vector<uint8_t> phases(static_cast<size_t>(n));
  double slack_v[6] = {};
  const int slack = net.slack_id();
  for (int i = 0; i < n; ++i) phases[size_t(i)] = net.nodes[size_t(i)].phases.bits;
  if (slack >= 0)
    for (int p = 0; p < 3; ++p) {
      slack_v[2 * p] = net.nodes[size_t(slack)].slack_voltage[p].real();
      slack_v[2 * p + 1] = net.nodes[size_t(slack)].slack_voltage[p].imag();
    }
  const size_t nb = net.branches.size();
  std::vector<int32_t> bf(nb), bt(nb);
  std::vector<double> ys(nb * 18), sf(nb * 18), sh(nb * 18);
  for (size_t b = 0; b < nb; ++b) {
    const Branch& br = net.branches[b];
    bf[b] = br.from;
    bt[b] = br.to;
    for (int e = 0; e < 9; ++e) {
      ys[b * 18 + size_t(2 * e)] = br.y_series.m[size_t(e)].real();
      ys[b * 18 + size_t(2 * e + 1)] = br.y_series.m[size_t(e)].imag();
      sf[b * 18 + size_t(2 * e)] = br.shunt_from.m[size_t(e)].real();
      sf[b * 18 + size_t(2 * e + 1)] = br.shunt_from.m[size_t(e)].imag();
      sh[b * 18 + size_t(2 * e)] = br.shunt_to.m[size_t(e)].real();
      sh[b * 18 + size_t(2 * e + 1)] = br.shunt_to.m[size_t(e)].imag();
    }
  }
  const krg_network cn{n, phases.data(), slack, slack_v, int32_t(nb), bf.data(), bt.data(), ys.data(), sf.data(),
                       sh.data()};
  // library -> krg_scenarios (the voltages the reference library solved)
  std::vector<double> inj(size_t(L) * 6 * n), volt(size_t(L) * 6 * n);
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < 3 * n; ++k) {
      const size_t o = (size_t(l) * 3 * n + size_t(k)) * 2;
      inj[o] = lib.scenarios[size_t(l)].injections[size_t(k)].real();
      inj[o + 1] = lib.scenarios[size_t(l)].injections[size_t(k)].imag();
      volt[o] = lib.scenarios[size_t(l)].voltages[size_t(k)].real();
      volt[o + 1] = lib.scenarios[size_t(l)].voltages[size_t(k)].imag();
    }
  const krg_scenarios sc{L, inj.data(), volt.data()};
  krg_ctx* ctx = nullptr;
  ck(krg_create(&cn, &sc, -1, &ctx));
  const krg_config kc{cfg.e_bar, cfg.objective == Objective::complex_error ? KRG_OBJ_COMPLEX : KRG_OBJ_MAGNITUDE,
                      cfg.target_reduction ? 1 : 0, cfg.target_reduction.value_or(0.0), cfg.use_delta ? 1 : 0,
                      cfg.workers};
  ReductionResult res;
  res.state = init_state(net, lib);  // the reference's own state machine, advanced per commit below
  ObserverState os{&observer, &res.state, &res.trace};
  krg_result* kr = nullptr;
  const int st = krg_run_reduction(ctx, &kc, observer_trampoline, &os, &kr);
  if (st != KRG_OK) {
    krg_destroy(ctx);
    throw_status(st);
  }
  // reduced model
  ReducedModel& m = res.model;
  const int nk = krg_result_n_kept(kr);
  std::vector<int32_t> kid(static_cast<size_t>(nk));
  std::vector<uint8_t> kph(static_cast<size_t>(nk));
  ck(krg_result_kept(kr, kid.data(), kph.data()));
  m.kept_ids.assign(kid.begin(), kid.end());
  for (uint8_t b : kph) m.kept_phases.push_back(PhaseMask{b});
  m.y_kron = BlockMatrix(nk);
  const int64_t nblk = krg_result_n_blocks(kr);
  std::vector<int32_t> bi(static_cast<size_t>(nblk)), bj(static_cast<size_t>(nblk));
  std::vector<double> bv(size_t(nblk) * 18);
  ck(krg_result_blocks(kr, bi.data(), bj.data(), bv.data()));
  std::vector<int> pos(size_t(n), -1);
  for (int k = 0; k < nk; ++k) pos[size_t(kid[size_t(k)])] = k;
  for (int64_t q = 0; q < nblk; ++q) {
    Mat3c& blk = m.y_kron.block(pos[size_t(bi[size_t(q)])], pos[size_t(bj[size_t(q)])]);
    for (int e = 0; e < 9; ++e) blk.m[size_t(e)] = cx{bv[size_t(q) * 18 + size_t(2 * e)], bv[size_t(q) * 18 + size_t(2 * e + 1)]};
  }
  const int ncl = krg_result_n_clusters(kr);
  std::vector<int32_t> csup(static_cast<size_t>(ncl)), coff(static_cast<size_t>(ncl) + 1), cmem(static_cast<size_t>(n));
  ck(krg_result_clusters(kr, csup.data(), coff.data(), cmem.data()));
  for (int c = 0; c < ncl; ++c)
    m.clusters[csup[size_t(c)]] = std::vector<int>(cmem.begin() + coff[size_t(c)], cmem.begin() + coff[size_t(c) + 1]);
  m.final_max_err.resize(size_t(L));
  ck(krg_result_final_max_err(kr, m.final_max_err.data()));
  m.e_bar = cfg.e_bar;
  m.objective = cfg.objective;
  m.scenario_ids = lib.ids();
  krg_result_free(kr);
  krg_destroy(ctx);
  return res;
}

}  // namespace kronred
