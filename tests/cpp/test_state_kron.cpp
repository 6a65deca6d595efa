// C++ port of the reference's "full run: invariants hold after every commit
// and errors stay bounded" (proj/tests/test_reduce.cpp:360-403, invariants at
// :34-95), written against the drop-in header and linked with
// libkronred_b200.so. It checks, through the public AssignmentState the
// observer and ReductionResult carry:
//   * every commit: column sums of A, slack self-owned, phase availability,
//     connected clusters, i_agg == (A (x) I3) I-hat to 1e-15, radial lambda;
//   * at the end: Kron consistency within 1e-10 -- the reduced-Y anchored
//     solve with res.state.i_agg at the kept nodes equals the full-Y solve
//     with the same injections at the kept nodes.
// The anchored solves here are a dense complex LU with partial pivoting
// (the reference's own test oracle, test_util.hpp:23-92): test code, not the
// product path.
//
// usage: test_state_kron net.json scen.csv e_bar
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <queue>

#include "kronred_b200.hpp"

using namespace kronred;

static int failures = 0;
#define CHECK(c)                                                       \
  do {                                                                 \
    if (!(c)) {                                                        \
      if (failures < 20) std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

// dense anchored solve: rows/cols = present phases of non-anchor nodes
static std::vector<cx> dense_anchored(const BlockMatrix& y, const std::vector<PhaseMask>& ph, int anchor,
                                      const Vec3c& v_anchor, const std::vector<cx>& inj) {
  const int n = y.n();
  std::vector<int> idx;  // scalar index (3i+p) of each unknown
  for (int i = 0; i < n; ++i)
    if (i != anchor)
      for (int p = 0; p < 3; ++p)
        if (ph[size_t(i)].has(p)) idx.push_back(3 * i + p);
  const int m = int(idx.size());
  std::vector<int> pos(size_t(3 * n), -1);
  for (int k = 0; k < m; ++k) pos[size_t(idx[size_t(k)])] = k;
  std::vector<cx> a(size_t(m) * size_t(m), cx{}), b(size_t(m), cx{});
  for (int k = 0; k < m; ++k) b[size_t(k)] = inj[size_t(idx[size_t(k)])];
  for (int i = 0; i < n; ++i)
    for (const auto& [j, blk] : y.row(i))
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
          const int r = pos[size_t(3 * i + p)];
          if (r < 0) continue;
          if (j == anchor) {
            b[size_t(r)] -= blk(p, q) * v_anchor[q];
            continue;
          }
          const int c = pos[size_t(3 * j + q)];
          if (c >= 0) a[size_t(r) * size_t(m) + size_t(c)] += blk(p, q);
        }
  for (int k = 0; k < m; ++k) {  // LU with partial pivoting
    int pv = k;
    for (int r = k + 1; r < m; ++r)
      if (std::abs(a[size_t(r) * m + k]) > std::abs(a[size_t(pv) * m + k])) pv = r;
    if (pv != k) {
      for (int c = 0; c < m; ++c) std::swap(a[size_t(k) * m + c], a[size_t(pv) * m + c]);
      std::swap(b[size_t(k)], b[size_t(pv)]);
    }
    for (int r = k + 1; r < m; ++r) {
      const cx f = a[size_t(r) * m + k] / a[size_t(k) * m + k];
      if (f == cx{}) continue;
      for (int c = k; c < m; ++c) a[size_t(r) * m + c] -= f * a[size_t(k) * m + c];
      b[size_t(r)] -= f * b[size_t(k)];
    }
  }
  std::vector<cx> x(static_cast<size_t>(m));
  for (int k = m - 1; k >= 0; --k) {
    cx s = b[size_t(k)];
    for (int c = k + 1; c < m; ++c) s -= a[size_t(k) * m + c] * x[size_t(c)];
    x[size_t(k)] = s / a[size_t(k) * m + k];
  }
  std::vector<cx> v(size_t(3 * n), cx{});
  for (int p = 0; p < 3; ++p) v[size_t(3 * anchor + p)] = ph[size_t(anchor)].has(p) ? v_anchor[p] : cx{};
  for (int k = 0; k < m; ++k) v[size_t(idx[size_t(k)])] = x[size_t(k)];
  return v;
}

static void check_state_invariants(const AssignmentState& st, const Network& net, const ScenarioLibrary& lib) {
  const auto masks = phase_masks(net);
  const int n = st.n;
  // A has exactly one 1 per column (sup is a map) and owners are super-nodes
  for (int j = 0; j < n; ++j) {
    const int i = st.sup[size_t(j)];
    CHECK(i >= 0 && i < n);
    CHECK(st.sup[size_t(i)] == i);
    CHECK(masks[size_t(j)].subset_of(masks[size_t(i)]));
  }
  CHECK(st.sup[size_t(st.slack)] == st.slack);
  const auto adj = net.neighbor_lists();
  int covered = 0;
  for (int i : st.supernodes) {
    const auto& mem = st.members[size_t(i)];
    covered += int(mem.size());
    std::vector<char> in(size_t(n), 0), seen(size_t(n), 0);
    for (int j : mem) in[size_t(j)] = 1;
    std::queue<int> q;
    q.push(mem.front());
    seen[size_t(mem.front())] = 1;
    int reached = 0;
    while (!q.empty()) {
      const int u = q.front();
      q.pop();
      ++reached;
      for (int v : adj[size_t(u)])
        if (in[size_t(v)] && !seen[size_t(v)]) {
          seen[size_t(v)] = 1;
          q.push(v);
        }
    }
    CHECK(reached == int(mem.size()));
  }
  CHECK(covered == n);
  CHECK(st.i_agg.size() == lib.scenarios.size());
  for (size_t l = 0; l < lib.scenarios.size() && l < st.i_agg.size(); ++l) {
    std::vector<cx> expect(size_t(3 * n), cx{});
    for (int j = 0; j < n; ++j)
      for (int p = 0; p < 3; ++p)
        expect[size_t(3 * st.sup[size_t(j)] + p)] += lib.scenarios[l].injections[size_t(3 * j + p)];
    double d = 0;
    for (int k = 0; k < 3 * n; ++k) d = std::max(d, std::abs(st.i_agg[l][size_t(k)] - expect[size_t(k)]));
    CHECK(d < 1e-15);
  }
  int edges = 0;
  for (int i : st.supernodes) edges += int(st.lambda[size_t(i)].size());
  CHECK(edges == 2 * (st.supernode_count() - 1));
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s net.json scen.csv e_bar\n", argv[0]);
    return 2;
  }
  const Network net = read_network_json(argv[1]);
  const ScenarioLibrary lib = load_library(net, argv[2]);
  ReductionConfig cfg;
  cfg.e_bar = std::strtod(argv[3], nullptr);
  int commits = 0;
  const ReductionResult res = run_reduction(net, lib, cfg, [&](const AssignmentState& st, const TraceRow& row) {
    check_state_invariants(st, net, lib);
    for (double e : row.max_err) CHECK(e <= cfg.e_bar);
    CHECK(row.candidate_count <= 2 * st.supernode_count());
    CHECK(row.supernode_count == st.supernode_count());
    ++commits;
  });
  CHECK(commits == int(res.trace.size()));
  CHECK(res.model.kept_ids.size() == size_t(res.state.supernode_count()));
  check_state_invariants(res.state, net, lib);
  for (double e : res.model.final_max_err) CHECK(e <= cfg.e_bar * (1 + 1e-9));

  // Kron consistency (test_reduce.cpp:383-402)
  const BlockAdmittance y = assemble_admittance(net);
  const auto masks = phase_masks(net);
  const int slack = net.slack_id();
  const Vec3c vs = net.nodes[size_t(slack)].slack_voltage;
  int slack_pos = -1;
  for (size_t k = 0; k < res.model.kept_ids.size(); ++k)
    if (res.model.kept_ids[k] == slack) slack_pos = int(k);
  CHECK(slack_pos >= 0);
  double worst = 0;
  for (size_t l = 0; l < lib.scenarios.size(); ++l) {
    const std::vector<cx> v_full = dense_anchored(y, masks, slack, vs, res.state.i_agg[l]);
    const size_t nk = res.model.kept_ids.size();
    std::vector<cx> i_kept(3 * nk, cx{});
    for (size_t k = 0; k < nk; ++k)
      for (int p = 0; p < 3; ++p) i_kept[3 * k + size_t(p)] = res.state.i_agg[l][size_t(3 * res.model.kept_ids[k] + p)];
    const std::vector<cx> v_kept = dense_anchored(res.model.y_kron, res.model.kept_phases, slack_pos, vs, i_kept);
    for (size_t k = 0; k < nk; ++k)
      for (int p = 0; p < 3; ++p) {
        if (!res.model.kept_phases[k].has(p)) continue;
        const double d = std::abs(v_kept[3 * k + size_t(p)] - v_full[size_t(3 * res.model.kept_ids[k] + p)]);
        worst = std::max(worst, d);
        CHECK(d < 1e-10);
      }
  }
  std::printf("commits %d kept %zu kron_consistency_max %.3e failures %d\n", commits, res.model.kept_ids.size(), worst,
              failures);
  return failures == 0 ? 0 : 1;
}
