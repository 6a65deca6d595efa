// Host side of the assignment (the integer half of Algorithm 1 plus the
// aggregated-injection bookkeeping), behaviour-matched to
//   init_state            reduce.cpp:39-61   identity assignment, adjacency lists
//   enumerate_candidates  reduce.cpp:63-73   s ascending, r ascending in lambda[s],
//                                            r != slack, phi(r) subset of phi(s)
//   commit                reduce.cpp:299-344 re-parent, contract lambda, move i_agg
//
// The device loop commits on the GPU; this state machine replays the committed
// trace so that clusters, the public AssignmentState (i_agg included) and the
// observer see exactly what the reference's state holds after each commit.
//
// Representation notes. The contraction of the super-node graph is done as a
// sorted-set union: lambda(s) := (lambda(s) U lambda(r)) \ {s, r}, and every
// neighbour t of r relabels its entry r -> s. i_agg is kept per scenario as 3n
// complex values; moving r onto s is the reference's complex `+=` (a pair of
// IEEE additions), so the mirror is bit-identical to the device copy.
#include <algorithm>
#include <iterator>

#include "kr_internal.hpp"

namespace kronred::b200 {

namespace {

// replace `from` by `to` in an ascending list that contains `from`
// (`to` may already be present: then `from` simply disappears)
void relabel_sorted(std::vector<int>& v, int from, int to) {
  const auto f = std::lower_bound(v.begin(), v.end(), from);
  if (f == v.end() || *f != from) return;
  v.erase(f);
  const auto t = std::lower_bound(v.begin(), v.end(), to);
  if (t == v.end() || *t != to) v.insert(t, to);
}

}  // namespace

void HostState::init(const Network& net, const std::vector<double>* injections, int scenarios) {
  n = net.size();
  slack = net.slack_id();
  sup.resize(size_t(n));
  supernodes.resize(size_t(n));
  members.assign(size_t(n), {});
  mask.resize(size_t(n));
  for (int i = 0; i < n; ++i) {
    sup[size_t(i)] = supernodes[size_t(i)] = i;
    members[size_t(i)].push_back(i);
    mask[size_t(i)] = net.nodes[size_t(i)].phases.bits;
  }
  // adjacency(net).neighbors(i): ascending and duplicate-free
  lambda = net.neighbor_lists();
  for (std::vector<int>& l : lambda) l.resize(size_t(std::unique(l.begin(), l.end()) - l.begin()));
  i_agg.clear();
  if (injections != nullptr) {
    const size_t dim = size_t(3 * n);
    i_agg.resize(size_t(scenarios));
    for (int l = 0; l < scenarios; ++l) {
      const double* src = injections->data() + size_t(l) * dim * 2;
      std::vector<cx>& dst = i_agg[size_t(l)];
      dst.resize(dim);
      for (size_t k = 0; k < dim; ++k) dst[k] = cx{src[2 * k], src[2 * k + 1]};
    }
  }
}

void HostState::enumerate(std::vector<int>& cs, std::vector<int>& cr) const {
  cs.clear();
  cr.clear();
  for (const int s : supernodes) {
    const unsigned ms = mask[size_t(s)];
    for (const int r : lambda[size_t(s)])
      if (r != slack && (mask[size_t(r)] | ms) == ms) {
        cs.push_back(s);
        cr.push_back(r);
      }
  }
}

void HostState::commit(int s, int r) {
  // the reference's preconditions and messages (reduce.cpp:302-307)
  if (r == slack) throw Error("commit: the slack node cannot be absorbed");
  const auto pos = std::lower_bound(supernodes.begin(), supernodes.end(), r);
  const bool r_active = pos != supernodes.end() && *pos == r;
  if (!r_active || members[size_t(s)].empty()) throw Error("commit: candidate references an inactive super-node");
  std::vector<int>& ns = lambda[size_t(s)];
  if (!std::binary_search(ns.begin(), ns.end(), r)) throw Error("commit: candidate nodes are not adjacent super-nodes");

  // cluster of r joins s (members keep the reference's append order)
  std::vector<int>& mr = members[size_t(r)];
  for (const int j : mr) sup[size_t(j)] = s;
  members[size_t(s)].insert(members[size_t(s)].end(), mr.begin(), mr.end());
  mr.clear();
  supernodes.erase(pos);

  // contracted adjacency: s inherits r's neighbours
  std::vector<int>& nr = lambda[size_t(r)];
  for (const int t : nr)
    if (t != s) relabel_sorted(lambda[size_t(t)], r, s);
  std::vector<int> joined;
  joined.reserve(ns.size() + nr.size());
  std::set_union(ns.begin(), ns.end(), nr.begin(), nr.end(), std::back_inserter(joined));
  joined.erase(std::remove_if(joined.begin(), joined.end(), [&](int t) { return t == s || t == r; }), joined.end());
  ns.swap(joined);
  nr.clear();

  // aggregated injections follow the assignment (all three phases)
  for (std::vector<cx>& v : i_agg)
    for (int p = 0; p < 3; ++p) {
      v[size_t(3 * s + p)] += v[size_t(3 * r + p)];
      v[size_t(3 * r + p)] = cx{};
    }
}

}  // namespace kronred::b200
