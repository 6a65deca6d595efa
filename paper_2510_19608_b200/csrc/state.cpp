// Host assignment state machine: the integer half of Algorithm 1.
//   init_state            reduce.cpp:39-61   (identity assignment, tree adjacency)
//   enumerate_candidates  reduce.cpp:63-73   (s ascending, r ascending in lambda[s],
//                                             r != slack, phi(r) subset of phi(s))
//   commit                reduce.cpp:299-344 (re-parent, contract lambda)
// The floating-point half of commit (moving i_agg[r] onto s) runs on the
// device (engine.cu, commit_kernel).
#include <algorithm>

#include "kr_internal.hpp"

namespace kronred::b200 {

void HostState::init(const Network& net) {
  n = net.size();
  slack = net.slack_id();
  sup.resize(size_t(n));
  members.assign(size_t(n), {});
  supernodes.resize(size_t(n));
  mask.resize(size_t(n));
  for (int i = 0; i < n; ++i) {
    sup[size_t(i)] = i;
    members[size_t(i)] = {i};
    supernodes[size_t(i)] = i;
    mask[size_t(i)] = net.nodes[size_t(i)].phases.bits;
  }
  lambda = net.neighbor_lists();
  for (auto& l : lambda) l.erase(std::unique(l.begin(), l.end()), l.end());
}

void HostState::enumerate(std::vector<int>& cs, std::vector<int>& cr) const {
  cs.clear();
  cr.clear();
  for (int s : supernodes)
    for (int r : lambda[size_t(s)]) {
      if (r == slack) continue;
      if ((mask[size_t(r)] & ~mask[size_t(s)]) == 0) {
        cs.push_back(s);
        cr.push_back(r);
      }
    }
}

void HostState::commit(int s, int r) {
  if (r == slack) throw Error("commit: the slack node cannot be absorbed");
  auto sit = std::lower_bound(supernodes.begin(), supernodes.end(), r);
  if (sit == supernodes.end() || *sit != r || members[size_t(s)].empty())
    throw Error("commit: candidate references an inactive super-node");
  auto& ls = lambda[size_t(s)];
  if (!std::binary_search(ls.begin(), ls.end(), r))
    throw Error("commit: candidate nodes are not adjacent super-nodes");
  for (int j : members[size_t(r)]) sup[size_t(j)] = s;
  auto& ms = members[size_t(s)];
  auto& mr = members[size_t(r)];
  ms.insert(ms.end(), mr.begin(), mr.end());
  mr.clear();
  supernodes.erase(sit);
  auto erase_sorted = [](std::vector<int>& v, int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it != v.end() && *it == x) v.erase(it);
  };
  auto insert_sorted = [](std::vector<int>& v, int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it == v.end() || *it != x) v.insert(it, x);
  };
  auto& lr = lambda[size_t(r)];
  erase_sorted(ls, r);
  for (int t : lr) {
    if (t == s) continue;
    erase_sorted(lambda[size_t(t)], r);
    insert_sorted(lambda[size_t(t)], s);
    insert_sorted(ls, t);
  }
  lr.clear();
}

}  // namespace kronred::b200
