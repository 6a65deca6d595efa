// Symbolic block elimination and device work lists.
//
// Replays BlockElimination::eliminate (solver.cpp:20-117) on the block
// sparsity pattern: greedy minimum degree over the requested set, lowest id on
// ties (solver.cpp:55-65), couplings in ascending neighbour order
// (solver.cpp:84-91: std::map iteration), fill insertion and the degree
// bookkeeping of solver.cpp:94-106 (including the decrement on erase). It
// produces no numbers: the device executor (engine.cu) performs the implied
// pinv / Schur-contribution / ordered-apply work level by level.
//
// The min-degree choice is made with a lazy binary heap keyed (degree, id),
// which selects exactly the reference's O(n) scan result (minimum degree,
// lowest id among ties) in O(log n).
#include <algorithm>
#include <functional>
#include <map>
#include <queue>

#include "kr_internal.hpp"

namespace kronred::b200 {

ElimSchedule build_schedule(const FlatBlocks& y, const std::vector<std::uint8_t>& mask,
                            const std::vector<int>& elim_set) {
  const int n = y.n;
  ElimSchedule s;
  s.n = n;
  s.mask = mask;
  s.n_input = int(y.row.size());
  s.nblocks = s.n_input;

  // working pattern: row -> (col -> working block id)
  std::vector<std::map<int, int>> work(static_cast<size_t>(n));
  for (int b = 0; b < s.n_input; ++b) work[size_t(y.row[size_t(b)])][y.col[size_t(b)]] = b;

  std::vector<char> to_elim(size_t(n), 0);
  for (int k : elim_set) {
    if (k < 0 || k >= n) throw ValidationError("elimination set references unknown node");
    if (to_elim[size_t(k)]) throw ValidationError("elimination set repeats a node");
    to_elim[size_t(k)] = 1;
  }
  std::vector<int> degree(size_t(n), 0);
  for (int i = 0; i < n; ++i)
    for (const auto& kv : work[size_t(i)])
      if (kv.first != i) ++degree[size_t(i)];

  using Key = std::pair<int, int>;  // (degree, id)
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
  for (int i = 0; i < n; ++i)
    if (to_elim[size_t(i)]) heap.push({degree[size_t(i)], i});

  s.eliminated.assign(size_t(n), 0);
  s.node_step.assign(size_t(n), -1);
  std::vector<int> final_level;  // per working block
  final_level.assign(size_t(s.nblocks), 0);
  std::vector<std::vector<int>> blk_slots;  // per working block, slots in order
  blk_slots.resize(size_t(s.nblocks));
  auto new_block = [&]() {
    const int id = s.nblocks++;
    final_level.push_back(0);
    blk_slots.emplace_back();
    return id;
  };

  s.cpl_off.push_back(0);
  s.slot_off.push_back(0);
  size_t remaining = elim_set.size();
  while (remaining > 0) {
    int k = -1;
    while (!heap.empty()) {
      const Key top = heap.top();
      heap.pop();
      const int i = top.second;
      if (!to_elim[size_t(i)] || s.eliminated[size_t(i)] || top.first != degree[size_t(i)]) continue;
      k = i;
      break;
    }
    if (k < 0) throw Error("symbolic elimination: heap exhausted");
    const int step = s.nsteps++;
    auto& row_k = work[size_t(k)];
    auto dit = row_k.find(k);
    const int diag = dit == row_k.end() ? -1 : dit->second;

    // couplings: active neighbours in ascending id (map order)
    std::vector<int> cn, cto, cfrom;
    for (const auto& kv : row_k) {
      const int j = kv.first;
      if (j == k || s.eliminated[size_t(j)]) continue;
      cn.push_back(j);
      cto.push_back(kv.second);  // A[k][j]
      auto& row_j = work[size_t(j)];
      auto it = row_j.find(k);
      if (it == row_j.end()) it = row_j.emplace(k, -1).first;  // operator[] inserts a zero block
      cfrom.push_back(it->second);  // A[j][k]
    }
    int lvl = 0;
    auto rd = [&](int b) {
      if (b >= 0) lvl = std::max(lvl, final_level[size_t(b)]);
    };
    rd(diag);
    for (size_t c = 0; c < cn.size(); ++c) {
      rd(cto[c]);
      rd(cfrom[c]);
    }
    lvl += 1;

    // Schur update pattern on all coupling pairs (solver.cpp:94-106)
    for (size_t a = 0; a < cn.size(); ++a) {
      auto& row_i = work[size_t(cn[a])];
      for (size_t b = 0; b < cn.size(); ++b) {
        auto [it, inserted] = row_i.try_emplace(cn[b], -2);
        if (inserted) {
          it->second = new_block();
          if (cn[a] != cn[b]) ++degree[size_t(cn[a])];
        }
        const int target = it->second;
        const int slot = s.nslots++;
        s.slot_from.push_back(cfrom[a]);
        s.slot_to.push_back(cto[b]);
        s.slot_target.push_back(target);
        blk_slots[size_t(target)].push_back(slot);
        final_level[size_t(target)] = std::max(final_level[size_t(target)], lvl);
      }
      row_i.erase(k);
      --degree[size_t(cn[a])];
      if (to_elim[size_t(cn[a])]) heap.push({degree[size_t(cn[a])], cn[a]});
    }
    row_k.clear();

    s.step_node.push_back(k);
    s.step_diag.push_back(diag);
    s.step_level.push_back(lvl);
    for (size_t c = 0; c < cn.size(); ++c) {
      s.cpl_node.push_back(cn[c]);
      s.cpl_to.push_back(cto[c]);
      s.cpl_from.push_back(cfrom[c]);
    }
    s.cpl_off.push_back(int(s.cpl_node.size()));
    s.slot_off.push_back(s.nslots);
    s.eliminated[size_t(k)] = 1;
    s.node_step[size_t(k)] = step;
    s.nlevels = std::max(s.nlevels, lvl);
    --remaining;
  }

  // kept rows after elimination (schur_complement, solver.cpp:150-166)
  for (int i = 0; i < n; ++i) {
    if (s.eliminated[size_t(i)]) continue;
    s.kept.push_back(i);
    for (const auto& kv : work[size_t(i)]) {
      if (s.eliminated[size_t(kv.first)]) continue;
      s.rem_i.push_back(i);
      s.rem_j.push_back(kv.first);
      s.rem_blk.push_back(kv.second);
    }
  }

  // per-level work lists (levels 1..nlevels; index level-1)
  const int L = s.nlevels;
  s.lvl_step_off.assign(size_t(L) + 1, 0);
  for (int st = 0; st < s.nsteps; ++st) ++s.lvl_step_off[size_t(s.step_level[size_t(st)])];
  for (int l = 0; l < L; ++l) s.lvl_step_off[size_t(l) + 1] += s.lvl_step_off[size_t(l)];
  {
    std::vector<int> fill(s.lvl_step_off.begin(), s.lvl_step_off.end() - 1);
    s.lvl_steps.assign(size_t(s.nsteps), 0);
    for (int st = 0; st < s.nsteps; ++st)
      s.lvl_steps[size_t(fill[size_t(s.step_level[size_t(st)] - 1)]++)] = st;
  }
  s.lvl_slot_off.assign(size_t(L) + 1, 0);
  for (int st = 0; st < s.nsteps; ++st)
    s.lvl_slot_off[size_t(s.step_level[size_t(st)])] += s.slot_off[size_t(st) + 1] - s.slot_off[size_t(st)];
  for (int l = 0; l < L; ++l) s.lvl_slot_off[size_t(l) + 1] += s.lvl_slot_off[size_t(l)];
  {
    std::vector<int> fill(s.lvl_slot_off.begin(), s.lvl_slot_off.end() - 1);
    s.lvl_slots.assign(size_t(s.nslots), 0);
    s.lvl_slot_step.assign(size_t(s.nslots), 0);
    for (int st = 0; st < s.nsteps; ++st)
      for (int sl = s.slot_off[size_t(st)]; sl < s.slot_off[size_t(st) + 1]; ++sl) {
        const int pos = fill[size_t(s.step_level[size_t(st)] - 1)]++;
        s.lvl_slots[size_t(pos)] = sl;
        s.lvl_slot_step[size_t(pos)] = st;
      }
  }
  s.lvl_apply_off.assign(size_t(L) + 1, 0);
  for (int b = 0; b < s.nblocks; ++b)
    if (!blk_slots[size_t(b)].empty()) ++s.lvl_apply_off[size_t(final_level[size_t(b)])];
  for (int l = 0; l < L; ++l) s.lvl_apply_off[size_t(l) + 1] += s.lvl_apply_off[size_t(l)];
  {
    std::vector<int> fill(s.lvl_apply_off.begin(), s.lvl_apply_off.end() - 1);
    const int na = s.lvl_apply_off[size_t(L)];
    s.apply_blk.assign(size_t(na), 0);
    for (int b = 0; b < s.nblocks; ++b)
      if (!blk_slots[size_t(b)].empty())
        s.apply_blk[size_t(fill[size_t(final_level[size_t(b)] - 1)]++)] = b;
    s.apply_off.assign(size_t(na) + 1, 0);
    for (int a = 0; a < na; ++a) {
      const auto& sl = blk_slots[size_t(s.apply_blk[size_t(a)])];
      s.apply_off[size_t(a) + 1] = s.apply_off[size_t(a)] + int(sl.size());
      s.apply_slots.insert(s.apply_slots.end(), sl.begin(), sl.end());
    }
  }

  // forward pulls: rhs_c -= A[c][k] t_k for eliminated couplings c of step k,
  // applied by c in k's elimination order (solver.cpp:123-133)
  std::vector<std::vector<std::pair<int, int>>> pulls(static_cast<size_t>(n));  // by node: (source node, block)
  for (int st = 0; st < s.nsteps; ++st)
    for (int c = s.cpl_off[size_t(st)]; c < s.cpl_off[size_t(st) + 1]; ++c) {
      const int cnode = s.cpl_node[size_t(c)];
      if (s.eliminated[size_t(cnode)])
        pulls[size_t(cnode)].push_back({s.step_node[size_t(st)], s.cpl_from[size_t(c)]});
    }
  s.in_off.assign(size_t(s.nsteps) + 1, 0);
  std::vector<int> flev(size_t(s.nsteps), 0), blev(size_t(s.nsteps), 0);
  for (int st = 0; st < s.nsteps; ++st) {
    const auto& pl = pulls[size_t(s.step_node[size_t(st)])];
    int lv = 0;
    for (const auto& pr : pl) {
      s.in_node.push_back(pr.first);
      s.in_blk.push_back(pr.second);
      lv = std::max(lv, flev[size_t(s.node_step[size_t(pr.first)])] + 1);
    }
    s.in_off[size_t(st) + 1] = int(s.in_node.size());
    flev[size_t(st)] = lv;
    s.nfw = std::max(s.nfw, lv + 1);
  }
  for (int st = s.nsteps - 1; st >= 0; --st) {
    int lv = 0;
    for (int c = s.cpl_off[size_t(st)]; c < s.cpl_off[size_t(st) + 1]; ++c) {
      const int cnode = s.cpl_node[size_t(c)];
      if (s.eliminated[size_t(cnode)]) lv = std::max(lv, blev[size_t(s.node_step[size_t(cnode)])] + 1);
    }
    blev[size_t(st)] = lv;
    s.nbw = std::max(s.nbw, lv + 1);
  }
  auto group = [&](const std::vector<int>& lev, int nl, std::vector<int>& off, std::vector<int>& out) {
    off.assign(size_t(nl) + 1, 0);
    for (int st = 0; st < s.nsteps; ++st) ++off[size_t(lev[size_t(st)]) + 1];
    for (int l = 0; l < nl; ++l) off[size_t(l) + 1] += off[size_t(l)];
    std::vector<int> fill(off.begin(), off.end() - 1);
    out.assign(size_t(s.nsteps), 0);
    for (int st = 0; st < s.nsteps; ++st) out[size_t(fill[size_t(lev[size_t(st)])]++)] = st;
  };
  group(flev, s.nfw, s.fw_off, s.fw_steps);
  group(blev, s.nbw, s.bw_off, s.bw_steps);
  return s;
}

}  // namespace kronred::b200
