// Host input path: phases, 3x3 blocks, network validation, admittance
// assembly, network-JSON and scenario-CSV parsing. Integer/bookkeeping work
// plus the exact (branch-order) Y assembly; no solves happen here.
//
// Reference semantics followed:
//   PhaseMask             phase.hpp:13-52
//   Mat3c helpers         complex3.hpp:38-124
//   validate              network.cpp:46-188
//   assemble_admittance   grid_model.cpp:17-74
//   parse_network_json    io.cpp:138-166 (nlohmann number semantics)
//   load_library CSV      scenario.cpp:100-212
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <numbers>
#include <queue>
#include <set>
#include <sstream>

#include "kr_internal.hpp"

namespace kronred {

// --- PhaseMask / Mat3c / BlockMatrix ------------------------------------------

PhaseMask PhaseMask::parse(const std::string& s) {
  PhaseMask m;
  for (char c : s) {
    if (c == 'a')
      m.bits |= 1;
    else if (c == 'b')
      m.bits |= 2;
    else if (c == 'c')
      m.bits |= 4;
    else
      throw ValidationError("invalid phase string '" + s + "'");
  }
  return m;
}

std::string PhaseMask::str() const {
  std::string s;
  for (int p = 0; p < 3; ++p)
    if (has(p)) s += char('a' + p);
  return s;
}

Mat3c Mat3c::identity() {
  Mat3c r;
  for (int i = 0; i < 3; ++i) r(i, i) = 1.0;
  return r;
}

Mat3c Mat3c::transpose() const {
  Mat3c r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (*this)(j, i);
  return r;
}

Mat3c Mat3c::masked(PhaseMask mask) const {
  Mat3c r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (mask.has(i) && mask.has(j)) r(i, j) = (*this)(i, j);
  return r;
}

bool Mat3c::confined_to(PhaseMask mask) const {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (!(mask.has(i) && mask.has(j)) && (*this)(i, j) != cx{}) return false;
  return true;
}

bool Mat3c::is_zero() const {
  return std::all_of(m.begin(), m.end(), [](const cx& z) { return z == cx{}; });
}

double Mat3c::max_abs() const {
  double r = 0;
  for (const cx& z : m) r = std::max(r, std::abs(z));
  return r;
}

const Mat3c* BlockMatrix::find(int i, int j) const {
  const auto& r = rows_[size_t(i)];
  auto it = r.find(j);
  return it == r.end() ? nullptr : &it->second;
}

int BlockMatrix::block_count() const {
  int c = 0;
  for (const auto& r : rows_) c += int(r.size());
  return c;
}

double BlockMatrix::max_abs() const {
  double m = 0;
  for (const auto& r : rows_)
    for (const auto& kv : r) m = std::max(m, kv.second.max_abs());
  return m;
}

void BlockMatrix::prune_zero_blocks() {
  for (auto& r : rows_)
    std::erase_if(r, [](const auto& kv) { return kv.second.is_zero(); });
}

std::vector<int> Adjacency::neighbors(int i) const {
  std::vector<int> v;
  for (int j = 0; j < n; ++j)
    if (at(i, j)) v.push_back(j);
  return v;
}

int Adjacency::edge_count() const {
  int c = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) c += at(i, j);
  return c;
}

// --- network --------------------------------------------------------------------

int Network::slack_id() const {
  int found = -1;
  for (const Node& nd : nodes)
    if (nd.is_slack) {
      if (found >= 0) return -1;
      found = nd.id;
    }
  return found;
}

std::vector<std::vector<int>> Network::neighbor_lists() const {
  std::vector<std::vector<int>> adj(nodes.size());
  for (const Branch& b : branches)
    if (b.from >= 0 && b.from < size() && b.to >= 0 && b.to < size()) {
      adj[size_t(b.from)].push_back(b.to);
      adj[size_t(b.to)].push_back(b.from);
    }
  for (auto& l : adj) std::sort(l.begin(), l.end());
  return adj;
}

Vec3c nominal_slack_voltage() {
  const double th = 2.0 * std::numbers::pi / 3.0;
  Vec3c v;
  v[0] = cx{1.0, 0.0};
  v[1] = cx{std::cos(-th), std::sin(-th)};
  v[2] = cx{std::cos(th), std::sin(th)};
  return v;
}

std::vector<PhaseMask> phase_masks(const Network& net) {
  std::vector<PhaseMask> m(net.nodes.size());
  for (const Node& nd : net.nodes) m[size_t(nd.id)] = nd.phases;
  return m;
}

Adjacency adjacency(const Network& net) {
  Adjacency a(net.size());
  for (const Branch& b : net.branches) a.set(b.from, b.to);
  return a;
}

namespace {

void violation(std::ostringstream& os, int& count, const char* code, const std::string& d) {
  os << code << ": " << d << "\n";
  ++count;
}

}  // namespace

void validate_or_throw(const Network& net) {
  // Invariants of network.cpp:46-188, same codes, report-then-throw.
  std::ostringstream os;
  int bad = 0;
  const int n = net.size();
  if (n == 0) throw ValidationError("invalid network:\nempty: network has no nodes\n");
  for (int i = 0; i < n; ++i) {
    const Node& nd = net.nodes[size_t(i)];
    if (nd.id != i) violation(os, bad, "node-id", "node ids must be dense 0..n-1");
    if (nd.phases.empty())
      violation(os, bad, "empty-phase-mask", "node " + std::to_string(i) + " carries no phases");
  }
  int slack_count = 0, slack = -1;
  for (const Node& nd : net.nodes)
    if (nd.is_slack) {
      ++slack_count;
      slack = nd.id;
    }
  if (slack_count != 1)
    violation(os, bad, "slack-count", std::to_string(slack_count) + " slack nodes (need exactly 1)");
  if (slack_count == 1 && (slack < 0 || slack >= n || !(net.nodes[size_t(slack)].phases == PhaseMask::abc())))
    violation(os, bad, "slack-phases", "slack node must carry all three phases");
  // duplicate endpoint pairs: every later branch of a pair reported, in branch order
  std::vector<char> dup(net.branches.size(), 0);
  {
    std::vector<std::pair<std::pair<int, int>, size_t>> keys;
    keys.reserve(net.branches.size());
    for (size_t bi = 0; bi < net.branches.size(); ++bi) {
      const Branch& b = net.branches[bi];
      if (b.from < 0 || b.from >= n || b.to < 0 || b.to >= n || b.from == b.to) continue;
      keys.push_back({std::minmax(b.from, b.to), bi});
    }
    std::sort(keys.begin(), keys.end());
    for (size_t i = 1; i < keys.size(); ++i)
      if (keys[i].first == keys[i - 1].first) dup[keys[i].second] = 1;
  }
  for (size_t bi = 0; bi < net.branches.size(); ++bi) {
    const Branch& b = net.branches[bi];
    if (b.from < 0 || b.from >= n || b.to < 0 || b.to >= n) {
      violation(os, bad, "branch-endpoint", "branch #" + std::to_string(bi) + " references unknown node");
      continue;
    }
    if (b.from == b.to) {
      violation(os, bad, "self-loop", "branch #" + std::to_string(bi));
      continue;
    }
    if (dup[bi]) violation(os, bad, "duplicate-branch", "branch #" + std::to_string(bi));
    const PhaseMask common = net.nodes[size_t(b.from)].phases.intersect(net.nodes[size_t(b.to)].phases);
    if (!b.y_series.confined_to(common))
      violation(os, bad, "branch-phase-leak", "branch #" + std::to_string(bi));
    if (!b.shunt_from.confined_to(net.nodes[size_t(b.from)].phases))
      violation(os, bad, "shunt-phase-leak", "branch #" + std::to_string(bi));
    if (!b.shunt_to.confined_to(net.nodes[size_t(b.to)].phases))
      violation(os, bad, "shunt-phase-leak", "branch #" + std::to_string(bi));
  }
  if (int(net.branches.size()) != n - 1)
    violation(os, bad, "not-radial", std::to_string(net.branches.size()) + " branches for " +
                                         std::to_string(n) + " nodes");
  // adjacency with branch ids (CSR; per node in branch order, as neighbor_lists)
  std::vector<int> aoff(size_t(n) + 1, 0), adj_n, adj_b;
  for (const Branch& b : net.branches)
    if (b.from >= 0 && b.from < n && b.to >= 0 && b.to < n && b.from != b.to) {
      ++aoff[size_t(b.from) + 1];
      ++aoff[size_t(b.to) + 1];
    }
  for (int i = 0; i < n; ++i) aoff[size_t(i) + 1] += aoff[size_t(i)];
  adj_n.resize(size_t(aoff[size_t(n)]));
  adj_b.resize(adj_n.size());
  {
    std::vector<int> fill(aoff.begin(), aoff.end() - 1);
    for (size_t bi = 0; bi < net.branches.size(); ++bi) {
      const Branch& b = net.branches[bi];
      if (b.from < 0 || b.from >= n || b.to < 0 || b.to >= n || b.from == b.to) continue;
      adj_n[size_t(fill[size_t(b.from)])] = b.to;
      adj_b[size_t(fill[size_t(b.from)]++)] = int(bi);
      adj_n[size_t(fill[size_t(b.to)])] = b.from;
      adj_b[size_t(fill[size_t(b.to)]++)] = int(bi);
    }
  }
  const int root = slack_count == 1 && slack >= 0 && slack < n ? slack : 0;
  std::vector<int> parent(size_t(n), -2), pbranch(size_t(n), -1);
  std::vector<int> q;
  q.reserve(size_t(n));
  q.push_back(root);
  parent[size_t(root)] = -1;
  for (size_t h = 0; h < q.size(); ++h) {
    const int u = q[h];
    for (int e = aoff[size_t(u)]; e < aoff[size_t(u) + 1]; ++e) {
      const int v = adj_n[size_t(e)];
      if (parent[size_t(v)] == -2) {
        parent[size_t(v)] = u;
        pbranch[size_t(v)] = adj_b[size_t(e)];
        q.push_back(v);
      }
    }
  }
  const int reached = int(q.size());
  if (reached != n) violation(os, bad, "disconnected", std::to_string(n - reached) + " nodes unreachable");
  if (slack_count == 1 && reached == n && int(net.branches.size()) == n - 1) {
    for (int v = 0; v < n; ++v) {
      if (v == slack || parent[size_t(v)] < 0) continue;
      const PhaseMask child = net.nodes[size_t(v)].phases;
      const PhaseMask par = net.nodes[size_t(parent[size_t(v)])].phases;
      if (!child.subset_of(par))
        violation(os, bad, "phase-monotonicity", "node " + std::to_string(v) + " widens its parent's phases");
      const Branch* b = &net.branches[size_t(pbranch[size_t(v)])];
      for (int p = 0; p < 3 && b != nullptr; ++p) {
        if (!child.has(p)) continue;
        bool coupled = false;
        for (int c = 0; c < 3; ++c) coupled = coupled || b->y_series(p, c) != cx{};
        if (!coupled)
          violation(os, bad, "disconnected-phase",
                    "phase " + std::string(1, char('a' + p)) + " of node " + std::to_string(v));
      }
    }
  }
  if (bad) throw ValidationError("invalid network:\n" + os.str());
}

BlockAdmittance assemble_admittance(const Network& net) {
  // Branch-list order matters for the diagonal bits (grid_model.cpp:22-33).
  const int n = net.size();
  BlockAdmittance y(n);
  std::set<std::pair<int, int>> seen;
  for (const Branch& b : net.branches) {
    const auto key = std::minmax(b.from, b.to);
    if (!seen.insert(key).second)
      throw StructuralError("duplicate branch (" + std::to_string(key.first) + "," +
                            std::to_string(key.second) + ")");
    const Mat3c yt = b.y_series.transpose();
    Mat3c& ft = y.block(b.from, b.to);
    for (int k = 0; k < 9; ++k) ft.m[size_t(k)] -= b.y_series.m[size_t(k)];
    Mat3c& tf = y.block(b.to, b.from);
    for (int k = 0; k < 9; ++k) tf.m[size_t(k)] -= yt.m[size_t(k)];
    Mat3c& ff = y.block(b.from, b.from);
    for (int k = 0; k < 9; ++k) ff.m[size_t(k)] += b.y_series.m[size_t(k)];
    Mat3c& tt = y.block(b.to, b.to);
    for (int k = 0; k < 9; ++k) tt.m[size_t(k)] += yt.m[size_t(k)];
    Mat3c& ff2 = y.block(b.from, b.from);
    for (int k = 0; k < 9; ++k) ff2.m[size_t(k)] += b.shunt_from.m[size_t(k)];
    Mat3c& tt2 = y.block(b.to, b.to);
    for (int k = 0; k < 9; ++k) tt2.m[size_t(k)] += b.shunt_to.m[size_t(k)];
  }
  // mask every stored block to present phases (grid_model.cpp:36-50); only
  // the row's stored blocks are visited (O(blocks), not O(n^2) lookups)
  std::vector<int> cols;
  for (int i = 0; i < n; ++i) {
    const PhaseMask mi = net.nodes[size_t(i)].phases;
    cols.clear();
    for (const auto& kv : y.row(i)) cols.push_back(kv.first);
    for (const int j : cols) {
      Mat3c& blk = y.block(i, j);
      const PhaseMask mj = net.nodes[size_t(j)].phases;
      Mat3c masked;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          if (mi.has(r) && mj.has(c)) masked(r, c) = blk(r, c);
      blk = masked;
    }
  }
  for (int i = 0; i < n; ++i) {
    if (net.nodes[size_t(i)].is_slack) continue;
    const PhaseMask mi = net.nodes[size_t(i)].phases;
    for (int p = 0; p < 3; ++p) {
      if (!mi.has(p)) continue;
      bool nonzero = false;
      for (const auto& kv : y.row(i))
        for (int c = 0; c < 3; ++c) nonzero = nonzero || kv.second(p, c) != cx{};
      if (!nonzero)
        throw StructuralError("phase " + std::string(1, char('a' + p)) + " of node " +
                              std::to_string(i) + " has an all-zero admittance row");
    }
  }
  y.prune_zero_blocks();
  return y;
}

std::vector<std::string> ScenarioLibrary::ids() const {
  std::vector<std::string> r;
  for (const Scenario& s : scenarios) r.push_back(s.id);
  return r;
}

int KronResult::pos(int original_id) const {
  auto it = std::lower_bound(kept_ids.begin(), kept_ids.end(), original_id);
  return (it == kept_ids.end() || *it != original_id) ? -1 : int(it - kept_ids.begin());
}

// Host Gauss-Jordan inverse of the present-phase submatrix, used only to turn
// an input z_block into y_series while parsing (io.cpp:155-159 semantics).
static bool host_masked_inverse(const Mat3c& in, PhaseMask mask, Mat3c& out) {
  out = Mat3c{};
  int idx[3], k = 0;
  for (int p = 0; p < 3; ++p)
    if (mask.has(p)) idx[k++] = p;
  if (k == 0) return true;
  cx a[3][3], inv[3][3] = {};
  for (int i = 0; i < k; ++i) {
    inv[i][i] = 1.0;
    for (int j = 0; j < k; ++j) a[i][j] = in(idx[i], idx[j]);
  }
  for (int col = 0; col < k; ++col) {
    int piv = col;
    double best = std::abs(a[col][col]);
    for (int r = col + 1; r < k; ++r)
      if (std::abs(a[r][col]) > best) {
        best = std::abs(a[r][col]);
        piv = r;
      }
    if (best <= 1e-13) return false;
    if (piv != col)
      for (int j = 0; j < 3; ++j) {
        std::swap(a[piv][j], a[col][j]);
        std::swap(inv[piv][j], inv[col][j]);
      }
    const cx d = a[col][col];
    for (int j = 0; j < k; ++j) {
      a[col][j] /= d;
      inv[col][j] /= d;
    }
    for (int r = 0; r < k; ++r) {
      if (r == col) continue;
      const cx f = a[r][col];
      if (f == cx{}) continue;
      for (int j = 0; j < k; ++j) {
        a[r][j] -= f * a[col][j];
        inv[r][j] -= f * inv[col][j];
      }
    }
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) out(idx[i], idx[j]) = inv[i][j];
  return true;
}

// --- minimal JSON reader ---------------------------------------------------------
// Numbers follow nlohmann/json 3.x: a token without '.', 'e' or 'E' is an
// integer (so "-0" reads back as +0.0), otherwise strtod (correctly rounded).
namespace {

struct JVal {
  enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool is_number() const { return kind == Int || kind == Float; }
  double num() const { return kind == Int ? double(i) : d; }
};

struct JParser {
  const char* p;
  const char* e;
  [[noreturn]] void fail() { throw ValidationError("network: malformed JSON"); }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  JVal parse() {
    ws();
    if (p >= e) fail();
    JVal v;
    const char c = *p;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      for (;;) {
        ws();
        JVal k = parse();
        if (k.kind != JVal::Str) fail();
        ws();
        if (p >= e || *p != ':') fail();
        ++p;
        v.obj.emplace_back(k.s, parse());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return v;
        }
        fail();
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      for (;;) {
        v.arr.push_back(parse());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return v;
        }
        fail();
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      ++p;
      while (p < e && *p != '"') {
        if (*p == '\\') {
          ++p;
          if (p >= e) fail();
          const char x = *p;
          v.s += x == 'n' ? '\n' : x == 't' ? '\t' : x == 'r' ? '\r' : x;
        } else {
          v.s += *p;
        }
        ++p;
      }
      if (p >= e) fail();
      ++p;
      return v;
    }
    if (std::strncmp(p, "true", 4) == 0) {
      v.kind = JVal::Bool;
      v.b = true;
      p += 4;
      return v;
    }
    if (std::strncmp(p, "false", 5) == 0) {
      v.kind = JVal::Bool;
      p += 5;
      return v;
    }
    if (std::strncmp(p, "null", 4) == 0) {
      p += 4;
      return v;
    }
    const char* start = p;
    bool is_float = false;
    while (p < e && (std::isdigit((unsigned char)*p) || *p == '-' || *p == '+' || *p == '.' ||
                     *p == 'e' || *p == 'E')) {
      if (*p == '.' || *p == 'e' || *p == 'E') is_float = true;
      ++p;
    }
    if (p == start) fail();
    const std::string tok(start, p);
    if (!is_float) {
      errno = 0;
      char* endp = nullptr;
      const long long iv = std::strtoll(tok.c_str(), &endp, 10);
      if (errno == 0 && endp && *endp == 0) {
        v.kind = JVal::Int;
        v.i = iv;
        return v;
      }
    }
    v.kind = JVal::Float;
    v.d = std::strtod(tok.c_str(), nullptr);
    return v;
  }
};

cx json_pair(const JVal& j, const std::string& ctx) {
  if (j.kind != JVal::Arr || j.arr.size() != 2 || !j.arr[0].is_number() || !j.arr[1].is_number())
    throw ValidationError(ctx + ": expected [re,im]");
  return {j.arr[0].num(), j.arr[1].num()};
}

Mat3c json_block(const JVal& j, const std::string& ctx) {
  if (j.kind != JVal::Arr || j.arr.size() != 9)
    throw ValidationError(ctx + ": expected 9 [re,im] pairs, row-major");
  Mat3c b;
  for (int k = 0; k < 9; ++k) b.m[size_t(k)] = json_pair(j.arr[size_t(k)], ctx);
  return b;
}

std::string read_text(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ValidationError("cannot open '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

}  // namespace

Network parse_network_text(const std::string& text) {
  JParser jp{text.data(), text.data() + text.size()};
  const JVal root = jp.parse();
  const JVal* jn = root.get("nodes");
  const JVal* jb = root.get("branches");
  if (jn == nullptr || jn->kind != JVal::Arr) throw ValidationError("network: missing 'nodes' array");
  if (jb == nullptr || jb->kind != JVal::Arr) throw ValidationError("network: missing 'branches' array");
  Network net;
  for (const JVal& nj : jn->arr) {
    Node nd;
    const JVal* id = nj.get("id");
    if (id == nullptr || id->kind != JVal::Int) throw ValidationError("network: node without integer id");
    nd.id = int(id->i);
    const JVal* ph = nj.get("phases");
    if (ph == nullptr || ph->kind != JVal::Str)
      throw ValidationError("network: node " + std::to_string(nd.id) + " without phases");
    nd.phases = PhaseMask::parse(ph->s);
    const JVal* sl = nj.get("slack");
    nd.is_slack = sl != nullptr && sl->kind == JVal::Bool && sl->b;
    if (nd.is_slack) {
      const JVal* sv = nj.get("slack_voltage");
      if (sv != nullptr) {
        if (sv->kind != JVal::Arr || sv->arr.size() != 3)
          throw ValidationError("network: slack_voltage needs 3 [re,im] pairs");
        for (int p = 0; p < 3; ++p) nd.slack_voltage[p] = json_pair(sv->arr[size_t(p)], "slack_voltage");
      } else {
        nd.slack_voltage = nominal_slack_voltage();
      }
    }
    net.nodes.push_back(nd);
  }
  std::stable_sort(net.nodes.begin(), net.nodes.end(),
                   [](const Node& a, const Node& b) { return a.id < b.id; });
  for (const JVal& bj : jb->arr) {
    Branch b;
    const JVal* f = bj.get("from");
    const JVal* t = bj.get("to");
    if (f == nullptr || t == nullptr) throw ValidationError("network: branch without endpoints");
    b.from = int(f->num());
    b.to = int(t->num());
    const std::string ctx = "branch (" + std::to_string(b.from) + "," + std::to_string(b.to) + ")";
    if (b.from < 0 || b.from >= net.size() || b.to < 0 || b.to >= net.size())
      throw ValidationError(ctx + ": unknown endpoint");
    const JVal* zb = bj.get("z_block");
    const JVal* yb = bj.get("y_block");
    if ((zb != nullptr) == (yb != nullptr))
      throw ValidationError(ctx + ": exactly one of z_block / y_block required");
    const PhaseMask common = net.nodes[size_t(b.from)].phases.intersect(net.nodes[size_t(b.to)].phases);
    if (yb != nullptr) {
      b.y_series = json_block(*yb, ctx).masked(common);
    } else if (!host_masked_inverse(json_block(*zb, ctx).masked(common), common, b.y_series)) {
      throw ValidationError(ctx + ": z_block singular on the common phases");
    }
    if (const JVal* s = bj.get("shunt_from"))
      b.shunt_from = json_block(*s, ctx).masked(net.nodes[size_t(b.from)].phases);
    if (const JVal* s = bj.get("shunt_to"))
      b.shunt_to = json_block(*s, ctx).masked(net.nodes[size_t(b.to)].phases);
    net.branches.push_back(b);
  }
  return net;
}

Network read_network_json(const std::string& path) { return parse_network_text(read_text(path)); }

namespace b200 {

FlatBlocks FlatBlocks::from(const BlockMatrix& y) {
  FlatBlocks f;
  f.n = y.n();
  f.row_off.assign(size_t(f.n) + 1, 0);
  size_t nblk = 0;
  for (int i = 0; i < f.n; ++i) nblk += y.row(i).size();
  f.row.reserve(nblk);
  f.col.reserve(nblk);
  f.val.reserve(nblk * 18);
  for (int i = 0; i < f.n; ++i) {
    for (const auto& kv : y.row(i)) {
      f.row.push_back(i);
      f.col.push_back(kv.first);
      for (int k = 0; k < 9; ++k) {
        f.val.push_back(kv.second.m[size_t(k)].real());
        f.val.push_back(kv.second.m[size_t(k)].imag());
      }
    }
    f.row_off[size_t(i) + 1] = int(f.row.size());
  }
  return f;
}

double FlatBlocks::max_abs() const {
  double m = 0;
  for (size_t b = 0; b < row.size(); ++b)
    for (int k = 0; k < 9; ++k) m = std::max(m, std::abs(cx{val[b * 18 + 2 * k], val[b * 18 + 2 * k + 1]}));
  return m;
}

Network network_from_c(const krg_network* cn) {
  if (cn == nullptr || cn->n_nodes < 0 || cn->n_branches < 0)
    throw ValidationError("krg_network: null or negative sizes");
  Network net;
  net.nodes.resize(size_t(cn->n_nodes));
  for (int i = 0; i < cn->n_nodes; ++i) {
    Node& nd = net.nodes[size_t(i)];
    nd.id = i;
    nd.phases.bits = cn->phases[i];
    nd.is_slack = (i == cn->slack);
    if (nd.is_slack)
      for (int p = 0; p < 3; ++p)
        nd.slack_voltage[p] = cx{cn->slack_voltage[2 * p], cn->slack_voltage[2 * p + 1]};
  }
  auto blk = [](const double* v, size_t b) {
    Mat3c m;
    if (v == nullptr) return m;
    for (int k = 0; k < 9; ++k) m.m[size_t(k)] = cx{v[b * 18 + 2 * k], v[b * 18 + 2 * k + 1]};
    return m;
  };
  for (int b = 0; b < cn->n_branches; ++b) {
    Branch br;
    br.from = cn->br_from[b];
    br.to = cn->br_to[b];
    br.y_series = blk(cn->y_series, size_t(b));
    br.shunt_from = blk(cn->shunt_from, size_t(b));
    br.shunt_to = blk(cn->shunt_to, size_t(b));
    net.branches.push_back(br);
  }
  return net;
}

void validate_network(const Network& net) { validate_or_throw(net); }

}  // namespace b200
}  // namespace kronred
