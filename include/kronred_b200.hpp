// kronred_b200.hpp — C++ drop-in API of the B200-native reduction.
//
// Same type names, fields and semantics as the reference's public C++ API
// (namespace kronred; proj/include/kronred/{phase,complex3,block_matrix,network,
// scenario,kron,reduce,radialize}.hpp) so a caller of
//   kronred::run_reduction(net, lib, cfg, observer)          (reduce.hpp:168-170)
//   kronred::radialize(model, net, y, &lib)                   (radialize.hpp:38-39)
//   kronred::kron_reduce(y, phases, partition)                (kron.hpp:33-34)
// relinks against libkronred_b200.so unchanged. The numeric work runs on an
// sm_100a device through the C ABI in kronred_b200.h; there is no CPU path.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace kronred {

using cx = std::complex<double>;

// --- errors (errors.hpp:10-37) -------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : Error {
  using Error::Error;
};
struct StructuralError : ValidationError {
  using ValidationError::ValidationError;
};
struct ConfigError : ValidationError {
  using ValidationError::ValidationError;
};
struct SolverError : Error {
  SolverError(const std::string& msg, double pivot = 0.0, int node_in = -1)
      : Error(msg), smallest_pivot(pivot), node(node_in) {}
  double smallest_pivot;
  int node;
};

// --- phases and 3x3 blocks (phase.hpp:13-52, complex3.hpp:15-124) --------
struct PhaseMask {
  std::uint8_t bits = 0;  // bit 0 = a, bit 1 = b, bit 2 = c
  static constexpr PhaseMask abc() { return PhaseMask{7}; }
  static constexpr PhaseMask none() { return PhaseMask{0}; }
  static PhaseMask parse(const std::string& s);
  std::string str() const;
  constexpr bool has(int p) const { return (bits >> p) & 1; }
  constexpr bool empty() const { return bits == 0; }
  constexpr int count() const { return (bits & 1) + ((bits >> 1) & 1) + ((bits >> 2) & 1); }
  constexpr bool subset_of(PhaseMask o) const { return (bits & ~o.bits) == 0; }
  constexpr PhaseMask intersect(PhaseMask o) const {
    return PhaseMask{static_cast<std::uint8_t>(bits & o.bits)};
  }
  friend constexpr bool operator==(PhaseMask a, PhaseMask b) { return a.bits == b.bits; }
};

struct Vec3c {
  std::array<cx, 3> v{};
  cx& operator[](int i) { return v[size_t(i)]; }
  const cx& operator[](int i) const { return v[size_t(i)]; }
};

struct Mat3c {
  std::array<cx, 9> m{};  // row-major
  cx& operator()(int r, int c) { return m[size_t(r * 3 + c)]; }
  const cx& operator()(int r, int c) const { return m[size_t(r * 3 + c)]; }
  static Mat3c identity();
  Mat3c transpose() const;
  Mat3c masked(PhaseMask mask) const;
  bool confined_to(PhaseMask mask) const;
  bool is_zero() const;
  double max_abs() const;
};

/// Node-indexed sparse matrix of 3x3 blocks (block_matrix.hpp:15-60).
class BlockMatrix {
 public:
  BlockMatrix() = default;
  explicit BlockMatrix(int n) : n_(n), rows_(size_t(n)) {}
  int n() const { return n_; }
  int scalar_dim() const { return 3 * n_; }
  Mat3c& block(int i, int j) { return rows_[size_t(i)][j]; }
  const Mat3c* find(int i, int j) const;
  const std::map<int, Mat3c>& row(int i) const { return rows_[size_t(i)]; }
  int block_count() const;
  double max_abs() const;
  void prune_zero_blocks();

 private:
  int n_ = 0;
  std::vector<std::map<int, Mat3c>> rows_;
};
using BlockAdmittance = BlockMatrix;

struct Adjacency {
  int n = 0;
  std::vector<std::uint8_t> a;
  Adjacency() = default;
  explicit Adjacency(int n_in) : n(n_in), a(size_t(n_in) * size_t(n_in), 0) {}
  bool at(int i, int j) const { return a[size_t(i) * size_t(n) + size_t(j)] != 0; }
  void set(int i, int j) {
    a[size_t(i) * size_t(n) + size_t(j)] = 1;
    a[size_t(j) * size_t(n) + size_t(i)] = 1;
  }
  std::vector<int> neighbors(int i) const;
  int edge_count() const;
};

// --- network (network.hpp:13-52) ------------------------------------------
struct Node {
  int id = -1;
  PhaseMask phases;
  bool is_slack = false;
  Vec3c slack_voltage;
};
struct Branch {
  int from = -1, to = -1;
  Mat3c y_series, shunt_from, shunt_to;
};
struct Network {
  std::vector<Node> nodes;
  std::vector<Branch> branches;
  int size() const { return int(nodes.size()); }
  int slack_id() const;
  std::vector<std::vector<int>> neighbor_lists() const;
};
Vec3c nominal_slack_voltage();
void validate_or_throw(const Network& net);
BlockAdmittance assemble_admittance(const Network& net);
std::vector<PhaseMask> phase_masks(const Network& net);
Adjacency adjacency(const Network& net);
Network read_network_json(const std::string& path);

// --- scenarios (scenario.hpp:15-33) ---------------------------------------
struct Scenario {
  std::string id;
  std::vector<cx> injections;  // 3n
  std::vector<cx> voltages;    // 3n
};
struct ScenarioLibrary {
  int n = 0;
  std::vector<Scenario> scenarios;
  int size() const { return int(scenarios.size()); }
  std::vector<std::string> ids() const;
};
/// load_library (scenario.cpp:141-220): constant-current or constant-PQ CSV,
/// voltages solved on the device.
ScenarioLibrary load_library(const Network& net, const std::string& path);

// --- reduction (reduce.hpp:19-170) ----------------------------------------
enum class Objective { magnitude, complex_error };
struct ReductionConfig {
  double e_bar = 1e-3;
  Objective objective = Objective::magnitude;
  std::optional<double> target_reduction;
  int workers = 1;
  bool use_delta = true;
  double topology_tol = 1e-9;
};
struct Candidate {
  int s = -1, r = -1;
};
struct AssignmentState {
  int n = 0;
  int slack = -1;
  std::vector<int> sup;
  std::vector<std::vector<int>> members;
  std::vector<int> supernodes;
  std::vector<std::vector<int>> lambda;
  std::vector<std::vector<cx>> i_agg;  // per scenario, 3n aggregated injections (reduce.hpp:53)
  int supernode_count() const { return int(supernodes.size()); }
  double reduction_fraction() const {
    return n == 0 ? 0.0 : double(n - supernode_count()) / double(n);
  }
};
struct TraceRow {
  int iteration = 0;
  int s = -1, r = -1;
  double smice = 0;
  std::vector<double> max_err;
  int supernode_count = 0;
  int candidate_count = 0;
  double wall_ms = 0;
};
struct ReducedModel {
  std::vector<int> kept_ids;
  std::vector<PhaseMask> kept_phases;
  BlockMatrix y_kron;
  std::map<int, std::vector<int>> clusters;
  bool radial = false;
  std::vector<int> reinserted;
  double e_bar = 0;
  Objective objective = Objective::magnitude;
  std::vector<std::string> scenario_ids;
  std::vector<double> final_max_err;
};
struct ReductionResult {
  ReducedModel model;
  std::vector<TraceRow> trace;
  AssignmentState state;
};
using IterationObserver = std::function<void(const AssignmentState&, const TraceRow&)>;

ReductionResult run_reduction(const Network& net, const ScenarioLibrary& lib,
                              const ReductionConfig& cfg,
                              const IterationObserver& observer = {});
/// The device engine behind run_reduction / model_max_errors is cached per
/// calling thread and reused for networks of the same structure (values are
/// re-uploaded; KRONRED_ENGINE_CACHE=0 disables). Frees it.
void release_engine_cache();

// --- Kron (kron.hpp:13-49) --------------------------------------------------
struct Partition {
  std::vector<int> keep, reduce;
};
struct KronResult {
  BlockMatrix y_kron;
  std::vector<int> kept_ids;
  std::vector<PhaseMask> kept_phases;
  int pos(int original_id) const;
};
void check_partition(const Partition& part, int n, int slack);
KronResult kron_reduce(const BlockMatrix& y, const std::vector<PhaseMask>& phases,
                       const Partition& part);
Adjacency block_topology(const BlockMatrix& y, double tol = 1e-9);

// --- radialization (radialize.hpp:14-39) -----------------------------------
struct Clique {
  std::vector<int> members;
};
std::vector<Clique> find_maximal_cliques(const Adjacency& adj);
std::vector<int> critical_nodes(const std::vector<int>& member_ids, const Network& original);
bool is_tree(const Adjacency& adj);
ReducedModel radialize(const ReducedModel& model, const Network& original, const BlockMatrix& y,
                       const ScenarioLibrary* lib = nullptr);
std::vector<double> model_max_errors(const ReducedModel& model, const Network& net,
                                     const ScenarioLibrary& lib);

// --- validation report (io.hpp:62-71, io.cpp:385-416) ----------------------
struct ValidateReport {
  std::vector<std::string> scenario_ids;
  std::vector<double> max_err;    // per scenario (model_max_errors, on the device)
  std::vector<double> bin_edges;  // histogram over max_err, size bins+1
  std::vector<int> bin_counts;    // size bins
};
ValidateReport make_validate_report(const ReducedModel& model, const Network& net, const ScenarioLibrary& lib,
                                    int bins = 20);
void write_validate_report(const ValidateReport& rep, const std::string& path);

// --- writers (io.cpp:216-359) ------------------------------------------------
std::string format_double(double v);
std::string reduced_json_string(const ReducedModel& model);
void write_reduced_json(const ReducedModel& model, const std::string& path);
void write_trace_csv(const std::string& path, const std::vector<TraceRow>& trace,
                     const std::vector<std::string>& scenario_ids,
                     const std::vector<double>& final_max_err,
                     const std::vector<std::string>& header_comments = {});

}  // namespace kronred
