// Internal types of libkronred_b200: host-side symbolic schedules (integer
// work only), the assignment state machine, and the device engine interface.
// No CUDA types appear here; engine.cu implements the Engine class.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "kronred_b200.h"
#include "kronred_b200.hpp"

namespace kronred::b200 {

struct CudaError : Error {
  using Error::Error;
};

// Thread-local error state behind krg_last_error().
void set_error(const std::string& msg, double pivot = 0.0, int node = -1);
int status_from_current_exception();

// ---------------------------------------------------------------------------
// Flattened block matrix: blocks in (row ascending, col ascending) order, the
// order a std::map-row BlockMatrix iterates (block_matrix.hpp:15-60).
struct FlatBlocks {
  int n = 0;
  std::vector<int> row, col;   // per block
  std::vector<double> val;     // per block 18 doubles (9 complex, row-major)
  std::vector<int> row_off;    // CSR over rows (n+1)
  static FlatBlocks from(const BlockMatrix& y);
  double max_abs() const;      // BlockMatrix::max_abs (uses std::abs = cabs)
};

// ---------------------------------------------------------------------------
// Symbolic block elimination. Replays BlockElimination::eliminate
// (solver.cpp:20-117) on the sparsity pattern only: greedy minimum degree with
// lowest-id ties, fill creation, degree bookkeeping and coupling order are the
// reference's; the numeric work it implies is emitted as a level-scheduled DAG
// for the device executor.
//
// Levels. Step k reads blocks (k,k), (k,c), (c,k); every Schur contribution
// (c_i,c_j) -= (A_ik pinv_k) A_kj is stored in its own slot and a block applies
// its slots in elimination order once the last one is computed ("pull"), so a
// block's bits equal the reference's sequential update chain. level(k) = 1 +
// max final level of the blocks it reads; final(B) = max level of B's writers.
struct ElimSchedule {
  int n = 0;
  std::vector<std::uint8_t> mask;     // per node
  int n_input = 0;                    // input blocks (FlatBlocks order)
  int nblocks = 0;                    // working blocks: [0,n_input) input, rest fill
  int nsteps = 0, nslots = 0, nlevels = 0;
  // steps (elimination order)
  std::vector<int> step_node, step_diag, step_level;
  std::vector<int> cpl_off, cpl_node, cpl_to, cpl_from;   // couplings, ascending node id
  // slots (Schur contributions), grouped by step
  std::vector<int> slot_off, slot_from, slot_to, slot_target;
  // per-level work lists
  std::vector<int> lvl_step_off, lvl_steps;
  std::vector<int> lvl_slot_off, lvl_slots, lvl_slot_step;
  std::vector<int> lvl_apply_off, apply_blk, apply_off, apply_slots;
  // solve (solve_interior, solver.cpp:119-148), pull form
  std::vector<char> eliminated;        // per node
  std::vector<int> node_step;          // per node, -1 when kept
  std::vector<int> in_off, in_node, in_blk;   // per step: ordered forward pulls
  int nfw = 0, nbw = 0;
  std::vector<int> fw_off, fw_steps, bw_off, bw_steps;
  // kept rows after elimination: (i, j, working block), i then j ascending
  std::vector<int> rem_i, rem_j, rem_blk;
  std::vector<int> kept;               // ascending kept node ids
};

ElimSchedule build_schedule(const FlatBlocks& y, const std::vector<std::uint8_t>& mask,
                            const std::vector<int>& elim_set);

// ---------------------------------------------------------------------------
// Host assignment state machine (reduce.cpp:39-73, 299-344): the public
// AssignmentState (so observers receive it without a copy) plus phase masks.
struct HostState : AssignmentState {
  std::vector<std::uint8_t> mask;
  // injections: [L][3n][2] scenario currents (the i_agg mirror), or null
  void init(const Network& net, const std::vector<double>* injections = nullptr, int scenarios = 0);
  void enumerate(std::vector<int>& cs, std::vector<int>& cr) const;
  void commit(int s, int r);
};

// ---------------------------------------------------------------------------
// Problem as handed to the device: validated network, assembled Y.
struct Problem {
  Network net;
  std::vector<std::uint8_t> mask;
  int slack = -1;
  FlatBlocks y;
  std::vector<std::string> scenario_ids;
  int L = 0;
  std::vector<double> injections;  // [L][3n][2]
  std::vector<double> voltages;    // [L][3n][2] (empty: device solve)
};

// Network from the C struct (copy) and back.
Network network_from_c(const krg_network* cn);
void validate_network(const Network& net);  // throws ValidationError

// ---------------------------------------------------------------------------
// Device engine (engine.cu).
struct ResultData {
  ReducedModel model;
  std::vector<TraceRow> trace;
  long long total_candidates = 0;
  int L = 0;
  HostState state;
  double device_ms = 0;  // CUDA-event time of the whole run on the engine stream
};

struct KernelStats {
  long long launches = 0;
  double ms = 0, flops = 0, bytes = 0;  // summed over launches (algorithmic work)
};

class Engine {
 public:
  Engine(const Problem& prob, int device);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Problem& problem() const;
  std::int64_t launches() const;
  bool last_run_device_loop() const;
  void set_profile(bool on);
  KernelStats stats(int which) const;  // 0 = scorer (score1 when it runs), 1 = base-refresh solve, 2 = score3 next to score1
  void set_exchange(int rank, int world, krg_exchange_fn fn, void* user);
  // in-graph exchange over an NCCL communicator (unique_id: KRG_NCCL_ID_BYTES)
  void set_comm(int rank, int world, const void* unique_id);

  // scenario voltages (V-hat) [L][3n][2]
  void scenario_voltages(double* out);
  const std::vector<double>& vhat() const;  // [L][3n][2] V-hat of the loaded library
  // batched anchored solve on the full Y
  void solve(const double* inj, int nrhs, double* out);

  // full run_reduction
  using Observer = std::function<void(const HostState&, const TraceRow&)>;
  void run(const ReductionConfig& cfg, const Observer& obs, ResultData& out);
  // (re)load the scenario library: injections [L][3n][2]; voltages may be empty
  // (then V-hat = device anchored solve of the injections)
  void set_scenarios(const std::vector<std::string>& ids, const std::vector<double>& inj,
                     const std::vector<double>& volt);
  // new values for the same network structure (host -> device, refactorize)
  void reload(const Problem& p);
  // constant-PQ conversion (scenario_from_pq, scenario.cpp:52-98), device solves
  void pq_to_currents(const std::vector<std::vector<std::pair<int, cx>>>& loads,
                      std::vector<double>& inj, std::vector<double>& volt);

  // loop parity hooks
  void loop_begin(const ReductionConfig& cfg);
  void debug_base_refresh(int reps, double* ms, long long* clocks);
  std::int64_t loop_candidates(std::vector<int>& cs, std::vector<int>& cr);
  void loop_score_all(double* smice, std::uint8_t* feasible, double* max_err);
  void loop_best(krg_best* out, double* max_err);
  void loop_commit(int s, int r);
  void loop_base(double* out);
  void zcols(double* out, std::int64_t cap);

  // Kron reduction of the full Y onto keep (kron.cpp:34-46)
  void kron(const std::vector<int>& reduce, ReducedModel& model);
  // per-scenario max error of a reduced model (reduce.cpp:490-550)
  std::vector<double> model_errors(const ReducedModel& model);
  void radialize(ReducedModel& model, bool with_errors);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// writers (io.cpp)
std::string reduced_json(const ReducedModel& m);
std::string trace_csv(const std::vector<TraceRow>& trace, const std::vector<std::string>& ids,
                      const std::vector<double>& final_max_err,
                      const std::vector<std::string>& comments);

ValidateReport validate_report(const std::vector<std::string>& ids, const std::vector<double>& max_err, int bins);
std::string validate_csv(const ValidateReport& rep);

// radialization host helpers
ReducedModel radialize_host(const ReducedModel& model, const Network& original,
                            const std::function<void(const std::vector<int>&, ReducedModel&)>& kron,
                            const std::function<std::vector<double>(const ReducedModel&)>* errors);

}  // namespace kronred::b200
