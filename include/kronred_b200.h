/*
 * kronred_b200.h — C ABI of the B200-native exhaustive-search Kron reduction.
 *
 * Drop-in boundary for the reference's hot path. Every entry
 * point below names the reference interface it replaces (file:line under
 * /root/reference/proj). All arrays are caller-owned host memory (plain
 * pointers + sizes, no torch types); the context owns every device buffer,
 * stream and schedule. A context is single-caller (not thread-safe), like the
 * reference's run_reduction (reduce.cpp:349) which is called from one thread.
 *
 * Layout conventions (identical to the reference's in-memory structures):
 *   complex numbers are interleaved (re, im) doubles;
 *   a 3x3 block is 9 complex row-major  (Mat3c, complex3.hpp:38-60)  = 18 doubles;
 *   a node vector is 3 complex per node, scalar index 3*node+phase (block_matrix.hpp:12-14);
 *   phase masks are bit 0 = a, bit 1 = b, bit 2 = c                 (phase.hpp:13-16).
 *
 * Status codes mirror the reference's exception hierarchy (errors.hpp:10-37):
 * KRG_E_VALIDATION ~ ValidationError/StructuralError/ConfigError (CLI exit 2),
 * KRG_E_SOLVER ~ SolverError{smallest_pivot,node} (CLI exit 3).
 */
#ifndef KRONRED_B200_H
#define KRONRED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRG_OK 0
#define KRG_E_VALIDATION 2   /* ValidationError / StructuralError / ConfigError */
#define KRG_E_SOLVER 3       /* SolverError (singular present-phase pivot)      */
#define KRG_E_CUDA 4         /* CUDA runtime failure or no device               */
#define KRG_E_INTERNAL 5     /* other error (exchange callback, I/O, ...)       */

#define KRG_OBJ_MAGNITUDE 0  /* Objective::magnitude     (reduce.hpp:19) */
#define KRG_OBJ_COMPLEX 1    /* Objective::complex_error (reduce.hpp:19) */

/* Network (network.hpp:13-52). Node ids are dense 0..n-1. */
typedef struct krg_network {
  int32_t n_nodes;
  const uint8_t* phases;        /* [n] phase masks                              */
  int32_t slack;                /* id of the unique slack node                  */
  const double* slack_voltage;  /* [3][2]                                       */
  int32_t n_branches;
  const int32_t* br_from;       /* [nb]                                         */
  const int32_t* br_to;         /* [nb]                                         */
  const double* y_series;       /* [nb][9][2]                                   */
  const double* shunt_from;     /* [nb][9][2] or NULL (zero)                    */
  const double* shunt_to;       /* [nb][9][2] or NULL (zero)                    */
} krg_network;

/* ScenarioLibrary (scenario.hpp:15-33). voltages may be NULL: they are then
 * produced by the device anchored solve (scenario_from_currents,
 * scenario.cpp:39-50). */
typedef struct krg_scenarios {
  int32_t n_scenarios;
  const double* injections;     /* [L][3n][2] */
  const double* voltages;       /* [L][3n][2] or NULL */
} krg_scenarios;

/* ReductionConfig (reduce.hpp:21-28). `workers` has no device meaning and is
 * ignored; use_delta=0 selects the naive per-candidate anchored-solve scorer
 * (reduce.cpp:132-192) on the device. */
typedef struct krg_config {
  double e_bar;
  int32_t objective;            /* KRG_OBJ_* */
  int32_t has_target;
  double target_reduction;
  int32_t use_delta;
  int32_t workers;
} krg_config;

/* Best candidate of one scoring pass (the argmin of reduce.cpp:397-404). */
typedef struct krg_best {
  double smice;                 /* +inf when no feasible candidate            */
  int64_t index;                /* global candidate index, -1 when none       */
  int32_t s, r;
} krg_best;

typedef struct krg_ctx krg_ctx;
typedef struct krg_result krg_result;
typedef struct krg_host_problem krg_host_problem;

/* Multi-GPU exchange hook: all-gather `bytes` from every rank into `recv`
 * (world*bytes, rank order). Called once per iteration on every rank with a
 * fixed-size min-loc record (smice, global index, max_err[L]); the bench wires
 * it to torch.distributed (NCCL over NVLink). Return 0 on success. */
typedef int (*krg_exchange_fn)(void* user, const void* send, void* recv, size_t bytes);

/* Per-iteration observer (IterationObserver, reduce.hpp:160-161). */
typedef void (*krg_observer_fn)(void* user, int32_t iteration, int32_t s, int32_t r,
                                double smice, const double* max_err, int32_t supernode_count,
                                int32_t candidate_count, double wall_ms);

/* ---- error reporting -------------------------------------------------- */
const char* krg_last_error(void);                 /* thread-local message */
double krg_last_error_pivot(void);                /* SolverError::smallest_pivot */
int32_t krg_last_error_node(void);                /* SolverError::node */
const char* krg_version(void);

/* ---- host-side input path (no device needed) -------------------------- */
/* read_network_json (io.cpp:170) + load_library's CSV parse (scenario.cpp:141-212).
 * The CSV header selects constant-PQ or constant-current mode. */
int krg_host_load(const char* network_json_path, const char* scenario_csv_path,
                  krg_host_problem** out);
int krg_host_view(const krg_host_problem* p, krg_network* net, int32_t* n_scenarios,
                  int32_t* pq_mode, const double** injections_or_pq);
const char* krg_host_scenario_id(const krg_host_problem* p, int32_t l);
void krg_host_free(krg_host_problem* p);

/* validate (network.cpp:46-188): KRG_OK or KRG_E_VALIDATION with the report. */
int krg_validate(const krg_network* net);

/* Host-only parity hooks on the assignment state machine (reduce.cpp:39-73,
 * 299-344): simulate an (s,r) trajectory and enumerate the candidates of the
 * state it reaches. Returns the candidate count (<= cap written). */
int64_t krg_enumerate_after(const krg_network* net, const int32_t* traj_s,
                            const int32_t* traj_r, int32_t n_commits, int32_t* cand_s,
                            int32_t* cand_r, int64_t cap);

/* Candidate sharding and min-loc merge used by the multi-GPU loop
 * (parallel.cpp:11-34 split, reduce.cpp:397-404 tie-break). Host-only. */
void krg_shard_range(int64_t count, int32_t rank, int32_t world, int64_t* begin,
                     int64_t* end);
int32_t krg_merge_best(const double* smice, const int64_t* index, int32_t world);

/* ---- device context ---------------------------------------------------- */
/* Validates, assembles Y (grid_model.cpp:17-74), builds the elimination
 * schedule and factorizes on `device` (AnchoredSolver, solver.cpp:168-179). */
int krg_create(const krg_network* net, const krg_scenarios* scen, int32_t device,
               krg_ctx** out);
/* Same, from a parsed host problem (krg_host_load); constant-PQ libraries run
 * the I = -conj(S/V) fixed point with device solves (scenario.cpp:52-98). */
int krg_create_from_host(const krg_host_problem* p, int32_t device, krg_ctx** out);
void krg_destroy(krg_ctx* ctx);
/* Re-load a problem with the same network structure (node phases, branch
 * endpoints) into an existing context: admittances and scenarios are copied
 * host -> device and refactorized (AnchoredSolver ctor, solver.cpp:168-179;
 * load_library, scenario.cpp:141-220) without re-planning the elimination or
 * re-allocating. KRG_E_VALIDATION when the structure differs. */
int krg_reload_from_host(krg_ctx* ctx, const krg_host_problem* p);
/* Test hook: branch-free scorer sqrt vs IEEE __dsqrt_rn on n device-generated
 * inputs uniform in [lo, hi); returns the number of bit mismatches. */
int krg_selftest_sqrt(int64_t n, double lo, double hi, int64_t* mismatches);
/* Test hook: libgcc __divdc3 replica, in [N][4] = (a,b,c,d) -> out [N][2]. */
int krg_selftest_cdiv(const double* in, int32_t N, double* out, int32_t on_device);
int krg_set_exchange(krg_ctx* ctx, int32_t rank, int32_t world, krg_exchange_fn fn,
                     void* user);
/* Multi-GPU inside the device loop (the reference's worker split,
 * parallel.cpp:11-34, across GPUs): one context per rank and GPU, all built
 * from the same problem. Rank 0 makes an id with krg_nccl_unique_id and hands
 * it to every rank (any side channel); every rank then calls krg_set_comm
 * (collective: an NCCL communicator, a symmetric window of per-rank records,
 * a device communicator with one LSA barrier). Each iteration every rank
 * scores its contiguous range of the candidate list and the pick kernel
 * exchanges one {smice, index, max_err[L]} record per rank through the window
 * (NVLink peer stores + LSA barrier) inside the loop graph; all ranks commit
 * the same candidate. */
#define KRG_NCCL_ID_BYTES 128
int krg_nccl_unique_id(uint8_t* out /* KRG_NCCL_ID_BYTES */);
int krg_set_comm(krg_ctx* ctx, int32_t rank, int32_t world, const uint8_t* unique_id);
/* Number of kernels this context has launched so far. */
int64_t krg_launch_count(const krg_ctx* ctx);
/* 1 if the last krg_run_reduction ran as the device-resident loop graph (0:
 * the host-driven loop: use_delta = false, KRONRED_LOOP=host, profiling). */
int32_t krg_last_run_device_loop(const krg_ctx* ctx);
/* Per-kernel CUDA-event timing on the launching stream (bench/roofline only):
 * which = 0 scorer (score1_kernel: |phi(r)| = 1 candidates, the dominant
 * kernel), 1 base-refresh solve, 2 score3_kernel (|phi(r)| >= 2 candidates
 * next to score1). Sums over launches of the
 * event time and of the algorithmic flops/bytes. */
int krg_set_profile(krg_ctx* ctx, int32_t on);
int krg_kernel_stats(const krg_ctx* ctx, int32_t which, int64_t* launches, double* ms,
                     double* flops, double* bytes);
/* Measured unfused FP64 op rate of the device (GFLOP/s), the roofline peak. */
int krg_fp64_probe(int32_t device, double* gflops);
/* Device-side V-hat (scenario voltages) as used by the scorer, [L][3n][2]. */
int krg_scenario_voltages(krg_ctx* ctx, double* out);

/* run_reduction (reduce.cpp:349-451). */
int krg_run_reduction(krg_ctx* ctx, const krg_config* cfg, krg_observer_fn obs,
                      void* obs_user, krg_result** out);

/* AnchoredSolver::solve (solver.cpp:181-186), batched: inj/out [nrhs][3n][2]. */
int krg_solve(krg_ctx* ctx, const double* inj, int32_t nrhs, double* out);

/* Parity hooks on the loop: begin a loop state, score every
 * enumerated candidate of the current iteration, commit one. */
int krg_loop_begin(krg_ctx* ctx, const krg_config* cfg);
int64_t krg_loop_candidates(krg_ctx* ctx, int32_t* cand_s, int32_t* cand_r, int64_t cap);
int krg_loop_score_all(krg_ctx* ctx, double* smice, uint8_t* feasible, double* max_err);
int krg_loop_best(krg_ctx* ctx, krg_best* out, double* max_err);
int krg_loop_commit(krg_ctx* ctx, int32_t s, int32_t r);
/* Present-row Z block (solve(e_k) - v0, reduce.cpp:272-290): [n_phi][n_phi][2]
 * column-major (column = unit injection), rows/cols = present node-phases. */
int krg_zcols(krg_ctx* ctx, double* out, int64_t cap);
/* Per-iteration base voltages (refresh_base, reduce.cpp:265-268): [L][3n][2]. */
int krg_loop_base(krg_ctx* ctx, double* out);
/* Benchmark hook: mean time of `reps` base refreshes and block-0 phase clocks. */
int krg_debug_base_refresh(krg_ctx* ctx, int32_t reps, double* ms, long long* clocks);

/* kron_reduce (kron.cpp:34-46) of the context's Y onto keep = complement of
 * `reduce`; result read back with krg_result_* accessors (model part only). */
int krg_kron_reduce(krg_ctx* ctx, const int32_t* reduce, int32_t m, krg_result** out);

/* radialize (radialize.cpp:121-171) of a result's model, re-Kron on device. */
int krg_radialize(krg_ctx* ctx, krg_result* res, int32_t with_errors);

/* ---- result accessors (ReductionResult / ReducedModel, reduce.hpp:130-158) */
int32_t krg_result_iterations(const krg_result* res);
int krg_result_trace(const krg_result* res, int32_t* s, int32_t* r, double* smice,
                     double* max_err /*[it][L]*/, int32_t* supernode_count,
                     int32_t* candidate_count, double* wall_ms);
int32_t krg_result_n_kept(const krg_result* res);
int32_t krg_result_n_scenarios(const krg_result* res);
int krg_result_kept(const krg_result* res, int32_t* ids, uint8_t* phases);
int64_t krg_result_n_blocks(const krg_result* res);
int krg_result_blocks(const krg_result* res, int32_t* bi, int32_t* bj, double* vals /*[nb][18]*/);
int krg_result_final_max_err(const krg_result* res, double* out);
/* clusters: super-node ids (ascending) with CSR member lists (sorted). */
int32_t krg_result_n_clusters(const krg_result* res);
int krg_result_clusters(const krg_result* res, int32_t* sup, int32_t* off, int32_t* members);
int32_t krg_result_n_reinserted(const krg_result* res);
int krg_result_reinserted(const krg_result* res, int32_t* ids);
int64_t krg_result_total_candidates(const krg_result* res);
/* CUDA-event time (ms) of the whole run on the context's stream. */
double krg_result_device_ms(const krg_result* res);
/* Byte-compatible writers (io.cpp:216-265 and io.cpp:338-359). */
int krg_result_write_reduced_json(const krg_result* res, const char* path);
int krg_result_write_trace_csv(const krg_result* res, const char* path, int32_t zero_wall);
/* Validation report of a reduced model against the context's network and
 * scenario library: per-scenario max errors (model_max_errors on the device)
 * and a `bins`-bin histogram, as the CSV the reference writes
 * (make_validate_report + write_validate_report, io.cpp:385-416). Writes up
 * to cap-1 bytes plus NUL into out (may be null); returns the full length, or
 * minus a KRG_E_* status. */
int64_t krg_validate_report(krg_ctx* ctx, const krg_result* res, int32_t bins, char* out, int64_t cap);
void krg_result_free(krg_result* res);

#ifdef __cplusplus
}
#endif
#endif /* KRONRED_B200_H */
