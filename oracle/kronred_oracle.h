/*
 * kronred_oracle.h — TEST INFRASTRUCTURE ONLY. A plain-C restatement of the
 * reference's exhaustive-search reduction hot path (Opti-KRON, kronred),
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the checker. The product (libkronred_b200.so) never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this oracle bit-for-bit against
 * the golden vectors produced by the UNMODIFIED reference build
 * (oracle/_ref, tests/golden/make_golden.py): V-hat and every unit-injection
 * solve, per-candidate delta scores, and full (s, r, smice, max_err)
 * trajectories.
 */
#ifndef KRONRED_ORACLE_H
#define KRONRED_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Network as in include/kronred_b200.h (krg_network). */
typedef struct oracle_net {
  int32_t n;
  const uint8_t* phases;
  int32_t slack;
  const double* slack_v;   /* [3][2] */
  int32_t nb;
  const int32_t* from;
  const int32_t* to;
  const double* y;         /* [nb][9][2] */
  const double* sh_from;   /* [nb][9][2] or NULL */
  const double* sh_to;     /* [nb][9][2] or NULL */
  const uint8_t* is_z;     /* [nb]: y holds a z_block to invert, or NULL */
} oracle_net;

/* Anchored solves (AnchoredSolver::solve, solver.cpp:181-186) of `nrhs`
 * right-hand sides [nrhs][3n][2] -> out [nrhs][3n][2]. Returns 0 or -node-1
 * on a singular pivot. */
int oracle_solve(const oracle_net* net, const double* inj, int32_t nrhs, double* out);

/* run_reduction (reduce.cpp:349-451) on constant-current scenarios
 * (injections [L][3n][2]; voltages = anchored solve, scenario.cpp:39-50).
 * Trace rows (up to `cap`): s, r, smice, max_err [cap][L], super-node count
 * after the commit, candidate count; out_final [L] = model_max_errors of the
 * final clusters (reduce.cpp:490-550). objective 0 = magnitude, 1 = complex.
 * The first `score_iters` iterations' per-candidate scores (iteration, s, r,
 * feasible, smice, max_err[L]) go to the sc_* arrays (up to score_cap rows).
 * Returns the number of committed iterations, or < 0 on error. */
int oracle_run(const oracle_net* net, int32_t L, const double* inj, double e_bar,
               int32_t objective, double target, int32_t has_target, int32_t cap, int32_t* out_s,
               int32_t* out_r, double* out_smice, double* out_maxerr, int32_t* out_nsup,
               int32_t* out_cands, double* out_final, int32_t score_iters, int32_t score_cap,
               int32_t* sc_iter, int32_t* sc_s, int32_t* sc_r, int32_t* sc_feas, double* sc_smice,
               double* sc_maxerr, int32_t* nscores);

/* kron_reduce (kron.cpp:34-46): eliminate `reduce` and return the kept count
 * nk (or < 0); kept_ids [n], blocks [nk][nk][9][2], present [nk][nk]. */
int oracle_kron(const oracle_net* net, int32_t nred, const int32_t* reduce, int32_t* kept_ids,
                double* blocks, uint8_t* present);

/* GCC complex division (libgcc __divdc3): in [N][4] = (a,b,c,d) -> out [N][2]. */
void oracle_cdiv(const double* in, int32_t N, double* out);

#ifdef __cplusplus
}
#endif
#endif
