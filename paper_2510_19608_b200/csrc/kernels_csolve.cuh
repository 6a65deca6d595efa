// K1s (compact): anchored forward/backward sweeps on the present-phase
// compacted factor, one right-hand side per CTA. The right-hand side, the
// solution, the factor and its level program all live in shared memory (when
// they fit; the factor and program fall back to global/L1 otherwise), so a
// level costs a few shared-memory round trips plus one __syncthreads.
//
// Level program: per step a packed record (solution offset, present-phase
// count and mask, pinv offset, pull / coupling list) in level order, and per
// pull or coupling a packed (offset, phase count, block offset) pair.
//
// Compaction is exact: a block's entries outside the present-phase rows/cols
// are exact zeros, their products with finite operands are signed zeros, and
// adding a signed zero to an accumulator that starts at +0 never changes its
// bits; absent-phase entries of every solution are +0 (SURVEY §7.9 verified
// the pull order; this file keeps that order and the ascending-phase order of
// every Mat3c*Vec3c accumulation, complex3.hpp:85-90).
#pragma once

namespace kronred::b200 {
namespace {

enum CMode { CM_FULL = 0, CM_BASE = 1, CM_ZCOL = 2 };

// Device-resident loop state (kernels_loop.cuh): the iteration's sizes and
// scorer grid layout, written by the enumeration kernel, read by the scorer,
// the pick/commit kernel and the base refresh (which all exit when done).
// loop timeline stamps per iteration (KRONRED_LOOP_TRACE): 0/1 pick start/end,
// 2/3 enum start/end, 4/5 refresh start/end (CTA 0), 6 score start, 7 enum
// table done, 8 refresh staged (CTA 0), 9 refresh walk done (CTA 0), 10 last
// refresh CTA end
constexpr int kTdbg = 16;
// base values and cluster bounds of present row r, scenario l: one row holds
// the L base values, then the L bounds ({min, max} of the member magnitudes),
// so a scenario slice of either is one contiguous run
__host__ __device__ __forceinline__ size_t bv_base(size_t r, int L, int l) { return r * 2 * size_t(L) + size_t(l); }
__host__ __device__ __forceinline__ size_t bv_bnd(size_t r, int L, int l) { return r * 2 * size_t(L) + size_t(L + l); }
// Programmatic dependent launch: wait for the preceding kernel's results (a
// no-op when launched without the attribute)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct LoopState {
  int done, iter, ns, C, R, err;
  int S;             // scorer lanes per (candidate, scenario) pair this iteration
  int c0, Cl;        // this rank's candidate range [c0, c0 + Cl) of the C (lexicographic); c0 = 0, Cl = C on one GPU
  int last_s, last_r;  // the last committed candidate (incremental base refresh)
  int grp_start[4];  // candidate offset of each |phi(r)| group (index 1..3)
  int grp_cta[4];    // first CTA of each group; grp_cta[3] = CTAs in use
};

// offsets (in ints) of the packed program sections
struct CProg {
  int frec, fent, brec, bent, fw_off, bw_off, kept;  // kept: (x | m << 24, kept index)
  int nsteps, nfw, nbw, nkept, nmeta, ncf, nphi;
};

struct CSolveArgs {
  CProg P;
  const int* meta_g;
  const double2* cfac_g;
  const double2* kept_val;  // [nkept][3] (present phases in order)
  int smem_factor;          // stage cfac + program in shared memory
  int n;                    // nodes of this matrix
  const int* prow_off;      // [n+1]
  const std::uint8_t* mask; // [n]
  const int* prow_node;     // [nphi]
  const std::uint8_t* prow_phase;
  const double2* rhs_full;  // MODE_FULL: [nrhs][3n] or null
  double2* out_full;        // MODE_FULL: [nrhs][3n]
  const double2* iagg;      // MODE_BASE: [n][L][3]
  double2* base;            // MODE_BASE: bv [nphi][L][2], base in slot 0
  int L;
  int col0;                 // MODE_ZCOL
  const double2* v0p;
  double2* zout;            // [ncol][nphi]
  long long* dbg;           // optional phase timestamps (block 0, warp 0)
};

__device__ __forceinline__ int popc_below(unsigned m, int p) { return __popc(m & ((1u << p) - 1u)); }

template <int MODE>
__global__ void __launch_bounds__(256) csolve_kernel(CSolveArgs a) {
  extern __shared__ double2 smem[];
  const CProg& P = a.P;
  double2* x = smem;  // [nphi]: right-hand side, then t, then the solution
  const double2* cf = a.cfac_g;
  const int* M = a.meta_g;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int rhs = blockIdx.x;
  if (a.smem_factor) {
    double2* scf = smem + P.nphi;
    int* smeta = reinterpret_cast<int*>(scf + P.ncf);
    for (int i = tid; i < P.ncf; i += nt) scf[i] = a.cfac_g[i];
    const int4* g4 = reinterpret_cast<const int4*>(a.meta_g);
    int4* s4 = reinterpret_cast<int4*>(smeta);
    for (int i = tid; i < (P.nmeta + 3) / 4; i += nt) s4[i] = g4[i];
    cf = scf;
    M = smeta;
  }
  // right-hand side at present rows
  for (int r = tid; r < P.nphi; r += nt) {
    double2 b;
    if (MODE == CM_BASE) {
      b = a.iagg[(size_t(a.prow_node[r]) * a.L + rhs) * 3 + a.prow_phase[r]];
    } else if (MODE == CM_ZCOL) {
      b = (r == a.col0 + rhs) ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0);
    } else {
      b = a.rhs_full ? a.rhs_full[size_t(rhs) * 3 * a.n + size_t(a.prow_node[r]) * 3 + a.prow_phase[r]]
                     : make_double2(0.0, 0.0);
    }
    x[r] = b;
  }
  __syncthreads();
  // boundary (kept) values
  for (int k = tid; k < P.nkept; k += nt) {
    const int xe = M[P.kept + 2 * k], ki = M[P.kept + 2 * k + 1];
    const int x0 = xe & 0xffffff, m = xe >> 24;
    for (int i = 0; i < m; ++i) x[x0 + i] = a.kept_val[ki * 3 + i];
  }
  const int4* frec = reinterpret_cast<const int4*>(M + P.frec);
  const int2* fent = reinterpret_cast<const int2*>(M + P.fent);
  const int4* brec = reinterpret_cast<const int4*>(M + P.brec);
  const int2* bent = reinterpret_cast<const int2*>(M + P.bent);
  // forward: rhs_k = b_k - sum_j A_kj t_j in elimination order; t_k = pinv_k rhs_k
  for (int lev = 0; lev < P.nfw; ++lev) {
    const int o0 = M[P.fw_off + lev], o1 = M[P.fw_off + lev + 1];
    for (int idx = o0 + tid; idx < o1; idx += nt) {
      const int4 rc = frec[idx];
      const int xk = rc.x & 0xffffff, mk = (rc.x >> 24) & 3;
      const int po = rc.z, e0 = rc.w & 0xffffff, ne = (rc.w >> 24) & 0xff;
      C2 b[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) b[i] = i < mk ? ld2(x + xk + i) : C2{0.0, 0.0};
      for (int e = e0; e < e0 + ne; ++e) {
        const int2 en = fent[e];
        const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
        C2 tj[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) tj[c] = c < mj ? ld2(x + xj + c) : C2{0.0, 0.0};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r >= mk) continue;
          C2 acc = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < mj) acc = dev::cadd(acc, dev::cmul(ld2(cf + bo + r * mj + c), tj[c]));
          b[r] = dev::csub(b[r], acc);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= mk) continue;
        C2 acc = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < mk) acc = dev::cadd(acc, dev::cmul(ld2(cf + po + r * mk + c), b[c]));
        st2(x + xk + r, acc);
      }
    }
    __syncthreads();
  }
  // backward: x_k = t_k - pinv_k (sum_c A_kc x_c), couplings ascending
  for (int lev = 0; lev < P.nbw; ++lev) {
    const int o0 = M[P.bw_off + lev], o1 = M[P.bw_off + lev + 1];
    for (int idx = o0 + tid; idx < o1; idx += nt) {
      const int4 rc = brec[idx];
      const int xk = rc.x & 0xffffff, mk = (rc.x >> 24) & 3;
      const int po = rc.z, e0 = rc.w & 0xffffff, ne = (rc.w >> 24) & 0xff;
      C2 acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int e = e0; e < e0 + ne; ++e) {
        const int2 en = bent[e];
        const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
        C2 xv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) xv[c] = c < mj ? ld2(x + xj + c) : C2{0.0, 0.0};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r >= mk) continue;
          C2 u = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < mj) u = dev::cadd(u, dev::cmul(ld2(cf + bo + r * mj + c), xv[c]));
          acc[r] = dev::cadd(acc[r], u);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= mk) continue;
        C2 corr = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < mk) corr = dev::cadd(corr, dev::cmul(ld2(cf + po + r * mk + c), acc[c]));
        st2(x + xk + r, dev::csub(ld2(x + xk + r), corr));
      }
    }
    __syncthreads();
  }
  // outputs
  if (MODE == CM_BASE) {
    for (int r = tid; r < P.nphi; r += nt) a.base[bv_base(size_t(r), a.L, rhs)] = x[r];
  } else if (MODE == CM_ZCOL) {
    double2* zc = a.zout + size_t(a.col0 + rhs) * P.nphi;
    for (int r = tid; r < P.nphi; r += nt) st2(zc + r, dev::csub(ld2(x + r), ld2(a.v0p + r)));
  } else {
    double2* o = a.out_full + size_t(rhs) * 3 * a.n;
    for (int t = tid; t < 3 * a.n; t += nt) {
      const int node = t / 3, p = t % 3;
      const unsigned m = a.mask[node];
      o[t] = ((m >> p) & 1u) ? x[a.prow_off[node] + popc_below(m, p)] : make_double2(0.0, 0.0);
    }
  }
}

// Warp-per-right-hand-side variant: the CTA stages the factor and program
// into shared memory once; each warp then solves its own right-hand side with
// __syncwarp between levels (no CTA barriers on the level-serial path).
// W warps per CTA, solution vectors x[W][nphi] after the staged factor.
template <int MODE, bool SMEMF>
__global__ void __launch_bounds__(256) csolve_warp_kernel(CSolveArgs a, int nrhs) {
  extern __shared__ double2 smem[];
  const CProg& P = a.P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int W = nt >> 5;
  const int rhs = blockIdx.x * W + warp;
  const double2* cf;
  const int* M;
  double2* xall;
  if (SMEMF) {
    double2* scf = smem;
    int* smeta = reinterpret_cast<int*>(scf + P.ncf);
    for (int i = tid; i < P.ncf; i += nt) scf[i] = a.cfac_g[i];
    const int4* g4 = reinterpret_cast<const int4*>(a.meta_g);
    int4* s4 = reinterpret_cast<int4*>(smeta);
    for (int i = tid; i < (P.nmeta + 3) / 4; i += nt) s4[i] = g4[i];
    cf = scf;
    M = smeta;
    xall = reinterpret_cast<double2*>(smeta + P.nmeta);
    __syncthreads();
  } else {
    cf = a.cfac_g;
    M = a.meta_g;
    xall = smem;
  }
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[0] = clock64();
  if (rhs >= nrhs) return;
  double2* x = xall + size_t(warp) * P.nphi;
  for (int r = lane; r < P.nphi; r += 32) {
    double2 b;
    if (MODE == CM_BASE) {
      b = a.iagg[(size_t(a.prow_node[r]) * a.L + rhs) * 3 + a.prow_phase[r]];
    } else if (MODE == CM_ZCOL) {
      b = (r == a.col0 + rhs) ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0);
    } else {
      b = a.rhs_full ? a.rhs_full[size_t(rhs) * 3 * a.n + size_t(a.prow_node[r]) * 3 + a.prow_phase[r]]
                     : make_double2(0.0, 0.0);
    }
    x[r] = b;
  }
  __syncwarp();
  for (int k = lane; k < P.nkept; k += 32) {
    const int xe = M[P.kept + 2 * k], ki = M[P.kept + 2 * k + 1];
    const int x0 = xe & 0xffffff, m = xe >> 24;
    for (int i = 0; i < m; ++i) x[x0 + i] = a.kept_val[ki * 3 + i];
  }
  __syncwarp();
  const int4* frec = reinterpret_cast<const int4*>(M + P.frec);
  const int2* fent = reinterpret_cast<const int2*>(M + P.fent);
  const int4* brec = reinterpret_cast<const int4*>(M + P.brec);
  const int2* bent = reinterpret_cast<const int2*>(M + P.bent);
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[1] = clock64();
  for (int lev = 0; lev < P.nfw; ++lev) {
    const int o0 = M[P.fw_off + lev], o1 = M[P.fw_off + lev + 1];
    for (int idx = o0 + lane; idx < o1; idx += 32) {
      const int4 rc = frec[idx];
      const int xk = rc.x & 0xffffff, mk = (rc.x >> 24) & 3;
      const int po = rc.z, e0 = rc.w & 0xffffff, ne = (rc.w >> 24) & 0xff;
      if (rc.x & (1 << 29)) {
        // single-phase step with single-phase pulls: 1x1 complex blocks
        C2 b = ld2(x + xk);
        for (int e = e0; e < e0 + ne; ++e) {
          const int2 en = fent[e];
          const C2 acc = dev::cadd(C2{0.0, 0.0}, dev::cmul(ld2(cf + en.y), ld2(x + (en.x & 0xffffff))));
          b = dev::csub(b, acc);
        }
        st2(x + xk, dev::cadd(C2{0.0, 0.0}, dev::cmul(ld2(cf + po), b)));
        continue;
      }
      C2 b[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) b[i] = i < mk ? ld2(x + xk + i) : C2{0.0, 0.0};
      for (int e = e0; e < e0 + ne; ++e) {
        const int2 en = fent[e];
        const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
        C2 tj[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) tj[c] = c < mj ? ld2(x + xj + c) : C2{0.0, 0.0};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r >= mk) continue;
          C2 acc = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < mj) acc = dev::cadd(acc, dev::cmul(ld2(cf + bo + r * mj + c), tj[c]));
          b[r] = dev::csub(b[r], acc);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= mk) continue;
        C2 acc = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < mk) acc = dev::cadd(acc, dev::cmul(ld2(cf + po + r * mk + c), b[c]));
        st2(x + xk + r, acc);
      }
    }
    __syncwarp();
  }
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[2] = clock64();
  for (int lev = 0; lev < P.nbw; ++lev) {
    const int o0 = M[P.bw_off + lev], o1 = M[P.bw_off + lev + 1];
    for (int idx = o0 + lane; idx < o1; idx += 32) {
      const int4 rc = brec[idx];
      const int xk = rc.x & 0xffffff, mk = (rc.x >> 24) & 3;
      const int po = rc.z, e0 = rc.w & 0xffffff, ne = (rc.w >> 24) & 0xff;
      if (rc.x & (1 << 29)) {
        C2 acc = {0.0, 0.0};
        for (int e = e0; e < e0 + ne; ++e) {
          const int2 en = bent[e];
          acc = dev::cadd(acc, dev::cadd(C2{0.0, 0.0}, dev::cmul(ld2(cf + en.y), ld2(x + (en.x & 0xffffff)))));
        }
        const C2 corr = dev::cadd(C2{0.0, 0.0}, dev::cmul(ld2(cf + po), acc));
        st2(x + xk, dev::csub(ld2(x + xk), corr));
        continue;
      }
      C2 acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int e = e0; e < e0 + ne; ++e) {
        const int2 en = bent[e];
        const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
        C2 xv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) xv[c] = c < mj ? ld2(x + xj + c) : C2{0.0, 0.0};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r >= mk) continue;
          C2 u = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < mj) u = dev::cadd(u, dev::cmul(ld2(cf + bo + r * mj + c), xv[c]));
          acc[r] = dev::cadd(acc[r], u);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= mk) continue;
        C2 corr = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < mk) corr = dev::cadd(corr, dev::cmul(ld2(cf + po + r * mk + c), acc[c]));
        st2(x + xk + r, dev::csub(ld2(x + xk + r), corr));
      }
    }
    __syncwarp();
  }
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[3] = clock64();
  if (MODE == CM_BASE) {
    for (int r = lane; r < P.nphi; r += 32) a.base[bv_base(size_t(r), a.L, rhs)] = x[r];
  } else if (MODE == CM_ZCOL) {
    double2* zc = a.zout + size_t(a.col0 + rhs) * P.nphi;
    for (int r = lane; r < P.nphi; r += 32) st2(zc + r, dev::csub(ld2(x + r), ld2(a.v0p + r)));
  } else {
    double2* o = a.out_full + size_t(rhs) * 3 * a.n;
    for (int t = lane; t < 3 * a.n; t += 32) {
      const int node = t / 3, p = t % 3;
      const unsigned m = a.mask[node];
      o[t] = ((m >> p) & 1u) ? x[a.prow_off[node] + popc_below(m, p)] : make_double2(0.0, 0.0);
    }
  }
}

// ---------------------------------------------------------------------------
// Base refresh (reduce.cpp:265-268), one warp per scenario. The factor, the
// level program and each warp's right-hand side arrive in shared memory by
// TMA bulk copies (cp.async.bulk + mbarrier transaction count). The program
// is laid out in "lane slots": for every level round a record per lane, so a
// round needs no level bounds and the next round's record is loaded while the
// current one computes; single-phase steps with one pull/coupling carry it
// inline. Per round the critical path is: x load -> complex chain -> store.
//
// record int4: x = x_k | m_k<<24 | SCALAR<<29 | INLINE<<30 | EMPTY<<31,
//              y = pinv offset, z = inline ? x_j : first entry, w = inline ? block : count
constexpr int kRefreshWB = 8;  // warps per scenario in the global-program backward sweep

struct BaseArgs {
  int nphi, ncf, nmeta, L, W;
  int WB;                 // warps per scenario (backward sweep rounds of 32 * WB slots); 1: one warp per scenario
  int bfast;              // first backward round from which every round is scalar single-coupling only
  int fslot, fext, nfr, bslot, bext, nbr, fent, bent, kept, nkept;  // program offsets (ints)
  const double2* cfac;
  const int* meta;
  const double2* iaggp;   // [L][nphi]
  const double2* kept_val;
  double2* bv;            // [nphi][L][2], base in slot 0
  long long* dbg;
  const LoopState* st;    // device-resident loop: skip once the loop is done
  unsigned long long* tdbg;  // optional loop timeline [iter][8] (slots 4, 5)
  // incremental forward sweep: only the elimination-tree ancestors of the two
  // rows a commit changed are re-eliminated; the other nodes' forward values
  // are bit-identical to the previous refresh and come from tfwd
  double2* tfwd;          // [L][nphi] forward values of the last refresh (null: disabled)
  int inc;                // 1: incremental (s, r below or st->last_s/last_r), 0: full sweep
  int inc_s, inc_r;       // changed nodes (host-driven loop)
  int walk;               // ints offset in M of [node] int4 {record, parent, step, 0} (-1 record: kept)
  int rhs_staged;         // incremental: right-hand sides staged in a second buffer per warp
};

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(bar))), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(unsigned(__cvta_generic_to_shared(bar))),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(unsigned(__cvta_generic_to_shared(bar))),
      "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   unsigned(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes), "r"(unsigned(__cvta_generic_to_shared(bar)))
               : "memory");
}

__device__ __forceinline__ C2 lds2(unsigned addr) {
  double x, y;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
  return {x, y};
}
__device__ __forceinline__ void sts2(unsigned addr, C2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

#ifndef REFRESH_L2_KEEP
#define REFRESH_L2_KEEP 1
#endif
// The global-program refresh (large feeders) keeps its factor and program in
// L2 with an evict-last policy: between two refreshes the scorer streams Z
// (1.3 GB at 8,381 nodes) through L2.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Program record (int4) at a byte offset: shared memory (32-bit address)
// when the program is staged, global (read-only path) otherwise.
template <bool SM>
__device__ __forceinline__ int4 rec4(unsigned ms, const int4* g, int byteoff) {
  if constexpr (SM) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(ms + unsigned(byteoff)));
    return v;
  } else {
#if REFRESH_L2_KEEP
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(g + (byteoff >> 4)), "l"(l2_keep_policy()));
    return v;
#else
    return __ldg(g + (byteoff >> 4));
#endif
  }
}

// Factor coefficient at a byte offset: shared memory (32-bit address) when
// the program is staged, global (read-only path) otherwise.
template <bool SM>
__device__ __forceinline__ C2 cfl(unsigned cs, const double2* cf, int byteoff) {
  if constexpr (SM) {
    return lds2(cs + unsigned(byteoff));
  } else {
#if REFRESH_L2_KEEP
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(cf + (byteoff >> 4)), "l"(l2_keep_policy()));
#else
    const double2 v = __ldg(cf + (byteoff >> 4));
#endif
    return {v.x, v.y};
  }
}

// General (multi-phase) backward step, m_k, m_j <= 3. Every operand is loaded up
// front at a clamped (always in-block) index and the products are folded with
// selects, so the loads issue back to back instead of one predicated
// load -> product pair at a time; the folded operations and their order are
// those of the reference's Mat3c/Vec3c loops (only c < m_j / r < m_k terms).
template <bool SM>
__device__ __forceinline__ void gen_block_load(C2 (&A)[9], unsigned cs, const double2* cf, int blk, int mr, int mc) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) A[r * 3 + c] = cfl<SM>(cs, cf, (blk + min(r, mr - 1) * mc + min(c, mc - 1)) * 16);
}

// backward: x_k = t_k - pinv_k (sum_j U_kj x_j) (solver.cpp:136-147). x in
// shared memory (xs), the factor through cfl (shared or read-only global).
template <bool SM>
__device__ __forceinline__ void gen_bwd_step(const int4 rc, const int4 rx, unsigned xs, unsigned cs, double2* x,
                                             const double2* cf, const int2* be) {
  const int xk = rc.x >> 4, mk = rx.y, po = rc.y >> 4;
  C2 acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  C2 P[9], xo[3];
  gen_block_load<SM>(P, cs, cf, po, mk, mk);  // independent of the couplings: in flight first
#pragma unroll
  for (int r = 0; r < 3; ++r) xo[r] = lds2(xs + unsigned(xk + min(r, mk - 1)) * 16u);
  for (int e = rx.z; e < rx.z + rx.w; ++e) {
    const int2 en = be[e];
    const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
    C2 xv[3], A[9];
#pragma unroll
    for (int c = 0; c < 3; ++c) xv[c] = lds2(xs + unsigned(xj + min(c, mj - 1)) * 16u);
    gen_block_load<SM>(A, cs, cf, bo, mk, mj);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      C2 u = {0.0, 0.0};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const C2 t = dev::cadd(u, dev::cmul(A[r * 3 + c], xv[c]));
        u = c < mj ? t : u;
      }
      const C2 t = dev::cadd(acc[r], u);
      acc[r] = r < mk ? t : acc[r];
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    C2 corr = {0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const C2 t = dev::cadd(corr, dev::cmul(P[r * 3 + c], acc[c]));
      corr = c < mk ? t : corr;
    }
    if (r < mk) sts2(xs + unsigned(xk + r) * 16u, dev::csub(xo[r], corr));
  }
  (void)x;
}

// One row r of a backward general step split over its m_k lanes: the row's
// coupling sum acc_r (the loop of gen_bwd_step for that row alone), then,
// after the lanes exchanged their sums, the row's pivot product.
template <bool SM>
__device__ __forceinline__ C2 gen_bwd_acc_row(const int4 rx, unsigned xs, unsigned cs, const double2* cf,
                                              const int2* be, int r) {
  const int mk = rx.y;
  C2 acc = {0.0, 0.0};
  for (int e = rx.z; e < rx.z + rx.w; ++e) {
    const int2 en = be[e];
    const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
    C2 xv[3], Ar[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xv[c] = lds2(xs + unsigned(xj + min(c, mj - 1)) * 16u);
      Ar[c] = cfl<SM>(cs, cf, (bo + min(r, mk - 1) * mj + min(c, mj - 1)) * 16);
    }
    C2 u = {0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const C2 t = dev::cadd(u, dev::cmul(Ar[c], xv[c]));
      u = c < mj ? t : u;
    }
    acc = dev::cadd(acc, u);
  }
  return acc;
}

// One forward elimination step of the lane-slot program (pull form): node k's
// right-hand side minus its children's contributions in elimination order,
// times pinv_k (solver.cpp:125-134; the scalar fast path and the general
// 3x3 path).
template <bool SM>
__device__ __forceinline__ void tree_fwd_step(const int4 rc, const int4 rx, unsigned xs, unsigned cs, double2* x,
                                              const double2* cf, const int2* fe) {
  if (rc.x >= 0 && rc.z >= 0) {
      // scalar step: two pulls inline (zero pulls when absent), their
      // products in flight together; the subtractions keep elimination order
      const C2 b0 = lds2(xs + rc.x), tj = lds2(xs + rc.z), aa = cfl<SM>(cs, cf, rc.w), pv = cfl<SM>(cs, cf, rc.y);
      const C2 t1 = lds2(xs + rx.x), a1 = cfl<SM>(cs, cf, rx.y);
      const C2 u0 = dev::cadd(C2{0.0, 0.0}, dev::cmul(aa, tj));
      const C2 u1 = dev::cadd(C2{0.0, 0.0}, dev::cmul(a1, t1));
      C2 b = dev::csub(dev::csub(b0, u0), u1);
      int e = rx.z;
      const int e_end = rx.z + rx.w;
#pragma unroll 1
      for (; e < e_end; e += 3) {  // further children, predicated batches of three
        C2 u[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int2 en = fe[min(e + q, e_end - 1)];
          u[q] = dev::cadd(C2{0.0, 0.0}, dev::cmul(cfl<SM>(cs, cf, en.y * 16), lds2(xs + (en.x & 0xffffff) * 16)));
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (e + q < e_end) b = dev::csub(b, u[q]);
      }
      sts2(xs + rc.x, dev::cadd(C2{0.0, 0.0}, dev::cmul(pv, b)));
    } else if (rc.x >= 0) {
      const int xk = rc.x >> 4, mk = rx.y, po = rc.y >> 4;
      C2 b[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) b[i] = i < mk ? ld2(x + xk + i) : C2{0.0, 0.0};
      for (int e = rx.z; e < rx.z + rx.w; ++e) {
        const int2 en = fe[e];
        const int xj = en.x & 0xffffff, mj = en.x >> 24, bo = en.y;
        C2 tj[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) tj[c] = c < mj ? ld2(x + xj + c) : C2{0.0, 0.0};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r >= mk) continue;
          C2 acc = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (c < mj) acc = dev::cadd(acc, dev::cmul(ld2(cf + bo + r * mj + c), tj[c]));
          b[r] = dev::csub(b[r], acc);
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= mk) continue;
        C2 acc = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (c < mk) acc = dev::cadd(acc, dev::cmul(ld2(cf + po + r * mk + c), b[c]));
        st2(x + xk + r, acc);
      }
    }
}

// Full forward sweep of the lane-slot program, one level per round.
template <bool SM>
__device__ __forceinline__ void tree_forward(const BaseArgs& a, const int* M, unsigned xs, unsigned cs, double2* x,
                                             const double2* cf, int lane) {
  const int4* fs = reinterpret_cast<const int4*>(M + a.fslot);
  const int4* fx = reinterpret_cast<const int4*>(M + a.fext);
  const int2* fe = reinterpret_cast<const int2*>(M + a.fent);
  int4 rc = fs[lane];
  int4 rx = fx[lane];
  for (int fr = 0; fr < a.nfr; ++fr) {
    const int4 nx = fs[(fr + 1) * 32 + lane];
    const int4 nxx = fx[(fr + 1) * 32 + lane];
    tree_fwd_step<SM>(rc, rx, xs, cs, x, cf, fe);
    rc = nx;
    rx = nxx;
    __syncwarp();
  }
}

#ifndef BR_SUFFIX_UNROLL
#define BR_SUFFIX_UNROLL 4
#endif
constexpr int kBrSuffixUnroll = BR_SUFFIX_UNROLL;  // rounds per iteration of the all-scalar suffix loop

// Backward sweep of the lane-slot program (solver.cpp:136-147): every
// eliminated node resolved against its (already final) couplings, one level
// per round.
template <bool SM>
__device__ __forceinline__ void tree_backward(const BaseArgs& a, const int* M, unsigned xs, unsigned cs, double2* x,
                                              const double2* cf, int lane, int wb = 1, int wsub = 0) {
  const int4* bs = reinterpret_cast<const int4*>(M + a.bslot);
  const int4* bx = reinterpret_cast<const int4*>(M + a.bext);
  const int2* be = reinterpret_cast<const int2*>(M + a.bent);
  const int nbr = a.nbr;
  // Opaque copies: keeps the shared-window bases in registers instead of
  // re-deriving them (S2R) in front of the loads of every round.
  asm volatile("mov.b32 %0, %0;" : "+r"(xs));
  asm volatile("mov.b32 %0, %0;" : "+r"(cs));
  // Records are read two rounds ahead (the arrays carry one padding round, so
  // the index is clamped to it); a scalar step's coefficients and its own
  // forward value t_k one round ahead (the factor is read-only during the
  // sweep and x_k is written only by its own step).
  // records by byte offset from this lane's slot of round 0
  // a round is 32 * wb slots; this warp takes slots [32 wsub, 32 wsub + 32)
  // (multi-warp rounds only with the global program: a compile-time 1 otherwise)
  if constexpr (SM) {
    wb = 1;
    wsub = 0;
  }
  const int4* bsl = bs + wsub * 32 + lane;
  const int4* bxl = bx + wsub * 32 + lane;
  const int rstride = 512 * wb;  // bytes per round
  unsigned ssl = SM ? unsigned(__cvta_generic_to_shared(bsl)) : 0u, sxl = SM ? unsigned(__cvta_generic_to_shared(bxl)) : 0u;
  asm volatile("mov.b32 %0, %0;" : "+r"(ssl));
  asm volatile("mov.b32 %0, %0;" : "+r"(sxl));
  int4 rc = rec4<SM>(ssl, bsl, 0), rx = rec4<SM>(sxl, bxl, 0);
  int4 nx = rec4<SM>(ssl, bsl, min(1, nbr) * rstride), nxx = rec4<SM>(sxl, bxl, min(1, nbr) * rstride);
  const bool sc0 = rc.x >= 0 && rx.x == 0;
  C2 aa = sc0 ? cfl<SM>(cs, cf, rc.w) : C2{0.0, 0.0}, pv = sc0 ? cfl<SM>(cs, cf, rc.y) : C2{0.0, 0.0};
  C2 t = sc0 ? lds2(xs + rc.x) : C2{0.0, 0.0};
#ifdef BR_TRACE  // tuning aid: per-round cycles of CTA 0 / warp 0 (debug refresh only)
  long long tr_t[80], tr_b[80], tr_c[80];
  unsigned tr_a[80], tr_g[80];
  for (int i = 0; i < 80; ++i) tr_b[i] = tr_c[i] = 0;
  const bool tr_on = a.dbg && blockIdx.x == 0 && threadIdx.x < 32;
#endif
  const int bfast = min(a.bfast, nbr);
  int br = 0;
#pragma unroll 2
  for (; br < bfast; ++br) {
#ifdef BR_TRACE
    if (tr_on && br < 80) {
      tr_g[br] = __ballot_sync(0xffffffffu, rc.x >= 0 && rx.x != 0);
      tr_a[br] = __ballot_sync(0xffffffffu, rc.x >= 0);
      tr_t[br] = clock64();
    }
#endif
    // the parent's value first: it is the round's critical load (the shared
    // loads are ordered volatile asm, so it is issued ahead of the rest)
    const C2 xj = lds2(xs + (rc.x >= 0 ? rc.z : 0));
    // next round's scalar operands right behind it, so the shared-memory
    // pipe drains them while this round's products run (x_n is written only in
    // its own round, the factor not at all)
    const bool scn = nx.x >= 0 && nxx.x == 0;
    const C2 aa_n = cfl<SM>(cs, cf, scn ? nx.w : 0), pv_n = cfl<SM>(cs, cf, scn ? nx.y : 0);
    const C2 t_n = lds2(xs + (scn ? nx.x : 0));
    const int4 nx2 = rec4<SM>(ssl, bsl, min(br + 2, nbr) * rstride),
               nxx2 = rec4<SM>(sxl, bxl, min(br + 2, nbr) * rstride);
    const bool sc = rc.x >= 0 && rx.x == 0;
    if (__all_sync(0xffffffffu, rc.x < 0 || (rx.x == 0 && rx.w == 0))) {
      // every step of the round is scalar with the single coupling to its
      // parent: x_k = t_k - (0 + pinv (0 + (0 + A x_p))) (Mat3c * Vec3c from
      // zero, coupling sum from zero; adding +0 twice equals adding it once)
      if (rc.x >= 0) {
#ifdef BR_TRACE
        if (tr_on && br < 80 && xj.x != 1.2345e300) tr_b[br] = clock64();
#endif
        const C2 acc = dev::cadd(C2{0.0, 0.0}, dev::cmul(aa, xj));
        const C2 res = dev::csub(t, dev::cadd(C2{0.0, 0.0}, dev::cmul(pv, acc)));
#ifdef BR_TRACE
        if (tr_on && br < 80 && res.x != 1.2345e300) tr_c[br] = clock64();
#endif
        sts2(xs + rc.x, res);
      }
    } else if (sc) {
      C2 acc = dev::cadd(C2{0.0, 0.0}, dev::cmul(aa, xj));
      int e = rx.z;
      const int e_end = rx.z + rx.w;
#pragma unroll 1
      for (; e < e_end; e += 3) {  // predicated batches of three
        C2 u[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int2 en = be[min(e + q, e_end - 1)];
          u[q] = dev::cadd(C2{0.0, 0.0}, dev::cmul(cfl<SM>(cs, cf, en.y * 16), lds2(xs + (en.x & 0xffffff) * 16)));
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (e + q < e_end) acc = dev::cadd(acc, u[q]);
      }
      sts2(xs + rc.x, dev::csub(t, dev::cadd(C2{0.0, 0.0}, dev::cmul(pv, acc))));
    } else if (rc.x >= 0 && !(rx.x & 2)) {
      gen_bwd_step<SM>(rc, rx, xs, cs, x, cf, be);
    }
    // general steps split over their rows' lanes (host-assigned: ext.x bit 1,
    // the row in bits 8..15): coupling sums per lane, exchanged by shuffle,
    // then each lane's row of the pivot product
    if (__any_sync(0xffffffffu, rc.x >= 0 && (rx.x & 2))) {
      const bool sp = rc.x >= 0 && (rx.x & 2);
      const int r = sp ? (rx.x >> 8) & 0xff : 0, mk = sp ? rx.y : 1, po = rc.y >> 4, xk = rc.x >> 4;
      C2 Pr[3], xo = {0.0, 0.0}, accr = {0.0, 0.0};
      if (sp) {
#pragma unroll
        for (int c = 0; c < 3; ++c) Pr[c] = cfl<SM>(cs, cf, (po + r * mk + min(c, mk - 1)) * 16);
        xo = lds2(xs + unsigned(xk + r) * 16u);
        accr = gen_bwd_acc_row<SM>(rx, xs, cs, cf, be, r);
      }
      const int base = lane - r;
      C2 ac[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int srcl = base + min(c, mk - 1);
        ac[c] = C2{__shfl_sync(0xffffffffu, accr.x, srcl), __shfl_sync(0xffffffffu, accr.y, srcl)};
      }
      if (sp) {
        C2 corr = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const C2 t = dev::cadd(corr, dev::cmul(Pr[c], ac[c]));
          corr = c < mk ? t : corr;
        }
        sts2(xs + unsigned(xk + r) * 16u, dev::csub(xo, corr));
      }
    }
    aa = aa_n;
    pv = pv_n;
    t = t_n;
    rc = nx;
    rx = nxx;
    nx = nx2;
    nxx = nxx2;
    if (wb > 1)
      __syncthreads();  // the round's values, for every warp of the scenario
    else
      __syncwarp();
  }
  // Suffix of all-scalar rounds (host-checked: every slot empty or a scalar
  // step with its single coupling): no vote, no extension records.
#pragma unroll (kBrSuffixUnroll)
  for (; br < nbr; ++br) {
#ifdef BR_TRACE
    if (tr_on && br < 80) {
      tr_a[br] = __ballot_sync(0xffffffffu, rc.x >= 0);
      tr_g[br] = 0;
      tr_t[br] = clock64();
    }
#endif
    const C2 xj = lds2(xs + (rc.x >= 0 ? rc.z : 0));
    const bool scn = nx.x >= 0;
    const C2 aa_n = cfl<SM>(cs, cf, scn ? nx.w : 0), pv_n = cfl<SM>(cs, cf, scn ? nx.y : 0);
    const C2 t_n = lds2(xs + (scn ? nx.x : 0));
    const int4 nx2 = rec4<SM>(ssl, bsl, min(br + 2, nbr) * rstride);
    // computed on every lane (empty slots on zeros), stored on active ones:
    // keeps the parent's load a straight-line first load, ahead of the next
    // round's operand loads in the shared-memory queue
#ifdef BR_TRACE
    if (tr_on && br < 80 && xj.x != 1.2345e300) tr_b[br] = clock64();
#endif
    const C2 acc = dev::cadd(C2{0.0, 0.0}, dev::cmul(aa, xj));
    const C2 res = dev::csub(t, dev::cadd(C2{0.0, 0.0}, dev::cmul(pv, acc)));
#ifdef BR_TRACE
    if (tr_on && br < 80 && res.x != 1.2345e300) tr_c[br] = clock64();
#endif
    if (rc.x >= 0) sts2(xs + rc.x, res);
    aa = aa_n;
    pv = pv_n;
    t = t_n;
    rc = nx;
    nx = nx2;
    if (wb > 1)
      __syncthreads();
    else
      __syncwarp();
  }
#ifdef BR_TRACE
  if (tr_on && lane == 0) {
    const long long tend = clock64();
    for (int br = 0; br < nbr && br < 80; ++br)
      printf("round %d: %lld cycles active %d general %d | xj at %lld, result at %lld\n", br,
             (br + 1 < nbr && br + 1 < 80 ? tr_t[br + 1] : tend) - tr_t[br], __popc(tr_a[br]), __popc(tr_g[br]),
             tr_b[br] ? tr_b[br] - tr_t[br] : -1LL, tr_c[br] ? tr_c[br] - tr_t[br] : -1LL);
  }
#endif
}

// SM: factor and program staged in shared memory (TMA); otherwise they are
// read from global memory (large networks) and only the solution vectors
// are staged.
template <bool SM>
__global__ void __launch_bounds__(256) base_refresh_kernel(BaseArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ unsigned long long bar, bar_prog;
  // The factor and the program never change during a run: with programmatic
  // dependent launch their TMA staging starts before the wait on the pick
  // kernel (which triggers its dependents early), overlapping its commit.
  if (SM && threadIdx.x == 0) {
    mbar_init(&bar_prog, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_prog, unsigned(a.ncf) * 16u + unsigned(a.nmeta) * 4u);
    if (a.ncf) bulk_g2s(smem, a.cfac, unsigned(a.ncf) * 16u, &bar_prog);
    bulk_g2s(reinterpret_cast<int*>(smem + a.ncf), a.meta, unsigned(a.nmeta) * 4u, &bar_prog);
  }
  griddep_wait();
  if (a.st && a.st->done) {
    if (SM) mbar_wait(&bar_prog, 0);  // no copy may outlive the CTA
    return;
  }
  if (a.tdbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.tdbg[size_t(a.st->iter) * kTdbg + 4] = t;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // one warp per scenario, or (WB > 1) one scenario per CTA with WB warps
  const int WB = a.WB, slot = WB > 1 ? 0 : warp;
  const bool lead = WB == 1 || warp == 0;  // the warp that runs the serial parts
  const int rhs = blockIdx.x * a.W + slot;
  const int nw = min(a.W, a.L - blockIdx.x * a.W);
  const double2* cf = SM ? smem : a.cfac;
  const int* M = SM ? reinterpret_cast<const int*>(smem + a.ncf) : a.meta;
  double2* xall = SM ? reinterpret_cast<double2*>(reinterpret_cast<int*>(smem + a.ncf) + a.nmeta) : smem;
  const bool stage_rhs = a.inc && a.rhs_staged;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // incremental: x <- last forward values, and the right-hand sides of the
    // re-eliminated path nodes from a second buffer (both TMA-staged)
    const unsigned per = unsigned(a.nphi) * 16u;
    const unsigned bytes = unsigned(nw) * per * (stage_rhs ? 2u : 1u);
    mbar_expect_tx(&bar, bytes);
    const double2* src = a.inc ? a.tfwd : a.iaggp;
    for (int w = 0; w < nw; ++w)
      bulk_g2s(xall + size_t(w) * a.nphi, src + size_t(blockIdx.x * a.W + w) * a.nphi, per, &bar);
    if (stage_rhs)
      for (int w = 0; w < nw; ++w)
        bulk_g2s(xall + size_t(a.W + w) * a.nphi, a.iaggp + size_t(blockIdx.x * a.W + w) * a.nphi, per, &bar);
  }
  __syncthreads();
  if (SM) mbar_wait(&bar_prog, 0);
  mbar_wait(&bar, 0);
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[0] = clock64();
  if (a.tdbg && blockIdx.x == 0 && tid == 0) a.tdbg[size_t(a.st->iter) * kTdbg + 8] = globaltimer_ns();
  if (slot >= nw) return;
  double2* x = xall + size_t(slot) * a.nphi;
  for (int k = lane; k < a.nkept && lead; k += 32) {
    const int xe = M[a.kept + 2 * k], ki = M[a.kept + 2 * k + 1];
    const int x0 = xe & 0xffffff, m = xe >> 24;
    for (int i = 0; i < m; ++i) x[x0 + i] = a.kept_val[ki * 3 + i];
  }
  __syncwarp();
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[1] = clock64();
  // records: int4 {x_k*16 (<0: empty), pinv*16, x_j0*16, block0*16} (byte
  // offsets into x / cf) + int4 {general?, m_k, first extra entry, extra count}.
  // Scalar steps (one present phase, single-phase pulls) run one straight-line
  // sequence on 32-bit shared addresses; the record arrays carry one padding
  // round so the prefetch of round i+1 is unconditional.
  const unsigned xs = unsigned(__cvta_generic_to_shared(x));
  const unsigned cs = SM ? unsigned(__cvta_generic_to_shared(cf)) : 0u;
  const int4* fs = reinterpret_cast<const int4*>(M + a.fslot);
  const int4* fx = reinterpret_cast<const int4*>(M + a.fext);
  const int2* fe = reinterpret_cast<const int2*>(M + a.fent);
  if (!a.inc && lead) {
    tree_forward<SM>(a, M, xs, cs, x, cf, lane);
    if (a.tfwd)  // keep the forward values for the next (incremental) refresh
      for (int r = lane; r < a.nphi; r += 32) a.tfwd[size_t(rhs) * a.nphi + r] = x[r];
  } else if (a.inc && lead && lane == 0) {
    // Walk the ancestors of the two changed nodes in elimination order. The
    // two path heads keep their walk entry and step records in registers; a
    // step issues its parent's record loads before its own arithmetic, and a
    // scalar step takes its right-hand side straight from the staged copy
    // (same operations and order as tree_fwd_step).
    const int4* W = reinterpret_cast<const int4*>(M + a.walk);
    // shared-space bases of the walk table and the forward records (program staged)
    const unsigned wsa = SM ? unsigned(__cvta_generic_to_shared(W)) : 0u;
    const unsigned fsa = SM ? unsigned(__cvta_generic_to_shared(fs)) : 0u;
    const unsigned fxa = SM ? unsigned(__cvta_generic_to_shared(fx)) : 0u;
    const double2* xr = stage_rhs ? xall + size_t(a.W + slot) * a.nphi : a.iaggp + size_t(rhs) * a.nphi;
    double2* tf = a.tfwd + size_t(rhs) * a.nphi;
    const int4 none = make_int4(-1, -1, 0x7fffffff, -1);
    int na = a.st ? a.st->last_s : a.inc_s, nb = a.st ? a.st->last_r : a.inc_r;
    int4 wa = na >= 0 ? rec4<SM>(wsa, W, na * 16) : none, wb = nb >= 0 ? rec4<SM>(wsa, W, nb * 16) : none;
    if (wa.x < 0) na = -1;  // kept (slack): no forward step
    if (wb.x < 0) nb = -1;
    int4 ra = na >= 0 ? rec4<SM>(fsa, fs, wa.x * 16) : none, xa = na >= 0 ? rec4<SM>(fxa, fx, wa.x * 16) : none;
    int4 rb = nb >= 0 ? rec4<SM>(fsa, fs, wb.x * 16) : none, xb = nb >= 0 ? rec4<SM>(fxa, fx, wb.x * 16) : none;
#ifdef BR_TRACE
    const long long wt0 = clock64();
    int wsteps = 0;
#endif
    while (na >= 0 || nb >= 0) {
#ifdef BR_TRACE
      ++wsteps;
#endif
      const bool ta = na >= 0 && (nb < 0 || wa.z <= wb.z);
      const bool tb = nb >= 0 && (na < 0 || wb.z <= wa.z);
      const int4 wk = ta ? wa : wb, rc = ta ? ra : rb, rx = ta ? xa : xb;
      const int4 wu = wk.y >= 0 ? rec4<SM>(wsa, W, wk.y * 16) : none;  // the parent's walk entry
      const int xk = rc.x >> 4;
      int4 ru = none, xu = none;  // the parent's step records, issued behind this step's operand loads
      const bool upok = wk.y >= 0;
      if (rc.x >= 0 && rc.z >= 0) {
        const C2 b0 = ld2(xr + xk), tj = lds2(xs + rc.z), t1 = lds2(xs + rx.x);
        const C2 aa = cfl<SM>(cs, cf, rc.w), pv = cfl<SM>(cs, cf, rc.y), a1 = cfl<SM>(cs, cf, rx.y);
        if (upok && wu.x >= 0) {
          ru = rec4<SM>(fsa, fs, wu.x * 16);
          xu = rec4<SM>(fxa, fx, wu.x * 16);
        }
        const C2 u0 = dev::cadd(C2{0.0, 0.0}, dev::cmul(aa, tj));
        const C2 u1 = dev::cadd(C2{0.0, 0.0}, dev::cmul(a1, t1));
        C2 bb = dev::csub(dev::csub(b0, u0), u1);
        for (int e = rx.z; e < rx.z + rx.w; ++e) {  // further children, elimination order
          const int2 en = fe[e];
          bb = dev::csub(bb, dev::cadd(C2{0.0, 0.0},
                                       dev::cmul(cfl<SM>(cs, cf, en.y * 16), lds2(xs + (en.x & 0xffffff) * 16))));
        }
        const C2 v = dev::cadd(C2{0.0, 0.0}, dev::cmul(pv, bb));
        sts2(xs + rc.x, v);
        st2(tf + xk, v);
      } else {
        // general step: the right-hand side into x, then tree_fwd_step
        const int mk = rx.y;
        for (int i = 0; i < mk; ++i) x[xk + i] = xr[xk + i];
        asm volatile("" ::: "memory");  // the step reads x through ld.shared asm
        tree_fwd_step<SM>(rc, rx, xs, cs, x, cf, fe);
        asm volatile("" ::: "memory");
        for (int i = 0; i < mk; ++i) tf[xk + i] = x[xk + i];
      }
      const int up = wk.y >= 0 && wu.x >= 0 ? wk.y : -1;  // stop below kept nodes
      if (up >= 0 && !(rc.x >= 0 && rc.z >= 0)) {
        ru = rec4<SM>(fsa, fs, wu.x * 16);
        xu = rec4<SM>(fxa, fx, wu.x * 16);
      }
      if (ta) {
        na = up;
        wa = wu;
        ra = ru;
        xa = xu;
      }
      if (tb) {
        nb = up;
        wb = wu;
        rb = ru;
        xb = xu;
      }
    }
#ifdef BR_TRACE
    if (a.st && blockIdx.x == 0 && warp == 0 && (a.st->iter % 100) == 1)
      printf("walk iter %d: %d steps, %lld cycles\n", a.st->iter, wsteps, clock64() - wt0);
#endif
  }
  if (WB > 1)
    __syncthreads();  // the lead warp's forward values
  else
    __syncwarp();  // the walk (lane 0) wrote x
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[2] = clock64();
  if (a.tdbg && blockIdx.x == 0 && tid == 0) a.tdbg[size_t(a.st->iter) * kTdbg + 9] = globaltimer_ns();
  tree_backward<SM>(a, M, xs, cs, x, cf, lane, WB, WB > 1 ? warp : 0);
  if (a.dbg && blockIdx.x == 0 && tid == 0) a.dbg[3] = clock64();
  if (a.tdbg && blockIdx.x == 0 && tid == 0) a.tdbg[size_t(a.st->iter) * kTdbg + 11] = globaltimer_ns();
  for (int r = WB > 1 ? tid : lane; r < a.nphi; r += 32 * WB) a.bv[bv_base(size_t(r), a.L, rhs)] = x[r];
  if (a.tdbg && blockIdx.x == 0 && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.tdbg[size_t(a.st->iter) * kTdbg + 5] = t;
  }
  if (a.tdbg && lane == 0) atomicMax(a.tdbg + size_t(a.st->iter) * kTdbg + 10, globaltimer_ns());
}

// cfac[i] = (src >= 0 ? (src & 1 ? pinv : blocks)[src >> 1] : 0)
__global__ void compact_gather_kernel(int ncf, const long long* src, const double2* blocks, const double2* pinv,
                                      double2* cfac) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncf) return;
  const long long s = src[i];
  cfac[i] = s < 0 ? make_double2(0.0, 0.0) : ((s & 1) ? pinv[s >> 1] : blocks[s >> 1]);
}

}  // namespace
}  // namespace kronred::b200
