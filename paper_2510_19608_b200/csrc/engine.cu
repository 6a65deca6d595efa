// engine.cu — sm_100a kernels and the device side of run_reduction.
//
// Kernels (SURVEY §2 "native components"):
//   K1f  elim_factor_kernel   level-scheduled block elimination: structural
//                             pseudo-inverse pivots, Schur contributions
//                             (A_ik pinv_k) A_kj into slots, ordered apply.
//                             Serves the anchored factorization
//                             (solver.cpp:20-117, 168-179) and kron_reduce
//                             (kron.cpp:34-46, Y_kk - Y_kr Y_rr^-1 Y_rk).
//   K1s  solve_kernel<MODE>   batched pull-form forward/backward sweeps
//                             (solver.cpp:119-148): scenario voltages, v0,
//                             the per-iteration base refresh (reduce.cpp:265)
//                             and the unit-injection Z columns (reduce.cpp:272).
//   K2/3 score_kernel         delta voltage Vc = base + sum_p c_p (Zs_p - Zr_p),
//                             |Vc|, voltage-margin feasibility and the ordered
//                             SMICE scan (reduce.cpp:80-123, 194-244).
//   K4   argmin_kernel        feasibility-masked lexicographic (smice, idx)
//                             argmin, warp shuffle then block (reduce.cpp:397-404).
//        commit_kernel        i_agg move + cluster min/max merge (reduce.cpp:336-343).
//
// Exactness: see kr_device.cuh. Every decision is bit-identical to the
// reference CPU program; the cluster max of |m - vhat_mag_j| over members is
// evaluated as max(m - min_j, max_j - m), which is exact because rounding is
// monotone (fl(m - v) is non-increasing in v).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <set>
#include <stdexcept>

#include "kr_device.cuh"
#include "kr_internal.hpp"

namespace kronred::b200 {

using dev::C2;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ C2 ld2(const double2* p) {
  const double2 v = *p;
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double2* p, C2 v) { *p = make_double2(v.x, v.y); }

__device__ __forceinline__ void load_blk(const double2* blocks, int id, C2 m[9]) {
  if (id < 0) {
#pragma unroll
    for (int e = 0; e < 9; ++e) m[e] = {0.0, 0.0};
    return;
  }
  const double2* p = blocks + size_t(id) * 9;
#pragma unroll
  for (int e = 0; e < 9; ++e) m[e] = ld2(p + e);
}

// Mat3c * Vec3c (complex3.hpp:85-90)
__device__ __forceinline__ void matvec(const C2 m[9], const C2 x[3], C2 r[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    C2 acc = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 3; ++j) acc = dev::cadd(acc, dev::cmul(m[i * 3 + j], x[j]));
    r[i] = acc;
  }
}

// Mat3c * Mat3c with exact-zero skip of the left entry (complex3.hpp:76-84)
__device__ __forceinline__ void matmul(const C2 a[9], const C2 b[9], C2 r[9]) {
#pragma unroll
  for (int e = 0; e < 9; ++e) r[e] = {0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const C2 aik = a[i * 3 + k];
      if (dev::cis0(aik)) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j) r[i * 3 + j] = dev::cadd(r[i * 3 + j], dev::cmul(aik, b[k * 3 + j]));
    }
}

__device__ __forceinline__ double cabs_dev(C2 z) { return hypot(z.x, z.y); }

// masked_inverse (complex3.cpp:9-61). Pivot magnitudes use hypot (glibc cabs
// on the host); they only select pivots / gate singularity.
__device__ bool masked_inverse(const C2 in[9], unsigned mask, C2 out[9], double tol, double& smallest) {
#pragma unroll
  for (int e = 0; e < 9; ++e) out[e] = {0.0, 0.0};
  int idx[3];
  int k = 0;
  for (int p = 0; p < 3; ++p)
    if ((mask >> p) & 1u) idx[k++] = p;
  smallest = 0.0;
  if (k == 0) return true;
  C2 a[3][3], inv[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      a[i][j] = {0.0, 0.0};
      inv[i][j] = {0.0, 0.0};
    }
  for (int i = 0; i < k; ++i) {
    inv[i][i] = {1.0, 0.0};
    for (int j = 0; j < k; ++j) a[i][j] = in[idx[i] * 3 + idx[j]];
  }
  smallest = __longlong_as_double(0x7ff0000000000000LL);
  for (int col = 0; col < k; ++col) {
    int piv = col;
    double best = cabs_dev(a[col][col]);
    for (int r = col + 1; r < k; ++r) {
      const double m = cabs_dev(a[r][col]);
      if (m > best) {
        best = m;
        piv = r;
      }
    }
    smallest = fmin(smallest, best);
    if (best <= tol) return false;
    if (piv != col)
      for (int j = 0; j < 3; ++j) {
        C2 t = a[piv][j];
        a[piv][j] = a[col][j];
        a[col][j] = t;
        t = inv[piv][j];
        inv[piv][j] = inv[col][j];
        inv[col][j] = t;
      }
    const C2 d = a[col][col];
    for (int j = 0; j < k; ++j) {
      a[col][j] = dev::cdiv(a[col][j], d);
      inv[col][j] = dev::cdiv(inv[col][j], d);
    }
    for (int r = 0; r < k; ++r) {
      if (r == col) continue;
      const C2 f = a[r][col];
      if (dev::cis0(f)) continue;
      for (int j = 0; j < k; ++j) {
        a[r][j] = dev::csub(a[r][j], dev::cmul(f, a[col][j]));
        inv[r][j] = dev::csub(inv[r][j], dev::cmul(f, inv[col][j]));
      }
    }
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) out[idx[i] * 3 + idx[j]] = inv[i][j];
  return true;
}

// ---------------------------------------------------------------------------
// K1f: elimination executor

struct ElimDev {
  int nlevels;
  const int *step_node, *step_diag;
  const int *lvl_step_off, *lvl_steps;
  const int *lvl_slot_off, *lvl_slots, *lvl_slot_step;
  const int *slot_from, *slot_to;
  const int *lvl_apply_off, *apply_blk, *apply_off, *apply_slots;
  const std::uint8_t* mask;
  double2* blocks;
  double2* pinv;
  double2* contrib;
  double pivot_floor;
  unsigned long long* fail;  // packed (step << 0) min; fail_info[step] gets pivot
  double* fail_pivot;
};

__global__ void __launch_bounds__(1024) elim_factor_kernel(ElimDev e) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int lev = 0; lev < e.nlevels; ++lev) {
    // A1: structural pseudo-inverse of every pivot at this level
    const int s0 = e.lvl_step_off[lev], s1 = e.lvl_step_off[lev + 1];
    for (int i = s0 + tid; i < s1; i += nt) {
      const int st = e.lvl_steps[i];
      const int k = e.step_node[st];
      C2 d[9], pv[9];
      load_blk(e.blocks, e.step_diag[st], d);
      double smallest;
      if (!masked_inverse(d, e.mask[k], pv, e.pivot_floor, smallest)) {
        const unsigned long long old = atomicMin(e.fail, (unsigned long long)st);
        (void)old;
        e.fail_pivot[st] = smallest;
      }
      double2* out = e.pinv + size_t(st) * 9;
#pragma unroll
      for (int q = 0; q < 9; ++q) st2(out + q, pv[q]);
    }
    __syncthreads();
    // A2: Schur contributions (A_ik pinv_k) A_kj (solver.cpp:94-100)
    const int q0 = e.lvl_slot_off[lev], q1 = e.lvl_slot_off[lev + 1];
    for (int i = q0 + tid; i < q1; i += nt) {
      const int sl = e.lvl_slots[i];
      const int st = e.lvl_slot_step[i];
      C2 a[9], p[9], t[9], b[9], c[9];
      load_blk(e.blocks, e.slot_from[sl], a);
      load_blk(e.pinv, st, p);
      matmul(a, p, t);
      load_blk(e.blocks, e.slot_to[sl], b);
      matmul(t, b, c);
      double2* out = e.contrib + size_t(sl) * 9;
#pragma unroll
      for (int q = 0; q < 9; ++q) st2(out + q, c[q]);
    }
    __syncthreads();
    // B: ordered apply, block -= contribution in elimination order
    const int a0 = e.lvl_apply_off[lev], a1 = e.lvl_apply_off[lev + 1];
    for (int i = a0 + tid; i < a1; i += nt) {
      const int b = e.apply_blk[i];
      C2 x[9];
      load_blk(e.blocks, b, x);
      for (int j = e.apply_off[i]; j < e.apply_off[i + 1]; ++j) {
        C2 c[9];
        load_blk(e.contrib, e.apply_slots[j], c);
#pragma unroll
        for (int q = 0; q < 9; ++q) x[q] = dev::csub(x[q], c[q]);
      }
      double2* out = e.blocks + size_t(b) * 9;
#pragma unroll
      for (int q = 0; q < 9; ++q) st2(out + q, x[q]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K1s: batched solves

enum SolveMode { MODE_FULL = 0, MODE_BASE = 1, MODE_ZCOL = 2 };

struct SolveDev {
  int n, nfw, nbw;
  const int *step_node, *in_off, *in_node, *in_blk;
  const int *fw_off, *fw_steps, *bw_off, *bw_steps;
  const int *cpl_off, *cpl_node, *cpl_to;
  const double2* blocks;
  const double2* pinv;
  int nkept;
  const int* kept;            // kept node ids
  const double2* kept_val;    // [nkept][3] preset voltages
  double2* w;                 // [n][NR][3]
  int NR;                     // rhs slots in w
  int nrhs;                   // rhs in this launch
  int G;                      // rhs per CTA
  // sources / sinks
  const double2* rhs_full;    // MODE_FULL: [nrhs][3n] or null (zero)
  double2* out_full;          // MODE_FULL: [nrhs][3n]
  const double2* iagg;        // MODE_BASE: [n][L][3]
  double2* base;              // MODE_BASE: [nphi][L]
  int L;
  int nphi;
  const int* prow_node;       // [nphi]
  const std::uint8_t* prow_phase;
  int col0;                   // MODE_ZCOL: first column of this launch
  const double2* v0p;         // [nphi]
  double2* zout;              // [ncol][nphi], column-major
};

template <int MODE>
__global__ void __launch_bounds__(512) solve_kernel(SolveDev a) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int r0 = blockIdx.x * a.G;
  const int gc = min(a.G, a.nrhs - r0);
  if (gc <= 0) return;
  auto W = [&](int node, int rhs) { return a.w + (size_t(node) * a.NR + rhs) * 3; };
  // forward: rhs_k = b_k - sum_j A_kj t_j (elimination order), t_k = pinv_k rhs_k
  for (int lev = 0; lev < a.nfw; ++lev) {
    const int o0 = a.fw_off[lev], cnt = a.fw_off[lev + 1] - o0;
    for (int idx = tid; idx < cnt * gc; idx += nt) {
      const int st = a.fw_steps[o0 + idx / gc];
      const int rhs = r0 + idx % gc;
      const int k = a.step_node[st];
      C2 b[3];
      if (MODE == MODE_FULL) {
        if (a.rhs_full) {
          const double2* src = a.rhs_full + size_t(rhs) * 3 * a.n + size_t(k) * 3;
          for (int p = 0; p < 3; ++p) b[p] = ld2(src + p);
        } else {
          for (int p = 0; p < 3; ++p) b[p] = {0.0, 0.0};
        }
      } else if (MODE == MODE_BASE) {
        const double2* src = a.iagg + (size_t(k) * a.L + rhs) * 3;
        for (int p = 0; p < 3; ++p) b[p] = ld2(src + p);
      } else {
        const int col = a.col0 + rhs;
        const int cn = a.prow_node[col];
        const int cp = a.prow_phase[col];
        for (int p = 0; p < 3; ++p) b[p] = (k == cn && p == cp) ? C2{1.0, 0.0} : C2{0.0, 0.0};
      }
      for (int e = a.in_off[st]; e < a.in_off[st + 1]; ++e) {
        C2 m[9], tj[3], u[3];
        load_blk(a.blocks, a.in_blk[e], m);
        const double2* tp = W(a.in_node[e], rhs);
        for (int p = 0; p < 3; ++p) tj[p] = ld2(tp + p);
        matvec(m, tj, u);
        for (int p = 0; p < 3; ++p) b[p] = dev::csub(b[p], u[p]);
      }
      C2 pv[9], t[3];
      load_blk(a.pinv, st, pv);
      matvec(pv, b, t);
      double2* wp = W(k, rhs);
      for (int p = 0; p < 3; ++p) st2(wp + p, t[p]);
    }
    __syncthreads();
  }
  // boundary values of kept nodes
  for (int idx = tid; idx < a.nkept * gc; idx += nt) {
    const int kk = idx / gc, rhs = r0 + idx % gc;
    double2* wp = W(a.kept[kk], rhs);
    for (int p = 0; p < 3; ++p) wp[p] = a.kept_val[kk * 3 + p];
  }
  __syncthreads();
  // backward: x_k = t_k - pinv_k (sum_c A_kc x_c), couplings ascending
  for (int lev = 0; lev < a.nbw; ++lev) {
    const int o0 = a.bw_off[lev], cnt = a.bw_off[lev + 1] - o0;
    for (int idx = tid; idx < cnt * gc; idx += nt) {
      const int st = a.bw_steps[o0 + idx / gc];
      const int rhs = r0 + idx % gc;
      const int k = a.step_node[st];
      C2 acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int c = a.cpl_off[st]; c < a.cpl_off[st + 1]; ++c) {
        C2 m[9], xj[3], u[3];
        load_blk(a.blocks, a.cpl_to[c], m);
        const double2* xp = W(a.cpl_node[c], rhs);
        for (int p = 0; p < 3; ++p) xj[p] = ld2(xp + p);
        matvec(m, xj, u);
        for (int p = 0; p < 3; ++p) acc[p] = dev::cadd(acc[p], u[p]);
      }
      C2 pv[9], corr[3];
      load_blk(a.pinv, st, pv);
      matvec(pv, acc, corr);
      double2* wp = W(k, rhs);
      for (int p = 0; p < 3; ++p) st2(wp + p, dev::csub(ld2(wp + p), corr[p]));
    }
    __syncthreads();
  }
  // outputs
  if (MODE == MODE_FULL) {
    for (int idx = tid; idx < gc * a.n * 3; idx += nt) {
      const int g = idx / (a.n * 3), t = idx % (a.n * 3);
      const int rhs = r0 + g;
      a.out_full[size_t(rhs) * 3 * a.n + t] = W(t / 3, rhs)[t % 3];
    }
  } else if (MODE == MODE_BASE) {
    for (int idx = tid; idx < a.nphi * gc; idx += nt) {
      const int rho = idx / gc, rhs = r0 + idx % gc;
      a.base[size_t(rho) * a.L + rhs] = W(a.prow_node[rho], rhs)[a.prow_phase[rho]];
    }
  } else {
    for (int idx = tid; idx < a.nphi * gc; idx += nt) {
      const int g = idx / a.nphi, rho = idx % a.nphi;
      const int rhs = r0 + g;
      const C2 x = ld2(W(a.prow_node[rho], rhs) + a.prow_phase[rho]);
      st2(a.zout + size_t(a.col0 + rhs) * a.nphi + rho, dev::csub(x, ld2(a.v0p + rho)));
    }
  }
}

// ---------------------------------------------------------------------------
// K2/K3: fused delta contraction + magnitude + feasibility + ordered SMICE

struct ScoreDev {
  int C;          // candidates in this launch
  int L;
  int nphi;
  int ns;         // active super-nodes
  const int* cand_s;
  const int* cand_r;
  const int* sn;  // active super-nodes, ascending
  const int* prow_off;
  const std::uint8_t* mask;
  const double2* Z;      // [nphi cols][nphi rows]
  const double2* base;   // [nphi][L]
  const double* vmin;    // [nphi][L]
  const double* vmax;    // [nphi][L]
  const double2* iagg;   // [n][L][3]
  int objective;
  const int* mem_off;    // complex objective: CSR members per super-node id
  const int* mem_list;
  const double2* vhatp;  // [nphi][L]
  double* out_smice;     // [C][L]
  double* out_maxerr;    // [C][L]
};

__global__ void __launch_bounds__(128) score_kernel(ScoreDev a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.C * a.L) return;
  const int c = q / a.L, l = q - c * a.L;
  const int s = a.cand_s[c], r = a.cand_r[c];
  const unsigned ms = a.mask[s], mr = a.mask[r];
  const int rs0 = a.prow_off[s], rr0 = a.prow_off[r];
  // loaded phases of r (reduce.cpp:225-233): c = i_agg[l][3r+p] != 0
  C2 cv[3];
  int zs[3], zr[3];
  int nl = 0;
  for (int p = 0; p < 3; ++p) {
    if (!((mr >> p) & 1u)) continue;
    const C2 cz = ld2(a.iagg + (size_t(r) * a.L + l) * 3 + p);
    if (dev::cis0(cz)) continue;
    cv[nl] = cz;
    zs[nl] = rs0 + __popc(ms & ((1u << p) - 1u));
    zr[nl] = rr0 + __popc(mr & ((1u << p) - 1u));
    ++nl;
  }
  const size_t nphi = size_t(a.nphi);
  double smice = 0.0, maxerr = 0.0;
  for (int k = 0; k < a.ns; ++k) {
    const int i = a.sn[k];
    if (i == r) continue;
    const unsigned mi = a.mask[i];
    const int ri0 = a.prow_off[i];
    double cm = 0.0;
    C2 vrow[3];
    int t = 0;
    for (int p = 0; p < 3; ++p) {
      if (!((mi >> p) & 1u)) continue;
      const int rho = ri0 + t;
      ++t;
      C2 v = ld2(a.base + size_t(rho) * a.L + l);
      for (int j = 0; j < nl; ++j) {
        const C2 za = ld2(a.Z + size_t(zs[j]) * nphi + rho);
        const C2 zb = ld2(a.Z + size_t(zr[j]) * nphi + rho);
        const double dr = dev::dsub(za.x, zb.x), di = dev::dsub(za.y, zb.y);
        v.x = dev::dadd(v.x, dev::dsub(dev::dmul(cv[j].x, dr), dev::dmul(cv[j].y, di)));
        v.y = dev::dadd(v.y, dev::dadd(dev::dmul(cv[j].x, di), dev::dmul(cv[j].y, dr)));
      }
      vrow[p] = v;
      const double m = dev::dsqrt(dev::dadd(dev::dmul(v.x, v.x), dev::dmul(v.y, v.y)));
      double lo = a.vmin[size_t(rho) * a.L + l], hi = a.vmax[size_t(rho) * a.L + l];
      if (i == s && ((mr >> p) & 1u)) {
        const int rr = rr0 + __popc(mr & ((1u << p) - 1u));
        lo = fmin(lo, a.vmin[size_t(rr) * a.L + l]);
        hi = fmax(hi, a.vmax[size_t(rr) * a.L + l]);
      }
      const double em = fmax(dev::dsub(m, lo), dev::dsub(hi, m));
      maxerr = fmax(maxerr, em);
      cm = fmax(cm, em);
    }
    if (a.objective == KRG_OBJ_COMPLEX) {
      // objective entries are complex distances (reduce.cpp:102-106)
      cm = 0.0;
      for (int pass = 0; pass < (i == s ? 2 : 1); ++pass) {
        const int owner = pass == 0 ? i : r;
        for (int e = a.mem_off[owner]; e < a.mem_off[owner + 1]; ++e) {
          const int j = a.mem_list[e];
          const unsigned mj = a.mask[j];
          int tj = 0;
          for (int p = 0; p < 3; ++p) {
            if (!((mj >> p) & 1u)) continue;
            const C2 vh = ld2(a.vhatp + size_t(a.prow_off[j] + tj) * a.L + l);
            ++tj;
            const double dr = dev::dsub(vrow[p].x, vh.x), di = dev::dsub(vrow[p].y, vh.y);
            const double eo = dev::dsqrt(dev::dadd(dev::dmul(dr, dr), dev::dmul(di, di)));
            cm = fmax(cm, eo);
          }
        }
      }
    }
    smice = dev::dadd(smice, cm);
  }
  a.out_smice[q] = smice;
  a.out_maxerr[q] = maxerr;
}

// ---------------------------------------------------------------------------
// K4: per-candidate scenario sum + feasibility, lexicographic argmin

struct BestRec {
  double smice;
  long long idx;
};

__device__ __forceinline__ bool better(double s1, long long i1, double s2, long long i2) {
  if (i1 < 0) return false;
  if (i2 < 0) return true;
  return s1 < s2 || (s1 == s2 && i1 < i2);
}

__global__ void __launch_bounds__(1024) argmin_kernel(int C, int L, double e_bar, long long c_base,
                                                      const double* smice_l, const double* maxerr_l,
                                                      double* out /* [2 + L] */) {
  __shared__ double ss[32];
  __shared__ long long si[32];
  double bs = __longlong_as_double(0x7ff0000000000000LL);
  long long bi = -1;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    bool feasible = true;
    double sum = 0.0;
    for (int l = 0; l < L; ++l) {
      feasible = feasible && !(maxerr_l[size_t(c) * L + l] > e_bar);
      sum = dev::dadd(sum, smice_l[size_t(c) * L + l]);
    }
    if (feasible && better(sum, c, bs, bi)) {
      bs = sum;
      bi = c;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double os = __shfl_down_sync(0xffffffffu, bs, off);
    const long long oi = __shfl_down_sync(0xffffffffu, bi, off);
    if (better(os, oi, bs, bi)) {
      bs = os;
      bi = oi;
    }
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    ss[warp] = bs;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    bs = lane < nw ? ss[lane] : __longlong_as_double(0x7ff0000000000000LL);
    bi = lane < nw ? si[lane] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_down_sync(0xffffffffu, bs, off);
      const long long oi = __shfl_down_sync(0xffffffffu, bi, off);
      if (better(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
      }
    }
    if (lane == 0) {
      si[0] = bi;
      ss[0] = bs;
    }
  }
  __syncthreads();
  bi = si[0];
  if (threadIdx.x == 0) {
    out[0] = ss[0];
    out[1] = __longlong_as_double(bi < 0 ? -1 : bi + c_base);
  }
  for (int l = threadIdx.x; l < L; l += blockDim.x)
    out[2 + l] = bi < 0 ? 0.0 : maxerr_l[size_t(bi) * L + l];
}

// commit: i_agg[s] += i_agg[r], i_agg[r] = 0 (reduce.cpp:336-343); the
// absorbing cluster's per-phase min/max of member |V-hat| takes r's.
__global__ void commit_kernel(int s, int r, int L, unsigned ms, unsigned mr, int rs0, int rr0,
                              double2* iagg, double* vmin, double* vmax) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  for (int p = 0; p < 3; ++p) {
    double2* ps = iagg + (size_t(s) * L + l) * 3 + p;
    double2* pr = iagg + (size_t(r) * L + l) * 3 + p;
    st2(ps, dev::cadd(ld2(ps), ld2(pr)));
    *pr = make_double2(0.0, 0.0);
    if ((mr >> p) & 1u) {
      const size_t a = size_t(rs0 + __popc(ms & ((1u << p) - 1u))) * L + l;
      const size_t b = size_t(rr0 + __popc(mr & ((1u << p) - 1u))) * L + l;
      vmin[a] = fmin(vmin[a], vmin[b]);
      vmax[a] = fmax(vmax[a], vmax[b]);
    }
  }
}

// scenario data prep: present-row V-hat, |V-hat| (kernels::magnitude order),
// initial cluster bounds and the [n][L][3] aggregated injections.
__global__ void prep_kernel(int n, int L, int nphi, const int* prow_node, const std::uint8_t* prow_phase,
                            const double2* vhat_full, const double2* inj_full, double2* vhatp,
                            double* vmag, double* vmin, double* vmax, double2* iagg) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < nphi * L) {
    const int rho = idx / L, l = idx % L;
    const C2 v = ld2(vhat_full + size_t(l) * 3 * n + size_t(prow_node[rho]) * 3 + prow_phase[rho]);
    const double m = dev::dsqrt(dev::dadd(dev::dmul(v.x, v.x), dev::dmul(v.y, v.y)));
    st2(vhatp + idx, v);
    vmag[idx] = m;
    vmin[idx] = m;
    vmax[idx] = m;
  }
  if (idx < n * L * 3) {
    const int node = idx / (L * 3), rem = idx % (L * 3), l = rem / 3, p = rem % 3;
    iagg[idx] = inj_full[size_t(l) * 3 * n + size_t(node) * 3 + p];
  }
}

// Unfused FP64 op-rate probe: 8 independent DMUL->DADD chains per thread.
__global__ void __launch_bounds__(256) fp64_probe_kernel(int iters, double a, double b, double* sink) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) sink[0] = s;
}

__global__ void selftest_cdiv_kernel(int N, const double* in, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const C2 r = dev::cdiv({in[4 * i], in[4 * i + 1]}, {in[4 * i + 2], in[4 * i + 3]});
  out[2 * i] = r.x;
  out[2 * i + 1] = r.y;
}

// ---------------------------------------------------------------------------
// device buffers

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) count = 1;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

}  // namespace

// ---------------------------------------------------------------------------
// Engine implementation

struct DevElim {
  ElimSchedule h;
  DBuf<int> ints;
  std::vector<size_t> off;  // offsets of each int array in `ints`
  DBuf<double2> blocks, pinv, contrib;
  DBuf<std::uint8_t> mask;
  DBuf<unsigned long long> fail;
  DBuf<double> fail_pivot;
  const int* P(int which) const { return ints.p + off[size_t(which)]; }
};

enum IntArr {
  A_STEP_NODE, A_STEP_DIAG, A_LVL_STEP_OFF, A_LVL_STEPS, A_LVL_SLOT_OFF, A_LVL_SLOTS,
  A_LVL_SLOT_STEP, A_SLOT_FROM, A_SLOT_TO, A_LVL_APPLY_OFF, A_APPLY_BLK, A_APPLY_OFF,
  A_APPLY_SLOTS, A_IN_OFF, A_IN_NODE, A_IN_BLK, A_FW_OFF, A_FW_STEPS, A_BW_OFF, A_BW_STEPS,
  A_CPL_OFF, A_CPL_NODE, A_CPL_TO, A_KEPT, A_COUNT
};

struct Engine::Impl {
  Problem prob;
  int device = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  int n = 0, L = 0, nphi = 0;
  std::vector<int> prow_off, prow_node;
  std::vector<std::uint8_t> prow_phase;
  DBuf<int> d_prow_off, d_prow_node;
  DBuf<std::uint8_t> d_prow_phase, d_mask;
  DBuf<double2> d_yin;        // assembled Y blocks (input, resident)
  double pivot_floor = 0;
  DevElim full;               // anchored factorization of Y
  DBuf<double2> d_w;          // solve scratch
  DBuf<double2> d_inj, d_vhat, d_v0, d_v0p, d_vhatp, d_iagg, d_base, d_Z;
  DBuf<double> d_vmag, d_vmin, d_vmax;
  std::vector<double> h_vhat;  // [L][3n][2]
  DBuf<int> d_cs, d_cr, d_sn, d_memoff, d_memlist;
  DBuf<double> d_psmice, d_pmaxerr, d_best;
  double* h_best = nullptr;    // pinned [2 + L]
  DBuf<double2> d_slackv;
  // multi-GPU
  int rank = 0, world = 1;
  krg_exchange_fn xfn = nullptr;
  void* xuser = nullptr;
  // loop state
  ReductionConfig cfg;
  HostState hs;
  std::vector<int> cs, cr;
  bool loop_active = false;
  bool z_valid = false;
  // kernel statistics (enabled on demand; CUDA events on the launching stream)
  bool profile = false;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_run0 = nullptr, ev_run1 = nullptr;
  KernelStats score_stats{}, solve_stats{};
  double last_run_ms = 0;

  void launched() { ++launches; }

  void ensure_events() {
    if (!ev_a) {
      CK(cudaEventCreate(&ev_a));
      CK(cudaEventCreate(&ev_b));
      CK(cudaEventCreate(&ev_run0));
      CK(cudaEventCreate(&ev_run1));
    }
  }

  // algorithmic work of one score launch: flops and bytes
  void score_work(long long c0, long long c1, double& flops, double& bytes) const {
    long long R = 0;
    for (int i : hs.supernodes) R += PhaseMask{prob.mask[size_t(i)]}.count();
    const long long ns = (long long)hs.supernodes.size();
    std::set<int> cols;
    flops = 0;
    for (long long c = c0; c < c1; ++c) {
      const int q = PhaseMask{prob.mask[size_t(cr[size_t(c)])]}.count();
      const double Rp = double(R - q);
      flops += 2.0 * q * Rp + double(L) * ((8.0 * q + 4.0) * Rp + 2.0 * nphi + double(ns - 1));
      cols.insert(cs[size_t(c)]);
      cols.insert(cr[size_t(c)]);
    }
    long long zc = 0;
    for (int node : cols) zc += PhaseMask{prob.mask[size_t(node)]}.count();
    bytes = 16.0 * double(zc) * double(R)          // Z columns of every endpoint over active rows
            + double(L) * double(R) * (16.0 + 16.0)  // base + cluster min/max
            + double(c1 - c0) * (8.0 + 48.0 * L)     // candidates + i_agg of r
            + 4.0 * double(ns) + 16.0 * double(c1 - c0) * L;  // super-node list + outputs
  }

  void upload_elim(DevElim& d, const FlatBlocks& y, const std::vector<std::uint8_t>& mask,
                   const std::vector<int>& elim) {
    d.h = build_schedule(y, mask, elim);
    const ElimSchedule& h = d.h;
    const std::vector<const std::vector<int>*> arrs = {
        &h.step_node, &h.step_diag, &h.lvl_step_off, &h.lvl_steps, &h.lvl_slot_off, &h.lvl_slots,
        &h.lvl_slot_step, &h.slot_from, &h.slot_to, &h.lvl_apply_off, &h.apply_blk, &h.apply_off,
        &h.apply_slots, &h.in_off, &h.in_node, &h.in_blk, &h.fw_off, &h.fw_steps, &h.bw_off,
        &h.bw_steps, &h.cpl_off, &h.cpl_node, &h.cpl_to, &h.kept};
    d.off.assign(A_COUNT + 1, 0);
    for (int i = 0; i < A_COUNT; ++i) d.off[size_t(i) + 1] = d.off[size_t(i)] + arrs[size_t(i)]->size();
    std::vector<int> packed(d.off[A_COUNT]);
    for (int i = 0; i < A_COUNT; ++i)
      std::copy(arrs[size_t(i)]->begin(), arrs[size_t(i)]->end(), packed.begin() + long(d.off[size_t(i)]));
    d.ints.alloc(packed.size());
    CK(cudaMemcpyAsync(d.ints.p, packed.data(), packed.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    d.blocks.alloc(size_t(h.nblocks) * 9);
    d.pinv.alloc(size_t(std::max(h.nsteps, 1)) * 9);
    d.contrib.alloc(size_t(std::max(h.nslots, 1)) * 9);
    d.mask.alloc(mask.size());
    CK(cudaMemcpyAsync(d.mask.p, mask.data(), mask.size(), cudaMemcpyHostToDevice, stream));
    d.fail.alloc(1);
    d.fail_pivot.alloc(size_t(std::max(h.nsteps, 1)));
    CK(cudaStreamSynchronize(stream));
  }

  // K1f on the device: blocks <- input, fill <- 0, then the level executor.
  void factorize(DevElim& d, const double2* d_input, double floor) {
    const ElimSchedule& h = d.h;
    if (h.n_input > 0)
      CK(cudaMemcpyAsync(d.blocks.p, d_input, size_t(h.n_input) * 9 * sizeof(double2),
                         cudaMemcpyDeviceToDevice, stream));
    if (h.nblocks > h.n_input)
      CK(cudaMemsetAsync(d.blocks.p + size_t(h.n_input) * 9, 0,
                         size_t(h.nblocks - h.n_input) * 9 * sizeof(double2), stream));
    const unsigned long long none = ~0ull;
    CK(cudaMemcpyAsync(d.fail.p, &none, sizeof(none), cudaMemcpyHostToDevice, stream));
    if (h.nlevels > 0) {
      ElimDev e;
      e.nlevels = h.nlevels;
      e.step_node = d.P(A_STEP_NODE);
      e.step_diag = d.P(A_STEP_DIAG);
      e.lvl_step_off = d.P(A_LVL_STEP_OFF);
      e.lvl_steps = d.P(A_LVL_STEPS);
      e.lvl_slot_off = d.P(A_LVL_SLOT_OFF);
      e.lvl_slots = d.P(A_LVL_SLOTS);
      e.lvl_slot_step = d.P(A_LVL_SLOT_STEP);
      e.slot_from = d.P(A_SLOT_FROM);
      e.slot_to = d.P(A_SLOT_TO);
      e.lvl_apply_off = d.P(A_LVL_APPLY_OFF);
      e.apply_blk = d.P(A_APPLY_BLK);
      e.apply_off = d.P(A_APPLY_OFF);
      e.apply_slots = d.P(A_APPLY_SLOTS);
      e.mask = d.mask.p;
      e.blocks = d.blocks.p;
      e.pinv = d.pinv.p;
      e.contrib = d.contrib.p;
      e.pivot_floor = floor;
      e.fail = d.fail.p;
      e.fail_pivot = d.fail_pivot.p;
      elim_factor_kernel<<<1, 1024, 0, stream>>>(e);
      launched();
      CK(cudaGetLastError());
    }
    unsigned long long failed = 0;
    CK(cudaMemcpyAsync(&failed, d.fail.p, sizeof(failed), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (failed != ~0ull) {
      double piv = 0;
      CK(cudaMemcpy(&piv, d.fail_pivot.p + failed, sizeof(double), cudaMemcpyDeviceToHost));
      const int node = h.step_node[size_t(failed)];
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.3e", piv);
      throw SolverError("singular present-phase diagonal while eliminating node " + std::to_string(node) +
                            " (smallest pivot " + buf + ", " + std::to_string(h.nsteps - int(failed)) +
                            " of " + std::to_string(h.nsteps) + " eliminations left)",
                        piv, node);
    }
  }

  SolveDev solve_args(DevElim& d, const double2* kept_val, int NR) {
    const ElimSchedule& h = d.h;
    SolveDev a{};
    a.n = h.n;
    a.nfw = h.nfw;
    a.nbw = h.nbw;
    a.step_node = d.P(A_STEP_NODE);
    a.in_off = d.P(A_IN_OFF);
    a.in_node = d.P(A_IN_NODE);
    a.in_blk = d.P(A_IN_BLK);
    a.fw_off = d.P(A_FW_OFF);
    a.fw_steps = d.P(A_FW_STEPS);
    a.bw_off = d.P(A_BW_OFF);
    a.bw_steps = d.P(A_BW_STEPS);
    a.cpl_off = d.P(A_CPL_OFF);
    a.cpl_node = d.P(A_CPL_NODE);
    a.cpl_to = d.P(A_CPL_TO);
    a.blocks = d.blocks.p;
    a.pinv = d.pinv.p;
    a.nkept = int(h.kept.size());
    a.kept = d.P(A_KEPT);
    a.kept_val = kept_val;
    d_w.alloc(size_t(h.n) * size_t(NR) * 3);
    a.w = d_w.p;
    a.NR = NR;
    return a;
  }

  // Full anchored solves: rhs [nrhs][3n] (device, may be null) -> out [nrhs][3n]
  void solve_full(DevElim& d, const double2* kept_val, const double2* rhs, int nrhs, double2* out) {
    const int chunk = 1024;
    for (int r0 = 0; r0 < nrhs; r0 += chunk) {
      const int nr = std::min(chunk, nrhs - r0);
      SolveDev a = solve_args(d, kept_val, nr);
      a.nrhs = nr;
      a.G = 4;
      a.rhs_full = rhs ? rhs + size_t(r0) * 3 * d.h.n : nullptr;
      a.out_full = out + size_t(r0) * 3 * d.h.n;
      solve_kernel<MODE_FULL><<<(nr + a.G - 1) / a.G, 512, 0, stream>>>(a);
      launched();
      CK(cudaGetLastError());
    }
  }

  SolveDev prow_args(SolveDev a) {
    a.nphi = nphi;
    a.prow_node = d_prow_node.p;
    a.prow_phase = d_prow_phase.p;
    return a;
  }

  void refresh_base() {
    SolveDev a = prow_args(solve_args(full, d_slackv.p, L));
    a.nrhs = L;
    a.G = 1;
    a.iagg = d_iagg.p;
    a.base = d_base.p;
    a.L = L;
    if (profile) CK(cudaEventRecord(ev_a, stream));
    solve_kernel<MODE_BASE><<<L, 512, 0, stream>>>(a);
    launched();
    CK(cudaGetLastError());
    if (profile) {
      CK(cudaEventRecord(ev_b, stream));
      CK(cudaEventSynchronize(ev_b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
      solve_stats.launches += 1;
      solve_stats.ms += ms;
      // forward + backward: per node and RHS ~ (in-degree + 2) Mat3c*Vec3c (54 flops each)
      solve_stats.flops += double(L) * double(full.h.nsteps) * 3.0 * 54.0;
      solve_stats.bytes += double(full.h.nsteps) * (3.0 * 144.0) + double(L) * n * 48.0 * 2.0;
    }
  }

  void build_z() {
    d_Z.alloc(size_t(nphi) * size_t(nphi));
    const int chunk = std::max(64, std::min(nphi, int((size_t(1) << 30) / (size_t(n) * 48))));
    for (int c0 = 0; c0 < nphi; c0 += chunk) {
      const int nc = std::min(chunk, nphi - c0);
      SolveDev a = prow_args(solve_args(full, d_slackv.p, nc));
      a.nrhs = nc;
      a.G = 8;
      a.col0 = c0;
      a.v0p = d_v0p.p;
      a.zout = d_Z.p;
      solve_kernel<MODE_ZCOL><<<(nc + a.G - 1) / a.G, 512, 0, stream>>>(a);
      launched();
      CK(cudaGetLastError());
    }
  }

  Impl(const Problem& p, int dev_id) : prob(p), device(dev_id) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw CudaError("no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0) CK(cudaGetDevice(&device));
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    n = prob.y.n;
    prow_off.assign(size_t(n) + 1, 0);
    for (int i = 0; i < n; ++i) {
      const PhaseMask m{prob.mask[size_t(i)]};
      prow_off[size_t(i) + 1] = prow_off[size_t(i)] + m.count();
      for (int ph = 0; ph < 3; ++ph)
        if (m.has(ph)) {
          prow_node.push_back(i);
          prow_phase.push_back(std::uint8_t(ph));
        }
    }
    nphi = prow_off[size_t(n)];
    d_prow_off.alloc(prow_off.size());
    CK(cudaMemcpy(d_prow_off.p, prow_off.data(), prow_off.size() * sizeof(int), cudaMemcpyHostToDevice));
    d_prow_node.alloc(prow_node.size());
    if (nphi > 0) {
      CK(cudaMemcpy(d_prow_node.p, prow_node.data(), prow_node.size() * sizeof(int), cudaMemcpyHostToDevice));
      d_prow_phase.alloc(prow_phase.size());
      CK(cudaMemcpy(d_prow_phase.p, prow_phase.data(), prow_phase.size(), cudaMemcpyHostToDevice));
    }
    d_mask.alloc(size_t(n));
    CK(cudaMemcpy(d_mask.p, prob.mask.data(), size_t(n), cudaMemcpyHostToDevice));
    d_yin.alloc(prob.y.row.size() * 9);
    if (!prob.y.row.empty())
      CK(cudaMemcpy(d_yin.p, prob.y.val.data(), prob.y.val.size() * sizeof(double), cudaMemcpyHostToDevice));
    pivot_floor = 1e-12 * std::max(prob.y.max_abs(), 1.0);
    if (prob.slack < 0) return;  // matrix-only engine (kron_reduce on a bare Y)
    std::vector<int> elim;
    for (int i = 0; i < n; ++i)
      if (i != prob.slack) elim.push_back(i);
    upload_elim(full, prob.y, prob.mask, elim);
    double sv[6];
    for (int q = 0; q < 3; ++q) {
      sv[2 * q] = prob.net.nodes[size_t(prob.slack)].slack_voltage[q].real();
      sv[2 * q + 1] = prob.net.nodes[size_t(prob.slack)].slack_voltage[q].imag();
    }
    d_slackv.alloc(3);
    CK(cudaMemcpy(d_slackv.p, sv, sizeof sv, cudaMemcpyHostToDevice));
    // the anchored factorization every solve of this engine uses (solver.cpp:168-179)
    factorize(full, d_yin.p, pivot_floor);
    d_v0.alloc(size_t(3) * n);
    d_v0p.alloc(size_t(std::max(nphi, 1)));
    d_cs.alloc(size_t(2 * n));
    d_cr.alloc(size_t(2 * n));
    d_sn.alloc(size_t(n));
    d_memoff.alloc(size_t(n) + 1);
    d_memlist.alloc(size_t(n));
    if (prob.L > 0) load_scenarios(prob.scenario_ids, prob.injections, prob.voltages);
  }

  // ScenarioLibrary on the device (load_library: V-hat = solve(I-hat) when
  // the voltages are not given, scenario.cpp:39-50).
  void load_scenarios(const std::vector<std::string>& ids, const std::vector<double>& inj,
                      const std::vector<double>& volt) {
    L = int(ids.size());
    prob.L = L;
    prob.scenario_ids = ids;
    prob.injections = inj;
    prob.voltages = volt;
    if (L == 0) return;
    d_inj.alloc(size_t(L) * 3 * n);
    CK(cudaMemcpy(d_inj.p, inj.data(), inj.size() * sizeof(double), cudaMemcpyHostToDevice));
    d_vhat.alloc(size_t(L) * 3 * n);
    if (!volt.empty()) {
      CK(cudaMemcpy(d_vhat.p, volt.data(), volt.size() * sizeof(double), cudaMemcpyHostToDevice));
      h_vhat = volt;
    } else {
      solve_full(full, d_slackv.p, d_inj.p, L, d_vhat.p);
      h_vhat.resize(size_t(L) * 6 * n);
      CK(cudaMemcpyAsync(h_vhat.data(), d_vhat.p, h_vhat.size() * sizeof(double), cudaMemcpyDeviceToHost,
                         stream));
      CK(cudaStreamSynchronize(stream));
      prob.voltages = h_vhat;
    }
    d_vhatp.alloc(size_t(nphi) * L);
    d_vmag.alloc(size_t(nphi) * L);
    d_vmin.alloc(size_t(nphi) * L);
    d_vmax.alloc(size_t(nphi) * L);
    d_iagg.alloc(size_t(n) * L * 3);
    d_base.alloc(size_t(nphi) * L);
    d_psmice.alloc(size_t(2 * n) * L);
    d_pmaxerr.alloc(size_t(2 * n) * L);
    d_best.alloc(size_t(2 + L));
    if (h_best) cudaFreeHost(h_best);
    CK(cudaMallocHost(&h_best, sizeof(double) * size_t(2 + L)));
  }

  ~Impl() {
    if (ev_a) {
      cudaEventDestroy(ev_a);
      cudaEventDestroy(ev_b);
      cudaEventDestroy(ev_run0);
      cudaEventDestroy(ev_run1);
    }
    if (h_best) cudaFreeHost(h_best);
    if (stream) cudaStreamDestroy(stream);
  }

  // ---- loop --------------------------------------------------------------
  void begin(const ReductionConfig& c) {
    if (!(c.e_bar >= 0)) throw ConfigError("e_bar must be non-negative");
    if (c.target_reduction && !(*c.target_reduction >= 0 && *c.target_reduction <= 1))
      throw ConfigError("target_reduction must lie in [0,1]");
    if (L == 0) throw ValidationError("scenario library is empty");
    cfg = c;
    // AnchoredSolver (re-factorized per run, as run_reduction does, reduce.cpp:359)
    factorize(full, d_yin.p, pivot_floor);
    solve_full(full, d_slackv.p, nullptr, 1, d_v0.p);
    {
      // v0 at present rows
      std::vector<double2> v0(size_t(3) * n);
      CK(cudaMemcpyAsync(v0.data(), d_v0.p, v0.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      std::vector<double2> v0p(static_cast<size_t>(nphi));
      for (int r = 0; r < nphi; ++r) v0p[size_t(r)] = v0[size_t(prow_node[size_t(r)]) * 3 + prow_phase[size_t(r)]];
      CK(cudaMemcpyAsync(d_v0p.p, v0p.data(), v0p.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
    }
    const int tot = std::max(nphi * L, n * L * 3);
    prep_kernel<<<(tot + 255) / 256, 256, 0, stream>>>(n, L, nphi, d_prow_node.p, d_prow_phase.p, d_vhat.p,
                                                       d_inj.p, d_vhatp.p, d_vmag.p, d_vmin.p, d_vmax.p,
                                                       d_iagg.p);
    launched();
    CK(cudaGetLastError());
    if (cfg.use_delta) build_z();
    refresh_base();
    hs.init(prob.net);
    loop_active = true;
  }

  bool target_reached() const {
    return cfg.target_reduction && hs.reduction_fraction() >= *cfg.target_reduction;
  }

  void upload_iteration(long long c0, long long c1) {
    const long long C = c1 - c0;
    if (C > 0) {
      CK(cudaMemcpyAsync(d_cs.p, cs.data() + c0, size_t(C) * sizeof(int), cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(d_cr.p, cr.data() + c0, size_t(C) * sizeof(int), cudaMemcpyHostToDevice, stream));
    }
    CK(cudaMemcpyAsync(d_sn.p, hs.supernodes.data(), hs.supernodes.size() * sizeof(int),
                       cudaMemcpyHostToDevice, stream));
    if (cfg.objective == Objective::complex_error) {
      std::vector<int> off(size_t(n) + 1, 0), lst;
      for (int i = 0; i < n; ++i) {
        for (int j : hs.members[size_t(i)]) lst.push_back(j);
        off[size_t(i) + 1] = int(lst.size());
      }
      CK(cudaMemcpy(d_memoff.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
      if (!lst.empty())
        CK(cudaMemcpy(d_memlist.p, lst.data(), lst.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
  }

  void launch_score(long long C) {
    if (C <= 0) return;
    ScoreDev a{};
    a.C = int(C);
    a.L = L;
    a.nphi = nphi;
    a.ns = int(hs.supernodes.size());
    a.cand_s = d_cs.p;
    a.cand_r = d_cr.p;
    a.sn = d_sn.p;
    a.prow_off = d_prow_off.p;
    a.mask = d_mask.p;
    a.Z = d_Z.p;
    a.base = d_base.p;
    a.vmin = d_vmin.p;
    a.vmax = d_vmax.p;
    a.iagg = d_iagg.p;
    a.objective = cfg.objective == Objective::complex_error ? KRG_OBJ_COMPLEX : KRG_OBJ_MAGNITUDE;
    a.mem_off = d_memoff.p;
    a.mem_list = d_memlist.p;
    a.vhatp = d_vhatp.p;
    a.out_smice = d_psmice.p;
    a.out_maxerr = d_pmaxerr.p;
    const long long pairs = C * L;
    if (profile) CK(cudaEventRecord(ev_a, stream));
    score_kernel<<<unsigned((pairs + 127) / 128), 128, 0, stream>>>(a);
    launched();
    CK(cudaGetLastError());
    if (profile) {
      CK(cudaEventRecord(ev_b, stream));
      CK(cudaEventSynchronize(ev_b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev_a, ev_b));
      double f, b;
      score_work(score_c0, score_c0 + C, f, b);
      score_stats.launches += 1;
      score_stats.ms += ms;
      score_stats.flops += f;
      score_stats.bytes += b;
    }
  }

  // score [c0,c1) and reduce to the local best; returns (smice, global idx) and max_err in h_best
  long long score_c0 = 0;
  void score_best(long long c0, long long c1) {
    const long long C = c1 - c0;
    score_c0 = c0;
    upload_iteration(c0, c1);
    launch_score(C);
    argmin_kernel<<<1, 1024, 0, stream>>>(int(std::max(C, 0LL)), L, cfg.e_bar, c0, d_psmice.p, d_pmaxerr.p,
                                          d_best.p);
    launched();
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_best, d_best.p, sizeof(double) * size_t(2 + L), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }

  long long best_index() const {
    long long idx;
    std::memcpy(&idx, &h_best[1], sizeof idx);
    return idx;
  }

  // multi-GPU min-loc over ranks (lexicographic (smice, idx))
  void exchange_best() {
    if (world <= 1 || xfn == nullptr) return;
    const size_t bytes = sizeof(double) * size_t(2 + L);
    std::vector<double> all(size_t(world) * size_t(2 + L));
    if (xfn(xuser, h_best, all.data(), bytes) != 0) throw Error("exchange callback failed");
    int bw = -1;
    double bs = 0;
    long long bi = -1;
    for (int w = 0; w < world; ++w) {
      const double* rec = all.data() + size_t(w) * size_t(2 + L);
      long long idx;
      std::memcpy(&idx, &rec[1], sizeof idx);
      if (idx < 0) continue;
      if (bi < 0 || rec[0] < bs || (rec[0] == bs && idx < bi)) {
        bs = rec[0];
        bi = idx;
        bw = w;
      }
    }
    if (bw >= 0)
      std::memcpy(h_best, all.data() + size_t(bw) * size_t(2 + L), bytes);
    else {
      const long long none = -1;
      std::memcpy(&h_best[1], &none, sizeof none);
    }
  }

  void commit_device(int s, int r) {
    const unsigned ms = prob.mask[size_t(s)], mr = prob.mask[size_t(r)];
    commit_kernel<<<(L + 127) / 128, 128, 0, stream>>>(s, r, L, ms, mr, prow_off[size_t(s)], prow_off[size_t(r)],
                                                       d_iagg.p, d_vmin.p, d_vmax.p);
    launched();
    CK(cudaGetLastError());
    if (cfg.use_delta) refresh_base();
  }
};

// ---------------------------------------------------------------------------

Engine::Engine(const Problem& prob, int device) : impl_(std::make_unique<Impl>(prob, device)) {}
Engine::~Engine() = default;

void Engine::set_profile(bool on) {
  impl_->ensure_events();
  impl_->profile = on;
  impl_->score_stats = KernelStats{};
  impl_->solve_stats = KernelStats{};
}
KernelStats Engine::stats(int which) const { return which == 0 ? impl_->score_stats : impl_->solve_stats; }
const Problem& Engine::problem() const { return impl_->prob; }
std::int64_t Engine::launches() const { return impl_->launches; }

void Engine::set_exchange(int rank, int world, krg_exchange_fn fn, void* user) {
  if (world < 1 || rank < 0 || rank >= world) throw ConfigError("bad rank/world");
  impl_->rank = rank;
  impl_->world = world;
  impl_->xfn = fn;
  impl_->xuser = user;
}

void Engine::scenario_voltages(double* out) {
  std::memcpy(out, impl_->h_vhat.data(), impl_->h_vhat.size() * sizeof(double));
}

void Engine::solve(const double* inj, int nrhs, double* out) {
  Impl& I = *impl_;
  DBuf<double2> rhs, res;
  rhs.alloc(size_t(nrhs) * 3 * I.n);
  res.alloc(size_t(nrhs) * 3 * I.n);
  CK(cudaMemcpyAsync(rhs.p, inj, size_t(nrhs) * 3 * I.n * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
  I.solve_full(I.full, I.d_slackv.p, rhs.p, nrhs, res.p);
  CK(cudaMemcpyAsync(out, res.p, size_t(nrhs) * 3 * I.n * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::loop_begin(const ReductionConfig& cfg) { impl_->begin(cfg); }

void Engine::set_scenarios(const std::vector<std::string>& ids, const std::vector<double>& inj,
                           const std::vector<double>& volt) {
  impl_->load_scenarios(ids, inj, volt);
}

void Engine::pq_to_currents(const std::vector<std::vector<std::pair<int, cx>>>& loads, std::vector<double>& inj,
                            std::vector<double>& volt) {
  // scenario_from_pq (scenario.cpp:52-98): I = -conj(S/V) fixed point, one
  // device anchored solve per sweep, all scenarios batched; each scenario
  // stops at its own convergence like the reference's per-scenario loop.
  Impl& I = *impl_;
  const int n = I.n;
  const int L = int(loads.size());
  const size_t dim = size_t(3 * n);
  std::vector<cx> v0(dim);
  {
    DBuf<double2> out;
    out.alloc(dim);
    I.solve_full(I.full, I.d_slackv.p, nullptr, 1, out.p);
    CK(cudaMemcpyAsync(v0.data(), out.p, dim * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaStreamSynchronize(I.stream));
  }
  const std::vector<cx> zeros(dim);
  std::vector<std::vector<cx>> S(static_cast<size_t>(L), zeros), V(static_cast<size_t>(L), v0), J(static_cast<size_t>(L), zeros);
  for (int l = 0; l < L; ++l)
    for (const auto& ld : loads[size_t(l)]) S[size_t(l)][size_t(ld.first)] += ld.second;
  std::vector<char> done(size_t(L), 0);
  std::vector<double> last_dv(size_t(L), 0.0);
  DBuf<double2> d_rhs, d_out;
  d_rhs.alloc(dim * size_t(std::max(L, 1)));
  d_out.alloc(dim * size_t(std::max(L, 1)));
  std::vector<cx> rhs(dim * size_t(L)), res(dim * size_t(L));
  for (int it = 0; it < 50; ++it) {
    std::vector<int> act;
    for (int l = 0; l < L; ++l)
      if (!done[size_t(l)]) act.push_back(l);
    if (act.empty()) break;
    for (size_t a = 0; a < act.size(); ++a) {
      const int l = act[a];
      for (size_t k = 0; k < dim; ++k) {
        const cx sk = S[size_t(l)][k];
        if (sk == cx{}) continue;
        if (std::abs(V[size_t(l)][k]) < 1e-6)
          throw SolverError("scenario '" + I.prob.scenario_ids[size_t(l)] + "': voltage collapse during PQ conversion");
        J[size_t(l)][k] = -std::conj(sk / V[size_t(l)][k]);
      }
      std::copy(J[size_t(l)].begin(), J[size_t(l)].end(), rhs.begin() + long(a * dim));
    }
    CK(cudaMemcpyAsync(d_rhs.p, rhs.data(), act.size() * dim * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
    I.solve_full(I.full, I.d_slackv.p, d_rhs.p, int(act.size()), d_out.p);
    CK(cudaMemcpyAsync(res.data(), d_out.p, act.size() * dim * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaStreamSynchronize(I.stream));
    for (size_t a = 0; a < act.size(); ++a) {
      const int l = act[a];
      double dv = 0;
      for (size_t k = 0; k < dim; ++k) dv = std::max(dv, std::abs(res[a * dim + k] - V[size_t(l)][k]));
      std::copy(res.begin() + long(a * dim), res.begin() + long((a + 1) * dim), V[size_t(l)].begin());
      last_dv[size_t(l)] = dv;
      if (dv < 1e-9) done[size_t(l)] = 1;
    }
  }
  for (int l = 0; l < L; ++l)
    if (!done[size_t(l)])
      throw SolverError("scenario '" + I.prob.scenario_ids[size_t(l)] +
                        "': PQ fixed point did not converge in 50 iterations");
  inj.assign(dim * 2 * size_t(L), 0.0);
  volt.assign(dim * 2 * size_t(L), 0.0);
  for (int l = 0; l < L; ++l)
    for (size_t k = 0; k < dim; ++k) {
      inj[(size_t(l) * dim + k) * 2] = J[size_t(l)][k].real();
      inj[(size_t(l) * dim + k) * 2 + 1] = J[size_t(l)][k].imag();
      volt[(size_t(l) * dim + k) * 2] = V[size_t(l)][k].real();
      volt[(size_t(l) * dim + k) * 2 + 1] = V[size_t(l)][k].imag();
    }
}

std::int64_t Engine::loop_candidates(std::vector<int>& cs, std::vector<int>& cr) {
  Impl& I = *impl_;
  if (!I.loop_active) throw Error("loop not started");
  I.hs.enumerate(I.cs, I.cr);
  cs = I.cs;
  cr = I.cr;
  return std::int64_t(I.cs.size());
}

void Engine::loop_score_all(double* smice, std::uint8_t* feasible, double* max_err) {
  Impl& I = *impl_;
  const long long C = (long long)I.cs.size();
  I.upload_iteration(0, C);
  I.launch_score(C);
  std::vector<double> ps(size_t(C) * I.L), pm(size_t(C) * I.L);
  if (C > 0) {
    CK(cudaMemcpyAsync(ps.data(), I.d_psmice.p, ps.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaMemcpyAsync(pm.data(), I.d_pmaxerr.p, pm.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  }
  CK(cudaStreamSynchronize(I.stream));
  for (long long c = 0; c < C; ++c) {
    bool feas = true;
    double sum = 0;
    for (int l = 0; l < I.L; ++l) {
      feas = feas && !(pm[size_t(c) * I.L + l] > I.cfg.e_bar);
      sum += ps[size_t(c) * I.L + l];
      if (max_err) max_err[size_t(c) * I.L + l] = pm[size_t(c) * I.L + l];
    }
    feasible[c] = feas ? 1 : 0;
    smice[c] = feas ? sum : std::numeric_limits<double>::infinity();
  }
}

void Engine::loop_best(krg_best* out, double* max_err) {
  Impl& I = *impl_;
  int64_t c0 = 0, c1 = (int64_t)I.cs.size();
  if (I.world > 1) krg_shard_range(c1, I.rank, I.world, &c0, &c1);
  I.score_best(c0, c1);
  I.exchange_best();
  const long long idx = I.best_index();
  out->index = idx;
  out->smice = idx < 0 ? std::numeric_limits<double>::infinity() : I.h_best[0];
  out->s = idx < 0 ? -1 : I.cs[size_t(idx)];
  out->r = idx < 0 ? -1 : I.cr[size_t(idx)];
  if (max_err) std::memcpy(max_err, I.h_best + 2, sizeof(double) * size_t(I.L));
}

void Engine::loop_commit(int s, int r) {
  Impl& I = *impl_;
  I.hs.commit(s, r);
  I.commit_device(s, r);
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::loop_base(double* out) {
  Impl& I = *impl_;
  std::vector<double2> b(size_t(I.nphi) * I.L);
  CK(cudaMemcpyAsync(b.data(), I.d_base.p, b.size() * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::memset(out, 0, sizeof(double) * size_t(I.L) * 6 * I.n);
  for (int r = 0; r < I.nphi; ++r)
    for (int l = 0; l < I.L; ++l) {
      const size_t o = (size_t(l) * 3 * I.n + size_t(I.prow_node[size_t(r)]) * 3 + I.prow_phase[size_t(r)]) * 2;
      out[o] = b[size_t(r) * I.L + l].x;
      out[o + 1] = b[size_t(r) * I.L + l].y;
    }
}

void Engine::zcols(double* out, std::int64_t cap) {
  Impl& I = *impl_;
  const size_t need = size_t(I.nphi) * I.nphi * 2;
  if (size_t(cap) < need) throw ValidationError("zcols: buffer too small");
  if (!I.d_Z.p) I.build_z();
  CK(cudaMemcpyAsync(out, I.d_Z.p, need * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void Engine::run(const ReductionConfig& cfg, const Observer& obs, ResultData& out) {
  Impl& I = *impl_;
  out = ResultData{};
  out.L = I.L;
  I.ensure_events();
  CK(cudaEventRecord(I.ev_run0, I.stream));
  I.begin(cfg);
  int iteration = 0;
  while (!I.target_reached()) {
    const auto t0 = std::chrono::steady_clock::now();
    I.hs.enumerate(I.cs, I.cr);
    const long long C = (long long)I.cs.size();
    if (C == 0) break;
    int64_t c0 = 0, c1 = C;
    if (I.world > 1) krg_shard_range(C, I.rank, I.world, &c0, &c1);
    I.score_best(c0, c1);
    I.exchange_best();
    const long long best = I.best_index();
    if (best < 0) break;
    const int s = I.cs[size_t(best)], r = I.cr[size_t(best)];
    I.commit_device(s, r);
    I.hs.commit(s, r);
    TraceRow row;
    row.iteration = ++iteration;
    row.s = s;
    row.r = r;
    row.smice = I.h_best[0];
    row.max_err.assign(I.h_best + 2, I.h_best + 2 + I.L);
    row.supernode_count = int(I.hs.supernodes.size());
    row.candidate_count = int(C);
    row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    out.total_candidates += C;
    if (obs) obs(I.hs, row);
    out.trace.push_back(std::move(row));
  }
  CK(cudaStreamSynchronize(I.stream));
  I.loop_active = false;
  // final Kron reduction over the surviving super-nodes (reduce.cpp:426-450)
  Partition part;
  part.keep = I.hs.supernodes;
  for (int i = 0; i < I.n; ++i)
    if (I.hs.sup[size_t(i)] != i) part.reduce.push_back(i);
  check_partition(part, I.n, I.prob.slack);
  ReducedModel& model = out.model;
  kron(part.reduce, model);
  for (int i : I.hs.supernodes) {
    std::vector<int> mem = I.hs.members[size_t(i)];
    std::sort(mem.begin(), mem.end());
    model.clusters[i] = std::move(mem);
  }
  model.e_bar = cfg.e_bar;
  model.objective = cfg.objective;
  model.scenario_ids = I.prob.scenario_ids;
  model.final_max_err = model_errors(model);
  out.state = I.hs;
  CK(cudaEventRecord(I.ev_run1, I.stream));
  CK(cudaEventSynchronize(I.ev_run1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, I.ev_run0, I.ev_run1));
  out.device_ms = ms;
  I.last_run_ms = ms;
}

void Engine::kron(const std::vector<int>& reduce, ReducedModel& model) {
  Impl& I = *impl_;
  DevElim e;
  I.upload_elim(e, I.prob.y, I.prob.mask, reduce);
  I.factorize(e, I.d_yin.p, 1e-12 * std::max(I.prob.y.max_abs(), 1.0));
  const ElimSchedule& h = e.h;
  std::vector<double2> blocks(size_t(h.nblocks) * 9);
  CK(cudaMemcpyAsync(blocks.data(), e.blocks.p, blocks.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                     I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::vector<int> pos(size_t(I.n), -1);
  for (size_t p = 0; p < h.kept.size(); ++p) pos[size_t(h.kept[p])] = int(p);
  model.kept_ids = h.kept;
  model.kept_phases.clear();
  for (int id : h.kept) model.kept_phases.push_back(PhaseMask{I.prob.mask[size_t(id)]});
  model.y_kron = BlockMatrix(int(h.kept.size()));
  for (size_t q = 0; q < h.rem_i.size(); ++q) {
    Mat3c m;
    const int b = h.rem_blk[q];
    for (int k = 0; k < 9; ++k) {
      const double2 v = b >= 0 ? blocks[size_t(b) * 9 + k] : make_double2(0.0, 0.0);
      m.m[size_t(k)] = cx{v.x, v.y};
    }
    if (m.is_zero()) continue;
    model.y_kron.block(pos[size_t(h.rem_i[q])], pos[size_t(h.rem_j[q])]) = m;
  }
}

std::vector<double> Engine::model_errors(const ReducedModel& model) {
  // model_max_errors (reduce.cpp:490-550): anchored solve on Y_kron with
  // cluster-aggregated injections; |.| via std::abs on the host read-back.
  Impl& I = *impl_;
  const Network& net = I.prob.net;
  const int slack = I.prob.slack;
  auto pos_of = [&](int id) {
    auto it = std::lower_bound(model.kept_ids.begin(), model.kept_ids.end(), id);
    if (it == model.kept_ids.end() || *it != id)
      throw ValidationError("reduced model does not keep node " + std::to_string(id));
    return int(it - model.kept_ids.begin());
  };
  const int slack_pos = pos_of(slack);
  const int nk = int(model.kept_ids.size());
  std::vector<int> assigned(size_t(net.size()), -1);
  for (const auto& [i, mem] : model.clusters) {
    const int pi = pos_of(i);
    for (int j : mem) {
      if (j < 0 || j >= net.size()) throw ValidationError("cluster references unknown node");
      assigned[size_t(j)] = pi;
    }
  }
  for (int p = 0; p < nk; ++p) assigned[size_t(model.kept_ids[size_t(p)])] = p;
  for (int j = 0; j < net.size(); ++j)
    if (assigned[size_t(j)] < 0)
      throw ValidationError("node " + std::to_string(j) + " is not covered by any cluster");

  const FlatBlocks yk = FlatBlocks::from(model.y_kron);
  std::vector<std::uint8_t> kmask(static_cast<size_t>(nk));
  for (int p = 0; p < nk; ++p) kmask[size_t(p)] = model.kept_phases[size_t(p)].bits;
  DevElim e;
  std::vector<int> elim;
  for (int p = 0; p < nk; ++p)
    if (p != slack_pos) elim.push_back(p);
  I.upload_elim(e, yk, kmask, elim);
  DBuf<double2> yin;
  yin.alloc(yk.row.size() * 9);
  if (!yk.row.empty())
    CK(cudaMemcpyAsync(yin.p, yk.val.data(), yk.val.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
  I.factorize(e, yin.p, 1e-12 * std::max(yk.max_abs(), 1.0));

  const int L = I.L;
  const int n = net.size();
  std::vector<double> rhs(size_t(L) * 6 * nk, 0.0);
  for (int l = 0; l < L; ++l) {
    std::vector<cx> ik(size_t(3 * nk), cx{});
    const double* inj = I.prob.injections.data() + size_t(l) * 6 * n;
    for (const auto& [i, mem] : model.clusters) {
      const int pi = pos_of(i);
      for (int j : mem)
        for (int p = 0; p < 3; ++p) ik[size_t(3 * pi + p)] += cx{inj[(3 * j + p) * 2], inj[(3 * j + p) * 2 + 1]};
    }
    for (int t = 0; t < 3 * nk; ++t) {
      rhs[size_t(l) * 6 * nk + size_t(t) * 2] = ik[size_t(t)].real();
      rhs[size_t(l) * 6 * nk + size_t(t) * 2 + 1] = ik[size_t(t)].imag();
    }
  }
  DBuf<double2> d_rhs, d_out, d_kv;
  d_rhs.alloc(size_t(L) * 3 * nk);
  d_out.alloc(size_t(L) * 3 * nk);
  CK(cudaMemcpyAsync(d_rhs.p, rhs.data(), rhs.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
  I.solve_full(e, I.d_slackv.p, d_rhs.p, L, d_out.p);
  std::vector<double> vk(size_t(L) * 6 * nk);
  CK(cudaMemcpyAsync(vk.data(), d_out.p, vk.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  std::vector<double> out;
  for (int l = 0; l < L; ++l) {
    double err = 0;
    for (int j = 0; j < n; ++j) {
      const int pj = assigned[size_t(j)];
      for (int p = 0; p < 3; ++p) {
        if (!I.prob.net.nodes[size_t(j)].phases.has(p)) continue;
        const double* a = &vk[size_t(l) * 6 * nk + size_t(3 * pj + p) * 2];
        const double* b = &I.h_vhat[size_t(l) * 6 * n + size_t(3 * j + p) * 2];
        const double e2 = std::fabs(std::abs(cx{a[0], a[1]}) - std::abs(cx{b[0], b[1]}));
        err = std::max(err, e2);
      }
    }
    out.push_back(err);
  }
  return out;
}

void Engine::radialize(ReducedModel& model, bool with_errors) {
  auto kr = [this](const std::vector<int>& reduce, ReducedModel& m) { this->kron(reduce, m); };
  std::function<std::vector<double>(const ReducedModel&)> errs = [this](const ReducedModel& m) {
    return this->model_errors(m);
  };
  model = radialize_host(model, impl_->prob.net, kr, with_errors ? &errs : nullptr);
}

// measured unfused FP64 rate (GFLOP/s, DMUL+DADD counted as 2) on `device`
extern "C" int krg_fp64_probe(int32_t device, double* gflops) {
  try {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw CudaError("no CUDA device");
    if (device >= 0) CK(cudaSetDevice(device));
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<double> sink;
    sink.alloc(1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    fp64_probe_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, sink.p);  // warm-up
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      fp64_probe_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, sink.p);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::max(best, 2.0 * 8.0 * iters * double(blocks) * threads / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *gflops = best;
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

// self test hook for the __divdc3 replica (device)
extern "C" int krg_selftest_cdiv(const double* in, int32_t N, double* out, int32_t on_device) {
  try {
    if (!on_device) {
      for (int i = 0; i < N; ++i) {
        const C2 r = dev::cdiv({in[4 * i], in[4 * i + 1]}, {in[4 * i + 2], in[4 * i + 3]});
        out[2 * i] = r.x;
        out[2 * i + 1] = r.y;
      }
      return KRG_OK;
    }
    DBuf<double> din, dout;
    din.alloc(size_t(N) * 4);
    dout.alloc(size_t(N) * 2);
    CK(cudaMemcpy(din.p, in, size_t(N) * 4 * sizeof(double), cudaMemcpyHostToDevice));
    selftest_cdiv_kernel<<<(N + 127) / 128, 128>>>(N, din.p, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout.p, size_t(N) * 2 * sizeof(double), cudaMemcpyDeviceToHost));
    return KRG_OK;
  } catch (...) {
    return status_from_current_exception();
  }
}

}  // namespace kronred::b200
