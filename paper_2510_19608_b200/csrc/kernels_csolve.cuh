// K1s (compact): anchored forward/backward sweeps on the present-phase
// compacted factor, one right-hand side per CTA, the solution vector and —
// when it fits — the whole factor and its level program staged in shared
// memory, so a level costs shared-memory latency plus one __syncthreads.
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

// offsets into the packed int program
struct CProg {
  int st_x, st_m, st_mask, st_node, st_pinv;
  int in_off, in_x, in_m, in_blk;
  int cp_off, cp_x, cp_m, cp_blk;
  int fw_off, fw, bw_off, bw;
  int kept_x, kept_m, kept_i;
  int nsteps, nfw, nbw, nkept, nmeta, ncf, nphi;
};

struct CSolveArgs {
  CProg P;
  const int* meta_g;
  const double2* cfac_g;
  const double2* kept_val;  // [nkept][3] (present phases in order)
  int smem_factor;          // stage cfac+meta in shared memory
  // sources / sinks
  int n;                    // nodes (MODE_FULL scatter)
  const int* prow_off;      // [n+1]
  const std::uint8_t* mask; // [n]
  const double2* rhs_full;  // [nrhs][3n] or null
  double2* out_full;        // [nrhs][3n]
  const double2* iagg;      // [n][L][3]
  double2* base;            // bv: [nphi][L][2], base in slot 0
  int L;
  int col0;
  const double2* v0p;
  double2* zout;            // [ncol][nphi]
};

__device__ __forceinline__ int popc_below(unsigned m, int p) { return __popc(m & ((1u << p) - 1u)); }

template <int MODE>
__global__ void __launch_bounds__(256) csolve_kernel(CSolveArgs a) {
  extern __shared__ double2 smem[];
  const CProg& P = a.P;
  double2* x = smem;                                   // [nphi]
  const double2* cf = a.cfac_g;
  const int* M = a.meta_g;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int rhs = blockIdx.x;
  if (a.smem_factor) {
    double2* scf = smem + P.nphi;
    int* smeta = reinterpret_cast<int*>(scf + P.ncf);
    for (int i = tid; i < P.ncf; i += nt) scf[i] = a.cfac_g[i];
    for (int i = tid; i < P.nmeta; i += nt) smeta[i] = a.meta_g[i];
    cf = scf;
    M = smeta;
    __syncthreads();
  }
  // boundary (kept) values
  for (int k = tid; k < P.nkept; k += nt) {
    const int x0 = M[P.kept_x + k], m = M[P.kept_m + k], ki = M[P.kept_i + k];
    for (int i = 0; i < m; ++i) x[x0 + i] = a.kept_val[ki * 3 + i];
  }
  __syncthreads();
  // forward: rhs_k = b_k - sum_j A_kj t_j in elimination order; t_k = pinv_k rhs_k
  for (int lev = 0; lev < P.nfw; ++lev) {
    const int o0 = M[P.fw_off + lev], o1 = M[P.fw_off + lev + 1];
    for (int idx = o0 + tid; idx < o1; idx += nt) {
      const int st = M[P.fw + idx];
      const int xk = M[P.st_x + st], mk = M[P.st_m + st];
      const unsigned msk = unsigned(M[P.st_mask + st]);
      const int node = M[P.st_node + st];
      C2 b[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        if (!((msk >> p) & 1u)) continue;
        const int i = popc_below(msk, p);
        C2 v;
        if (MODE == CM_BASE) {
          v = ld2(a.iagg + (size_t(node) * a.L + rhs) * 3 + p);
        } else if (MODE == CM_ZCOL) {
          v = (xk + i == a.col0 + rhs) ? C2{1.0, 0.0} : C2{0.0, 0.0};
        } else {
          v = a.rhs_full ? ld2(a.rhs_full + size_t(rhs) * 3 * a.n + size_t(node) * 3 + p) : C2{0.0, 0.0};
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if (j == i) b[j] = v;
      }
      for (int e = M[P.in_off + st]; e < M[P.in_off + st + 1]; ++e) {
        const int xj = M[P.in_x + e], mj = M[P.in_m + e], bo = M[P.in_blk + e];
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
      const int po = M[P.st_pinv + st];
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
      const int st = M[P.bw + idx];
      const int xk = M[P.st_x + st], mk = M[P.st_m + st];
      C2 acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int e = M[P.cp_off + st]; e < M[P.cp_off + st + 1]; ++e) {
        const int xj = M[P.cp_x + e], mj = M[P.cp_m + e], bo = M[P.cp_blk + e];
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
      const int po = M[P.st_pinv + st];
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
    for (int r = tid; r < P.nphi; r += nt) a.base[(size_t(r) * a.L + rhs) * 2] = x[r];
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
