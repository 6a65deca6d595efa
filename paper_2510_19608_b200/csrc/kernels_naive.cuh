// use_delta = false: the reference's full-solve candidate evaluation
// (eval_full_solve, reduce.cpp:132-167). Per (candidate, scenario) pair:
//
//   ic = i_agg[l]; ic[3s+p] += ic[3r+p]; ic[3r+p] = 0          reduce.cpp:147-151
//   Vc = AnchoredSolver::solve(ic)                              reduce.cpp:152 (full sweep)
//   |Vc| = sqrt(re^2 + im^2)                                    reduce.cpp:157
//   score_scenario with the cluster members                     reduce.cpp:89-123
//
// One warp per pair, pairs strided over the grid. The solve is the base
// refresh's lane-slot program (forward and backward sweeps on the factor and
// program staged once per CTA by TMA), so its bits are the reference's. The
// scoring walks the super-nodes and their members like the reference: lanes
// take super-nodes and compute each one's cluster maximum (magnitude or
// complex objective) and the running max_err; lane 0 then adds the cluster
// maxima in super-node order. Per-pair SMICE and max_err go to [L][ldc]; the
// argmin kernel sums scenarios in order and applies feasibility.
#pragma once

namespace kronred::b200 {
namespace {

struct NaiveArgs {
  BaseArgs b;                // program + factor (cf, meta, offsets), W, L, nphi, iaggp, kept_val
  int C;                     // candidates (lexicographic)
  const int* cs;             // [C] candidate s
  const int* cr;             // [C] candidate r
  int ns;                    // active super-nodes
  const int* sn_id;          // [ns] ascending
  const int* mem_off;        // [n+1] member CSR (by super-node id)
  const int* mem_list;
  const std::uint8_t* mask;  // [n]
  const int* prow_off;       // [n+1]
  const double2* vhat_full;  // [L][3n] scenario voltages
  int n;
  double e_bar;
  int complex_obj;
  double* out_sm;            // [L][ldc]
  double* out_mx;            // [L][ldc]
  int ldc;
};

__global__ void __launch_bounds__(256) naive_score_kernel(NaiveArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ unsigned long long bar;
  const BaseArgs& B = a.b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* cf = smem;
  int* M = reinterpret_cast<int*>(cf + B.ncf);
  double2* xall = reinterpret_cast<double2*>(M + B.nmeta);
  double* cmax_all = reinterpret_cast<double*>(xall + size_t(B.W) * B.nphi);  // [W][ns]
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, unsigned(B.ncf) * 16u + unsigned(B.nmeta) * 4u);
    if (B.ncf) bulk_g2s(cf, B.cfac, unsigned(B.ncf) * 16u, &bar);
    bulk_g2s(M, B.meta, unsigned(B.nmeta) * 4u, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  double2* x = xall + size_t(warp) * B.nphi;
  double* cmax = cmax_all + size_t(warp) * a.ns;
  const unsigned xs = unsigned(__cvta_generic_to_shared(x)), cs = unsigned(__cvta_generic_to_shared(cf));
  const int L = B.L;
  const long long pairs = (long long)a.C * L;
  for (long long p = (long long)blockIdx.x * B.W + warp; p < pairs; p += (long long)gridDim.x * B.W) {
    const int c = int(p / L), l = int(p - (long long)c * L);
    const int s = a.cs[c], r = a.cr[c];
    // ic = i_agg[l] with r's injection moved onto s (complex adds, reduce.cpp:149-150)
    for (int q = lane; q < B.nphi; q += 32) x[q] = B.iaggp[size_t(l) * B.nphi + q];
    __syncwarp();
    if (lane == 0) {
      const unsigned ms = a.mask[s], mr = a.mask[r];
      for (int ph = 0; ph < 3; ++ph) {
        if (!((mr >> ph) & 1u)) continue;  // phi(r) is a subset of phi(s)
        const int qs = a.prow_off[s] + popc_below(ms, ph), qr = a.prow_off[r] + popc_below(mr, ph);
        st2(x + qs, dev::cadd(ld2(x + qs), ld2(x + qr)));
        x[qr] = make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
    for (int k = lane; k < B.nkept; k += 32) {  // the slack is pinned (solver.cpp:181-186)
      const int xe = M[B.kept + 2 * k], ki = M[B.kept + 2 * k + 1];
      const int x0 = xe & 0xffffff, m = xe >> 24;
      for (int i = 0; i < m; ++i) x[x0 + i] = B.kept_val[ki * 3 + i];
    }
    __syncwarp();
    asm volatile("" ::: "memory");
    tree_forward<true>(B, M, xs, cs, x, cf, lane);
    __syncwarp();
    tree_backward<true>(B, M, xs, cs, x, cf, lane);
    __syncwarp();
    asm volatile("" ::: "memory");
    // score_scenario (reduce.cpp:89-123): per super-node i != r, the cluster
    // maximum over its members (and r's members when i == s) of the objective
    // entry; max_err over every magnitude error. Lanes take super-nodes.
    double mx = 0.0;
    for (int k = lane; k < a.ns; k += 32) {
      const int i = a.sn_id[k];
      double cm = 0.0;
      if (i != r) {
        const unsigned mi = a.mask[i];
        for (int pass = 0; pass < 2; ++pass) {
          const int cl = pass == 0 ? i : r;
          if (pass == 1 && i != s) break;
          for (int e = a.mem_off[cl]; e < a.mem_off[cl + 1]; ++e) {
            const int j = a.mem_list[e];
            const unsigned mj = a.mask[j];
            for (int ph = 0; ph < 3; ++ph) {
              if (!((mj >> ph) & 1u)) continue;
              const C2 v = ld2(x + a.prow_off[i] + popc_below(mi, ph));  // Vc at 3i+p
              const double m = dev::dsqrt(dev::dadd(dev::dmul(v.x, v.x), dev::dmul(v.y, v.y)));
              const C2 h = ld2(a.vhat_full + size_t(l) * 3 * a.n + size_t(3 * j + ph));  // V-hat at 3j+p
              const double hm = dev::dsqrt(dev::dadd(dev::dmul(h.x, h.x), dev::dmul(h.y, h.y)));
              const double em = fabs(dev::dsub(m, hm));
              if (em > mx) mx = em;
              double eo = em;
              if (a.complex_obj) {
                const double dr = dev::dsub(v.x, h.x), di = dev::dsub(v.y, h.y);
                eo = dev::dsqrt(dev::dadd(dev::dmul(dr, dr), dev::dmul(di, di)));
              }
              if (eo > cm) cm = eo;
            }
          }
        }
      }
      cmax[k] = cm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, mx, o);
      if (om > mx) mx = om;
    }
    __syncwarp();
    if (lane == 0) {
      double smice = 0.0;
      for (int k = 0; k < a.ns; ++k)  // super-node order; r contributes nothing (reduce.cpp:111)
        if (a.sn_id[k] != r) smice = dev::dadd(smice, cmax[k]);
      a.out_sm[size_t(l) * a.ldc + c] = smice;
      a.out_mx[size_t(l) * a.ldc + c] = mx;
    }
    __syncwarp();
  }
}

// The same evaluation for networks whose factor program does not fit in
// shared memory: the program and factor are read from global memory (L2
// evict-last, as base_refresh_kernel<false>), one pair per CTA of B.WB warps
// (the backward sweep's rounds span WB warps, as the program was laid out),
// the solution vector and the cluster maxima in shared memory.
__global__ void __launch_bounds__(256) naive_score_global_kernel(NaiveArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ double red[8];
  const BaseArgs& B = a.b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  double2* x = smem;
  double* cmax = reinterpret_cast<double*>(x + B.nphi);  // [ns]
  const double2* cf = B.cfac;
  const int* M = B.meta;
  const unsigned xs = unsigned(__cvta_generic_to_shared(x));
  const int L = B.L;
  const long long pairs = (long long)a.C * L;
  for (long long p = blockIdx.x; p < pairs; p += gridDim.x) {
    const int c = int(p / L), l = int(p - (long long)c * L);
    const int s = a.cs[c], r = a.cr[c];
    for (int q = tid; q < B.nphi; q += nt) x[q] = B.iaggp[size_t(l) * B.nphi + q];
    __syncthreads();
    if (tid == 0) {  // r's injection moved onto s (reduce.cpp:149-150)
      const unsigned ms = a.mask[s], mr = a.mask[r];
      for (int ph = 0; ph < 3; ++ph) {
        if (!((mr >> ph) & 1u)) continue;
        const int qs = a.prow_off[s] + popc_below(ms, ph), qr = a.prow_off[r] + popc_below(mr, ph);
        st2(x + qs, dev::cadd(ld2(x + qs), ld2(x + qr)));
        x[qr] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    for (int k = tid; k < B.nkept; k += nt) {
      const int xe = M[B.kept + 2 * k], ki = M[B.kept + 2 * k + 1];
      const int x0 = xe & 0xffffff, m = xe >> 24;
      for (int i = 0; i < m; ++i) x[x0 + i] = B.kept_val[ki * 3 + i];
    }
    __syncthreads();
    asm volatile("" ::: "memory");
    if (warp == 0) tree_forward<false>(B, M, xs, 0u, x, cf, lane);
    __syncthreads();
    tree_backward<false>(B, M, xs, 0u, x, cf, lane, B.WB, warp);
    __syncthreads();
    asm volatile("" ::: "memory");
    double mx = 0.0;
    for (int k = tid; k < a.ns; k += nt) {
      const int i = a.sn_id[k];
      double cm = 0.0;
      if (i != r) {
        const unsigned mi = a.mask[i];
        for (int pass = 0; pass < 2; ++pass) {
          const int cl = pass == 0 ? i : r;
          if (pass == 1 && i != s) break;
          for (int e = a.mem_off[cl]; e < a.mem_off[cl + 1]; ++e) {
            const int j = a.mem_list[e];
            const unsigned mj = a.mask[j];
            for (int ph = 0; ph < 3; ++ph) {
              if (!((mj >> ph) & 1u)) continue;
              const C2 v = ld2(x + a.prow_off[i] + popc_below(mi, ph));
              const double m = dev::dsqrt(dev::dadd(dev::dmul(v.x, v.x), dev::dmul(v.y, v.y)));
              const C2 h = ld2(a.vhat_full + size_t(l) * 3 * a.n + size_t(3 * j + ph));
              const double hm = dev::dsqrt(dev::dadd(dev::dmul(h.x, h.x), dev::dmul(h.y, h.y)));
              const double em = fabs(dev::dsub(m, hm));
              if (em > mx) mx = em;
              double eo = em;
              if (a.complex_obj) {
                const double dr = dev::dsub(v.x, h.x), di = dev::dsub(v.y, h.y);
                eo = dev::dsqrt(dev::dadd(dev::dmul(dr, dr), dev::dmul(di, di)));
              }
              if (eo > cm) cm = eo;
            }
          }
        }
      }
      cmax[k] = cm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, mx, o);
      if (om > mx) mx = om;
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nt / 32; ++w)
        if (red[w] > mx) mx = red[w];
      double smice = 0.0;
      for (int k = 0; k < a.ns; ++k)  // super-node order; r contributes nothing (reduce.cpp:111)
        if (a.sn_id[k] != r) smice = dev::dadd(smice, cmax[k]);
      a.out_sm[size_t(l) * a.ldc + c] = smice;
      a.out_mx[size_t(l) * a.ldc + c] = mx;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace kronred::b200
