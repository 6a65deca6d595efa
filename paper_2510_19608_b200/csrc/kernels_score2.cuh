// score2: the production magnitude-objective scorer (reduce.cpp:89-123,
// 194-244), one thread per (candidate, scenario) pair.
//
// A CTA owns G candidates x L scenarios (P = G*L threads) and walks the
// iteration's row table in tiles of K2 = 16 rows (four 4-row blocks; a block
// never splits a super-node). Tiles go through a three-slot shared-memory ring
// with ONE barrier per tile:
//
//   iteration j:  wait for tile j+1's cp.async group -> __syncthreads ->
//                 issue tile j+2 into the slot tile j-1 used ->
//                 form D = Zs - Zr of tile j+1 in place (once per candidate,
//                 not per scenario) -> compute tile j (its D was formed in
//                 iteration j-1 and is visible after this iteration's barrier).
//
// Shared layouts put the per-thread operands at compile-time offsets:
// D as [candidate][phase][row] (base, bounds as [row][l]), so the inner
// loop has no address arithmetic. Per 4-row block the common case (four
// single-row super-nodes, none of them the candidate's s or r, no padding) runs
// a straight-line body: Vc, |Vc| (branch-free correctly rounded sqrt),
// em = max(m - min_j v_j, max_j v_j - m) (exact cluster maximum), the ordered
// SMICE sum and the running max_err. Blocks holding s or r rows, padding or
// multi-row super-nodes take the general per-row path; a block whose |Vc|^2
// leaves the fast sqrt range is recomputed with __dsqrt_rn.
#pragma once

namespace kronred::b200 {
namespace {

constexpr int K2 = 16;  // rows per tile

struct Score2Layout {
  int L, G, NLmax;
  __host__ __device__ size_t tab_e() const { return (K2 * 4 + 15) / 16; }           // double2 units
  __host__ __device__ size_t bv_e() const { return size_t(L) * K2 * 2; }
  __host__ __device__ size_t z_e() const { return size_t(G) * NLmax * 2 * K2; }     // Zs and Zr staging
  __host__ __device__ size_t buf_e() const { return tab_e() + bv_e() + z_e(); }
  __host__ __device__ size_t smem_bytes(int P) const {
    const size_t ring = 3 * buf_e() * sizeof(double2) + size_t(G) * 3 * 2 * sizeof(int);
    const size_t epi = 2 * size_t(P) * sizeof(double);
    return (ring > epi ? ring : epi) + 64;
  }
};

// NR plain rows (single-row super-nodes, not the candidate's s or r): Vc,
// |Vc|, the exact cluster error, then NR super-node boundaries of the ordered
// fold. All NR rows are independent until the fold (ILP NR).
template <int NL, int NR>
__device__ __forceinline__ void score2_plain(const double2* __restrict__ bvp, const double2* __restrict__ zp, int L2,
                                             int u0, const C2 (&cv)[NL], double& smice, double& cm, double& mx) {
  double em[NR];
  bool bad = false;
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    const double2 b0 = bvp[(u0 + v) * L2], b1 = bvp[(u0 + v) * L2 + 1];
    double vx = b0.x, vy = b0.y;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double2 dz = zp[(k * 2) * K2 + u0 + v];
      vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
      vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
    }
    const double s2 = dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy));
    bad = bad || !sqrt_fast_ok(s2);
    const double m = sqrt_rn_fast(s2);
    em[v] = dmax(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
  }
  if (__any_sync(0xffffffffu, bad)) {  // |Vc|^2 outside the fast sqrt range: exact path
#pragma unroll
    for (int v = 0; v < NR; ++v) {
      const double2 b0 = bvp[(u0 + v) * L2], b1 = bvp[(u0 + v) * L2 + 1];
      double vx = b0.x, vy = b0.y;
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const double2 dz = zp[(k * 2) * K2 + u0 + v];
        vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
        vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
      }
      const double m = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
      em[v] = dmax(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
    }
  }
  // NR super-node boundaries (reduce.cpp:110-121): close the open cluster;
  // the row's error is the new cluster's maximum
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    smice = dev::dadd(smice, cm);
    cm = em[v];
    mx = dmax(mx, em[v]);
  }
}

__device__ __forceinline__ bool score2_block_plain(uint4 e4) {
  return ((e4.x & e4.y & e4.z & e4.w) & 4u) && ((e4.x & 3u) != 3u) && ((e4.y & 3u) != 3u) && ((e4.z & 3u) != 3u) &&
         ((e4.w & 3u) != 3u);
}

template <int NL>
__device__ __forceinline__ void score2_body(const RowArgs& a, int cta, int g_begin, int g_count, int R,
                                            double* smd) {
  const int L = a.L;
  const int P = blockDim.x;
  const int G = a.G;
  const int tid = threadIdx.x;
  const int gl = min(tid / L, G - 1);
  const int l = tid - gl * L < L ? tid - gl * L : 0;
  const int cg = cta * G + gl;
  const bool valid = tid < G * L && cg < g_count;
  const int c = g_begin + (valid ? cg : 0);
  const Score2Layout lay{L, G, NL};
  double2* base2 = reinterpret_cast<double2*>(smd);
  const size_t buf_e = lay.buf_e();
  auto tab_s = [&](int b) { return reinterpret_cast<unsigned*>(base2 + b * buf_e); };
  auto bv_s = [&](int b) { return base2 + b * buf_e + lay.tab_e(); };
  auto z_s = [&](int b) { return base2 + b * buf_e + lay.tab_e() + lay.bv_e(); };
  int* zcol = reinterpret_cast<int*>(base2 + 3 * buf_e);  // [G][NL][2]

  const int4 cd = a.cand[c];
  const int s = cd.x, r = cd.y;
  const int sblk = cd.z >> 2, rblk = cd.w >> 2;  // a super-node's rows share one 4-row block
  const int ts0 = cd.z, tr0 = cd.w;
  const unsigned ms = a.mask[s], mr = a.mask[r];
  const int ts1 = ts0 + __popc(ms), tr1 = tr0 + NL;
  const int rs0 = a.prow_off[s], rr0 = a.prow_off[r];
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  C2 cv[NL];
  double rlo0 = INF, rlo1 = INF, rlo2 = INF, rhi0 = -INF, rhi1 = -INF, rhi2 = -INF;
  {
    int j = 0;
#pragma unroll
    for (int ph = 0; ph < 3; ++ph) {
      if (!((mr >> ph) & 1u)) continue;
      const int rr = rr0 + popc_below(mr, ph);
      const double2 bnd = a.bv[(size_t(rr) * L + l) * 2 + 1];
      if (ph == 0) { rlo0 = bnd.x; rhi0 = bnd.y; }
      if (ph == 1) { rlo1 = bnd.x; rhi1 = bnd.y; }
      if (ph == 2) { rlo2 = bnd.x; rhi2 = bnd.y; }
      const C2 cz = ld2(a.iagg + (size_t(r) * L + l) * 3 + ph);
#pragma unroll
      for (int k = 0; k < NL; ++k)
        if (k == j) cv[k] = cz;
      if (l == 0 && tid < G * L) {
        zcol[(gl * NL + j) * 2 + 0] = rs0 + popc_below(ms, ph);
        zcol[(gl * NL + j) * 2 + 1] = rr;
      }
      ++j;
    }
  }
  __syncthreads();
  const size_t nphi = size_t(a.nphi);
  const int ntiles = (R + K2 - 1) / K2;

  // each thread stages a fixed 16-byte column of every bv row it owns when
  // the CTA width is a multiple of a row's 2L chunks (no divisions per chunk)
  const bool bv_fixed = (P % (2 * L)) == 0;
  const int bv_rem = tid % (2 * L), bv_u0 = tid / (2 * L), bv_du = P / (2 * L);
  auto stage = [&](int j, int b) {
    const int t0 = j * K2;
    for (int i = tid; i < K2 / 4; i += P) cp_async16(tab_s(b) + 4 * i, a.tab + t0 + 4 * i);
    // (base, bounds): global [rho][L][2] -> shared [row][L][2] (consecutive
    // scenarios contiguous: conflict-free 16-byte reads across a warp)
    if (bv_fixed) {
      for (int u = bv_u0; u < K2; u += bv_du) {
        const size_t rho = __ldg(a.tab + t0 + u) >> 3;
        cp_async16(bv_s(b) + size_t(u) * 2 * L + bv_rem, a.bv + rho * 2 * L + bv_rem);
      }
    } else {
      const int nbv = K2 * L * 2;
      for (int i = tid; i < nbv; i += P) {
        const int u = i / (2 * L);
        const int rem = i - u * 2 * L;
        const size_t rho = __ldg(a.tab + t0 + u) >> 3;
        cp_async16(bv_s(b) + size_t(u) * 2 * L + rem, a.bv + rho * 2 * L + rem);
      }
    }
    // Zs / Zr rows of the CTA's candidates: shared [g][k][2][row]
    const int nz = G * NL * 2 * K2;
    for (int i = tid; i < nz; i += P) {
      const int u = i % K2;
      const int col = zcol[i / K2];
      const size_t rho = __ldg(a.tab + t0 + u) >> 3;
      cp_async16(z_s(b) + i, a.Z + size_t(col) * nphi + rho);
    }
  };
  auto form_d = [&](int b) {  // D = Zs - Zr (scalar.cpp:16-17), once per (candidate, phase, row)
    double2* zz = z_s(b);
    const int nd = G * NL * K2;
    for (int i = tid; i < nd; i += P) {
      const int col2 = i / K2, u = i - col2 * K2;
      const double2 za = zz[(col2 * 2 + 0) * K2 + u], zr = zz[(col2 * 2 + 1) * K2 + u];
      zz[(col2 * 2 + 0) * K2 + u] = make_double2(dev::dsub(za.x, zr.x), dev::dsub(za.y, zr.y));
    }
  };

  double smice = 0.0, mx = 0.0, cm = 0.0;
  stage(0, 0);
  cp_async_commit();
  if (ntiles > 1) stage(1, 1);
  cp_async_commit();
  cp_async_wait1();
  __syncthreads();
  form_d(0);
  for (int j = 0; j < ntiles; ++j) {
    const int b = j % 3;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (j + 2 < ntiles) stage(j + 2, (j + 2) % 3);
    cp_async_commit();
    if (j + 1 < ntiles) form_d((j + 1) % 3);
    const int t0 = j * K2;
    const int L2 = 2 * L;
    const unsigned* tb = tab_s(b);
    const double2* bvp = bv_s(b) + size_t(l) * 2;  // this thread's scenario, row stride 2L
    const double2* zp = z_s(b) + size_t(gl) * NL * 2 * K2;
    int q = 0;
#pragma unroll 1
    while (q < K2 / 4) {
      const int blk = (t0 >> 2) + q;
      const uint4 e4 = *reinterpret_cast<const uint4*>(tb + 4 * q);
      const bool fast = score2_block_plain(e4) && !__any_sync(0xffffffffu, blk == sblk || blk == rblk);
      if (fast && q + 1 < K2 / 4) {
        const uint4 f4 = *reinterpret_cast<const uint4*>(tb + 4 * q + 4);
        if (score2_block_plain(f4) && !__any_sync(0xffffffffu, blk + 1 == sblk || blk + 1 == rblk)) {
          score2_plain<NL, 8>(bvp, zp, L2, 4 * q, cv, smice, cm, mx);
          q += 2;
          continue;
        }
      }
      const int u0 = 4 * q;
      const unsigned e[4] = {e4.x, e4.y, e4.z, e4.w};
      double em[4];
      if (fast) {
        score2_plain<NL, 4>(bvp, zp, L2, u0, cv, smice, cm, mx);
      } else {
        // general block: padding, multi-row super-nodes, the candidate's s
        // (bounds merged with r's, reduce.cpp:114-115) and r (skipped, :111)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int t = t0 + u0 + v;
          const unsigned ev = e[v];
          const unsigned ph = ev & 3u;
          const double2 b0 = bvp[(u0 + v) * L2], b1 = bvp[(u0 + v) * L2 + 1];
          double vx = b0.x, vy = b0.y;
#pragma unroll
          for (int k = 0; k < NL; ++k) {
            if (dev::cis0(cv[k])) continue;  // reduce.cpp:227: a zero current adds nothing
            const double2 dz = zp[(k * 2) * K2 + u0 + v];
            vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
            vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
          }
          const double m = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
          double lo = b1.x, hi = b1.y;
          if (t >= ts0 && t < ts1 && ph != 3u) {
            lo = dmin(lo, ph == 0u ? rlo0 : (ph == 1u ? rlo1 : rlo2));
            hi = dmax(hi, ph == 0u ? rhi0 : (ph == 1u ? rhi1 : rhi2));
          }
          em[v] = ((t >= tr0 && t < tr1) || ph == 3u) ? 0.0 : dmax(dev::dsub(m, lo), dev::dsub(hi, m));
          if (ev & 4u) {
            smice = dev::dadd(smice, cm);
            cm = 0.0;
          }
          cm = dmax(cm, em[v]);
          mx = dmax(mx, em[v]);
        }
      }
      ++q;
    }
  }
  smice = dev::dadd(smice, cm);
  // per-candidate epilogue: scenario sum in scenario order (reduce.cpp:240), feasibility
  __syncthreads();
  double* sh = smd;  // reuse: [2][P]
  sh[tid] = smice;
  sh[P + tid] = mx;
  __syncthreads();
  if (valid) {
    const int orig = a.cand_idx[c];
    a.out_maxerr[size_t(orig) * L + l] = mx;
    if (l == 0) {
      double sum = 0.0;
      bool feasible = true;
      for (int k = 0; k < L; ++k) {
        sum = dev::dadd(sum, sh[gl * L + k]);
        feasible = feasible && !(sh[P + gl * L + k] > a.e_bar);
      }
      a.out_cand[orig] = feasible ? sum : -1.0;
    }
  }
}

__global__ void __launch_bounds__(256) score2_kernel(RowArgs a) {
  extern __shared__ double sm_dyn[];
  const int b = blockIdx.x;
  int C = a.C, R = a.R;
  const int* gs = a.grp_start;
  const int* gc = a.grp_cta;
  if (a.st) {
    if (a.st->done) return;
    if (a.tdbg && b == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.tdbg[size_t(a.st->iter) * 8 + 6] = t;
    }
    C = a.st->C;
    R = a.st->R;
    gs = a.st->grp_start;
    gc = a.st->grp_cta;
    if (b >= gc[3]) return;
  }
  if (b < gc[1])
    score2_body<1>(a, b, gs[1], gs[2] - gs[1], R, sm_dyn);
  else if (b < gc[2])
    score2_body<2>(a, b - gc[1], gs[2], gs[3] - gs[2], R, sm_dyn);
  else
    score2_body<3>(a, b - gc[2], gs[3], C - gs[3], R, sm_dyn);
}

}  // namespace
}  // namespace kronred::b200
