// score3: the production magnitude-objective scorer (reduce.cpp:89-123,
// 194-244). S lanes per (candidate, scenario) pair, S in {1, 2, 4} chosen per
// iteration from the pair count (row split, below).
//
// A CTA owns Gk candidates x Ls scenarios (a scenario slice; Gk = G / |phi(r)|
// so the staged Z columns always fit G slots) and walks the iteration's row
// table in tiles of K3 = 16 rows (four 4-row blocks; a block never splits a
// super-node). Tiles stream through a three-slot shared-memory ring with one
// barrier per tile:
//
//   iteration j:  wait for tile j+1's cp.async group -> __syncthreads ->
//                 issue tile j+2 into the slot tile j-1 used ->
//                 form D = Zs - Zr of tile j+1 in place (once per candidate and
//                 phase, shared by the slice's scenarios) -> compute tile j.
//
// The scenario slice keeps the (base, bounds) tile small and independent of
// L, so occupancy does not fall as the scenario count grows. Each pair writes
// its SMICE and max_err; the scenario sum in scenario order and the
// feasibility test (reduce.cpp:221-242) run in the argmin/commit kernel.
//
// Per 4-row block the common case (single-row super-nodes, none of them the
// candidate's s or r, no padding) runs straight-line code over 8 or 4 rows:
// Vc = base + sum_p c_p D_p, |Vc| (branch-free correctly rounded sqrt),
// em = max(m - min_j v_j, max_j v_j - m) (exact cluster maximum), the ordered
// SMICE sum and the running max_err. Other blocks take the general per-row
// path; a block whose |Vc|^2 leaves the fast sqrt range is redone with
// __dsqrt_rn.
//
// Row split. A tile is four 4-row passes. With S lanes per pair (adjacent
// lanes of one warp), lane q computes passes q, q + S, ... of every tile, so a
// pair walks its rows S times faster and S times as many warps fill the GPU
// when the candidate set is small (mid and late iterations). The ordered
// SMICE fold stays one left-to-right chain: after each round of S passes the
// owner lanes fold their own rows in pass order, handing (smice, cm) on by
// warp shuffle; max_err is an order-free maximum, reduced over the S lanes at
// the end. Every rounding step is the S = 1 program's.
#pragma once

namespace kronred::b200 {
namespace {

constexpr int K3 = 16;  // rows per tile

struct S3Args {
  int C, L, nphi, R;
  int G;                     // Z column slots per CTA (candidates per CTA = G / |phi(r)| / S)
  int S;                     // lanes per pair (host-driven loop; the device loop reads st->S)
  int skip_nl1;              // 1: leave the |phi(r)| = 1 items to score1_kernel
  int s_multi;               // lanes per pair of the |phi(r)| >= 2 items when skip_nl1
  int Ls, nsl;               // scenario slice width and slice count
  const int4* cand;          // grouped by |phi(r)|: (s, r, table row of s, table row of r)
  const int* cand_idx;       // lexicographic index of each grouped slot
  const unsigned* tab;       // (rho << 3) | (first << 2) | phase, padded
  const std::uint8_t* mask;
  const int* prow_off;
  const double2* Z;          // [nphi cols][nphi rows]
  const double2* bv;         // [rho][L][2]
  const double2* iagg;       // [n][L][3]
  double* out_sm;            // [L][ldc] per-pair SMICE (lexicographic candidate index)
  double* out_mx;            // [L][ldc] per-pair max_err
  int ldc;                   // leading dimension (>= largest candidate count)
  double e_bar;
  double* out_cand;          // [C] per-candidate SMICE (scenario order) or -1 (infeasible)
  int* grp_done;             // [candidate groups] slice-completion counters (zeroed, self-resetting)
  const std::uint8_t* tplain;  // [tiles] 1: the tile's 16 rows are single-row super-nodes, no padding
  int grp_start[4];          // candidate offset of each |phi(r)| group (1..3)
  int grp_cta[4];            // first CTA of each group; grp_cta[3] = CTAs in use
  const LoopState* st;       // device-resident loop: C, R and the layout come from here
  unsigned long long* tdbg;
};

// candidates per CTA for |phi(r)| = NL at S lanes per pair
__host__ __device__ __forceinline__ int s3_cpc(int G, int NL, int S) { return G / NL / S > 1 ? G / NL / S : 1; }

// The row-split program (SF = 0, S = 2 or 4) runs a two-slot ring instead: it
// waits for tile j + 1 and forms its D after computing tile j (two barriers per
// tile) in 2/3 of the shared memory (5,991 nodes x 2 scenarios: -2 %,
// tools/s3ns_ab.sh; S3_NS_SPLIT=3 gives it the three-slot ring).
#ifndef S3_NS_SPLIT
#define S3_NS_SPLIT 2
#endif

struct S3Layout {
  int Ls, G;
  int S = 1;
  int NS = 3;  // ring slots  // lanes per pair: a CTA stages Z for G / S slots (the host sizes each split's launch)
  __host__ __device__ size_t tab_e() const { return (K3 * 4 + 15) / 16; }  // double2 units
  __host__ __device__ size_t bv_e() const { return size_t(Ls) * K3 * 2; }
  // Zs and Zr staging; each candidate's block padded by one 16-byte slot so
  // the candidates of a warp hit different banks (the largest over |phi(r)|)
  __host__ __device__ size_t z_e() const {
    size_t m = 0;
    for (int nl = 1; nl <= 3; ++nl) {
      const size_t e = size_t(s3_cpc(G, nl, S)) * size_t(nl * 2 * K3 + 1);
      m = e > m ? e : m;
    }
    return m;
  }
  __host__ __device__ size_t zcol_n() const {  // [Gk][NL][2] column indices
    size_t m = 0;
    for (int nl = 1; nl <= 3; ++nl) {
      const size_t e = size_t(s3_cpc(G, nl, S)) * size_t(nl * 2);
      m = e > m ? e : m;
    }
    return m;
  }
  __host__ __device__ size_t buf_e() const { return tab_e() + bv_e() + z_e(); }
  __host__ __device__ size_t smem_bytes() const { return size_t(NS) * buf_e() * sizeof(double2) + zcol_n() * sizeof(int) + 64; }
};

#ifndef S3_NNMAX
#define S3_NNMAX 1
#endif
#ifndef S3_MIN_BLOCKS  // tuning: resident CTAs the register budget is sized for
#define S3_MIN_BLOCKS 3
#endif

// max(a, b) for the scorer's error terms. Every call has at least one operand
// >= +0 (em = max(m - lo, hi - m) with lo <= hi: if m < lo then hi - m > 0;
// the running maxima start at +0), and a non-negative double orders like its
// bit pattern read as a signed 64-bit integer while any negative one (sign bit
// set) reads as a negative integer. So the integer maximum is the exact
// floating-point maximum here, and it runs on the integer pipes instead of
// a DSETP on the FP64 pipe.
__device__ __forceinline__ double s3max(double a, double b) {
#if S3_NNMAX
  const long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double(x > y ? x : y);
#else
  return dmax(a, b);
#endif
}

// max_err over a pass: a pairwise tree (max is exact and order-free), so the
// dependent chain is log2(NR) deep instead of NR
template <int NR>
__device__ __forceinline__ double s3_tree_max(const double (&em)[NR]) {
  double t[NR];
#pragma unroll
  for (int v = 0; v < NR; ++v) t[v] = em[v];
#pragma unroll
  for (int w = NR / 2; w >= 1; w /= 2)
#pragma unroll
    for (int v = 0; v < w; ++v) t[v] = s3max(t[v], t[v + w]);
  return t[0];
}

// NR plain rows: Vc, |Vc| and the exact cluster error of each row (ILP NR).
template <int NL, int NR>
__device__ __forceinline__ void s3_plain_em(const double2* __restrict__ bvp, const double2* __restrict__ zp, int RS,
                                            int u0, const C2 (&cv)[NL], double (&em)[NR]) {
  bool bad = false;
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    const double2 b0 = bvp[(u0 + v) * RS], b1 = bvp[(u0 + v) * RS + (RS >> 1)];
    double vx = b0.x, vy = b0.y;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double2 dz = zp[(k * 2) * K3 + u0 + v];
      vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
      vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
    }
    const double s2 = dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy));
    bad = bad || !sqrt_fast_ok(s2);
    const double m = sqrt_rn_fast(s2);
    em[v] = s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
  }
  if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
    for (int v = 0; v < NR; ++v) {
      const double2 b0 = bvp[(u0 + v) * RS], b1 = bvp[(u0 + v) * RS + (RS >> 1)];
      double vx = b0.x, vy = b0.y;
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const double2 dz = zp[(k * 2) * K3 + u0 + v];
        vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
        vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
      }
      const double m = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
      em[v] = s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
    }
  }
}

// the ordered fold over NR plain rows (every row a super-node boundary)
template <int NR>
__device__ __forceinline__ void s3_fold_plain(const double (&em)[NR], double& smice, double& cm) {
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    smice = dev::dadd(smice, cm);
    cm = em[v];
  }
}

__device__ __forceinline__ bool s3_block_plain(uint4 e4) {
  return ((e4.x & e4.y & e4.z & e4.w) & 4u) && ((e4.x & 3u) != 3u) && ((e4.y & 3u) != 3u) && ((e4.z & 3u) != 3u) &&
         ((e4.w & 3u) != 3u);
}

// Per-candidate scenario reduction of score3's per-pair results: SMICE summed
// in scenario order ((0 + s_0) + s_1) + ... (reduce.cpp:221-242), feasible
// iff every scenario's max_err <= e_bar.
__device__ __forceinline__ double s3_candidate(const double* sm, const double* mxv, int c, int L, int ldc,
                                               double e_bar) {
  double sum = 0.0;
  bool feasible = true;
  for (int l0 = 0; l0 < L; l0 += 8) {
    double v[8], m[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // issue the slice's loads together, then the ordered adds
      const bool in = l0 + u < L;
      v[u] = in ? __ldcg(sm + size_t(l0 + u) * ldc + c) : 0.0;  // L2: written by other CTAs
      m[u] = in ? __ldcg(mxv + size_t(l0 + u) * ldc + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (l0 + u < L) {
        sum = dev::dadd(sum, v[u]);
        feasible = feasible && !(m[u] > e_bar);
      }
  }
  return feasible ? sum : -1.0;  // a feasible SMICE is never negative
}


// Row context of the general (non-plain) passes: the candidate's s rows merge
// r's member bounds, r's rows and padding rows contribute nothing.
struct S3Fix {
  int ts0, ts1, tr0, tr1;
  double rlo0, rlo1, rlo2, rhi0, rhi1, rhi2;
};

// NR rows of a non-plain tile, still on the fast sqrt path. Per row (t =
// table row, e = table entry):
//   em = max(m - lo, hi - m)                              cluster error
//   s row: em = max(em, m - rlo_p, rhi_p - m)             = max(m - min(lo, rlo_p), max(hi, rhi_p) - m)
//          exactly, rounded subtraction being monotone (reduce.cpp:114-115)
//   r row or padding row: em = 0                          (reduce.cpp:111; +0 is an exact no-op below)
//   fold driven by the first-of-super-node bit            (reduce.cpp:110-121)
// A zero current c_p adds (+-0) to Vc, which leaves |Vc| bit-identical for
// finite Z, so the reference's skip (reduce.cpp:227) needs no branch here.
template <int NL, int NR>
__device__ __forceinline__ void s3_rows_gen_em(const double2* __restrict__ bvp, const double2* __restrict__ zp,
                                               int RS, int u0, int t0, const unsigned* tb, const C2 (&cv)[NL],
                                               const S3Fix& f, double (&em)[NR]) {
  bool bad = false;
  auto fix = [&](int v, double m, double e) {
    const int t = t0 + u0 + v;
    const unsigned ph = tb[u0 + v] & 3u;
    if (t >= f.ts0 && t < f.ts1 && ph != 3u) {
      const double rl = ph == 0u ? f.rlo0 : (ph == 1u ? f.rlo1 : f.rlo2);
      const double rh = ph == 0u ? f.rhi0 : (ph == 1u ? f.rhi1 : f.rhi2);
      e = s3max(e, s3max(dev::dsub(m, rl), dev::dsub(rh, m)));
    }
    return ((t >= f.tr0 && t < f.tr1) || ph == 3u) ? 0.0 : e;
  };
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    const double2 b0 = bvp[(u0 + v) * RS], b1 = bvp[(u0 + v) * RS + (RS >> 1)];
    double vx = b0.x, vy = b0.y;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double2 dz = zp[(k * 2) * K3 + u0 + v];
      vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
      vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
    }
    const double s2 = dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy));
    bad = bad || !sqrt_fast_ok(s2);
    const double m = sqrt_rn_fast(s2);
    em[v] = fix(v, m, s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m)));
  }
  if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
    for (int v = 0; v < NR; ++v) {
      const double2 b0 = bvp[(u0 + v) * RS], b1 = bvp[(u0 + v) * RS + (RS >> 1)];
      double vx = b0.x, vy = b0.y;
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const double2 dz = zp[(k * 2) * K3 + u0 + v];
        vx = dev::dadd(vx, dev::dsub(dev::dmul(cv[k].x, dz.x), dev::dmul(cv[k].y, dz.y)));
        vy = dev::dadd(vy, dev::dadd(dev::dmul(cv[k].x, dz.y), dev::dmul(cv[k].y, dz.x)));
      }
      const double m = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
      em[v] = fix(v, m, s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m)));
    }
  }
}

// the ordered fold over NR general rows, driven by the first-of-super-node bit
template <int NR>
__device__ __forceinline__ void s3_fold_gen(const double (&em)[NR], const unsigned* tb, int u0, double& smice,
                                            double& cm) {
#pragma unroll
  for (int v = 0; v < NR; ++v) {
    if (tb[u0 + v] & 4u) {
      smice = dev::dadd(smice, cm);
      cm = 0.0;
    }
    cm = s3max(cm, em[v]);
  }
}

// (smice, cm) of lane q of this lane's S-lane group, to every lane of the group
__device__ __forceinline__ void s3_handoff(double& smice, double& cm, int q, int S) {
  const int src = (int(threadIdx.x & 31u) & ~(S - 1)) | q;
  smice = __shfl_sync(0xffffffffu, smice, src);
  cm = __shfl_sync(0xffffffffu, cm, src);
}

// One work item (a group of candidates x one scenario slice). SF = 1: the
// one-lane-per-pair program compiled on its own (S = 1); SF = 0: S lanes per
// pair from the argument.
template <int NL, int LSC, int SF>  // LSC: compile-time slice width (0: runtime a.Ls)
__device__ __forceinline__ void s3_body(const S3Args& a, int S_arg, int local, int g_begin, int g_count, int R,
                                     double* smd, int g_base_group) {
  const int S = SF ? 1 : S_arg;
  const int L = a.L, Ls = LSC ? LSC : a.Ls;
  const int Gk = s3_cpc(a.G, NL, S);
  const int P = blockDim.x;
  const int tid = threadIdx.x;
  const int pr = tid / S, myq = tid - pr * S;  // pair slot, lane within the pair's group
  const int cgrp = local / a.nsl, sl = local - cgrp * a.nsl;
  const int gl = min(pr / Ls, Gk - 1);
  const int ll = pr - (pr / Ls) * Ls;
  const int l = min(sl * Ls + ll, L - 1);
  const int cg = cgrp * Gk + gl;
  const bool valid = pr < Gk * Ls && cg < g_count && sl * Ls + ll < L && myq == 0;
  const int c = g_begin + min(cg, g_count - 1);
  const S3Layout lay{Ls, a.G, S};
  double2* base2 = reinterpret_cast<double2*>(smd);
  // staging ring: NS slots sized for this item's candidates (a deeper ring
  // measured no faster: the copy latency is covered by one tile's compute)
  const size_t buf_e = lay.tab_e() + lay.bv_e() + size_t(Gk) * (NL * 2 * K3 + 1);
  constexpr int NS = SF ? 3 : S3_NS_SPLIT;
  auto tab_s = [&](int b) { return reinterpret_cast<unsigned*>(base2 + b * buf_e); };
  auto bv_s = [&](int b) { return base2 + b * buf_e + lay.tab_e(); };
  auto z_s = [&](int b) { return base2 + b * buf_e + lay.tab_e() + lay.bv_e(); };
  // the same slots as shared-space byte addresses for the copies (computed
  // once: a generic -> shared conversion per copy re-reads the CTA's shared
  // window register inside the tile loop)
  unsigned sbase = unsigned(__cvta_generic_to_shared(smd));
  asm volatile("mov.b32 %0, %0;" : "+r"(sbase));
  auto tab_a = [&](int b) { return sbase + unsigned(b * buf_e) * 16u; };
  auto bv_a = [&](int b) { return sbase + unsigned(b * buf_e + lay.tab_e()) * 16u; };
  auto z_a = [&](int b) { return sbase + unsigned(b * buf_e + lay.tab_e() + lay.bv_e()) * 16u; };
  int* zcol = reinterpret_cast<int*>(base2 + NS * lay.buf_e());  // [Gk][NL][2]

  const int4 cd = a.cand[c];
  const int s = cd.x, r = cd.y;
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
      const double2 bnd = a.bv[bv_bnd(size_t(rr), L, l)];
      if (ph == 0) { rlo0 = bnd.x; rhi0 = bnd.y; }
      if (ph == 1) { rlo1 = bnd.x; rhi1 = bnd.y; }
      if (ph == 2) { rlo2 = bnd.x; rhi2 = bnd.y; }
      const C2 cz = ld2(a.iagg + (size_t(r) * L + l) * 3 + ph);
#pragma unroll
      for (int k = 0; k < NL; ++k)
        if (k == j) cv[k] = cz;
      if (ll == 0 && myq == 0 && pr < Gk * Ls) {
        zcol[(gl * NL + j) * 2 + 0] = rs0 + popc_below(ms, ph);
        zcol[(gl * NL + j) * 2 + 1] = rr;
      }
      ++j;
    }
  }
  __syncthreads();
  const S3Fix fx{ts0, ts1, tr0, tr1, rlo0, rlo1, rlo2, rhi0, rhi1, rhi2};
  const size_t nphi = size_t(a.nphi);
  const int ntiles = (R + K3 - 1) / K3;
  // (base, bounds) slice staging: each row is 2*Ls contiguous 16-byte chunks
  const int RS = 2 * Ls;
  const int nsc = min(Ls, L - sl * Ls);  // scenarios of this slice
  const bool bv_fixed = (P % RS) == 0;
  const int bv_ch = tid % RS, bv_u0 = tid / RS, bv_du = P / RS;
  // a row's slice: Ls base values, then Ls bounds, both in global (row-planar
  // bv, bv_base/bv_bnd) and in shared memory
  const int bv_dst = bv_ch;
  const size_t bv_off = size_t(bv_ch / Ls) * L + size_t(sl) * Ls + size_t(bv_ch % Ls);
  const bool bv_in = (bv_ch % Ls) < nsc;

  const int nz = Gk * NL * 2 * K3;  // Z staging slots per tile (16-byte)
#ifndef S3_Z_EVICT_FIRST
#define S3_Z_EVICT_FIRST 1
#endif
  const unsigned long long zpol = S3_Z_EVICT_FIRST ? l2_evict_first_policy() : l2_evict_normal_policy();
  auto stage = [&](int j, int b) {
    const int t0 = j * K3;
    for (int i = tid; i < K3 / 4; i += P) cp_async16s(tab_a(b) + 16u * unsigned(i), a.tab + t0 + 4 * i);
    if (bv_fixed) {
      if (bv_in)
        for (int u = bv_u0; u < K3; u += bv_du) {
          const size_t rho = __ldg(a.tab + t0 + u) >> 3;
          cp_async16s(bv_a(b) + unsigned(u * RS + bv_dst) * 16u, a.bv + rho * 2 * L + bv_off);
        }
    } else {
      for (int i = tid; i < K3 * RS; i += P) {
        const int u = i / RS, ch = i - u * RS;
        if (ch % Ls >= nsc) continue;
        const size_t rho = __ldg(a.tab + t0 + u) >> 3;
        cp_async16s(bv_a(b) + unsigned(u * RS + ch) * 16u,
                    a.bv + rho * 2 * L + size_t(ch / Ls) * L + size_t(sl) * Ls + size_t(ch % Ls));
      }
    }
    for (int i = tid; i < nz; i += P) {
      const int u = i % K3;
      const int col = zcol[i / K3];
      const size_t rho = __ldg(a.tab + t0 + u) >> 3;
      cp_async16s_hint(z_a(b) + unsigned(i + i / (NL * 2 * K3)) * 16u, a.Z + size_t(col) * nphi + rho, zpol);
    }
  };
  // Fast staging: each thread owns at most two bv rows and one table row of
  // the Z block in every tile, and at most four fixed Z slots (same column for
  // the whole item), so the column sources are resolved once and the table
  // entries are prefetched raw one tile ahead: no dependent load in front of a
  // cp.async, and the prefetch is not consumed until the next tile.
  const bool fst = bv_fixed && (P % K3) == 0 && 2 * bv_du >= K3;
  const int u_a = bv_u0, u_b = bv_u0 + bv_du, u_z = tid % K3;
  const double2* zsrc[4];
  int zdst[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = min(tid + q * P, nz - 1);
    zsrc[q] = a.Z + size_t(zcol[i / K3]) * nphi;
    zdst[q] = i + i / (NL * 2 * K3);
  }
  auto load_rho = [&](int j, unsigned (&rr)[3]) {  // raw table entries: (rho << 3) | flags
    const int t0 = j * K3;
    rr[0] = (j < ntiles && u_a < K3) ? __ldg(a.tab + t0 + u_a) : 0u;
    rr[1] = (j < ntiles && u_b < K3) ? __ldg(a.tab + t0 + u_b) : 0u;
    rr[2] = j < ntiles ? __ldg(a.tab + t0 + u_z) : 0u;
  };
  auto stage_fast = [&](int j, int b, const unsigned (&rr)[3]) {
    const int t0 = j * K3;
    if (tid < K3 / 4) cp_async16s(tab_a(b) + 16u * unsigned(tid), a.tab + t0 + 4 * tid);
    if (bv_in) {
      if (u_a < K3)
        cp_async16s(bv_a(b) + unsigned(u_a * RS + bv_dst) * 16u, a.bv + size_t(rr[0] >> 3) * 2 * L + bv_off);
      if (u_b < K3)
        cp_async16s(bv_a(b) + unsigned(u_b * RS + bv_dst) * 16u, a.bv + size_t(rr[1] >> 3) * 2 * L + bv_off);
    }
    const size_t rz = rr[2] >> 3;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (tid + q * P < nz) cp_async16s_hint(z_a(b) + unsigned(zdst[q]) * 16u, zsrc[q] + rz, zpol);
    // small CTAs (few scenarios): the remaining slots, same table row (P % K3 == 0)
    for (int i = tid + 4 * P; i < nz; i += P)
      cp_async16s_hint(z_a(b) + unsigned(i + i / (NL * 2 * K3)) * 16u, a.Z + size_t(zcol[i / K3]) * nphi + rz, zpol);
  };
  // D = Zs - Zr (scalar.cpp:16-17), once per (candidate, phase, row); each
  // thread's element offsets are fixed for the item (at most two per thread
  // for 128-thread CTAs: both pairs loaded before either difference)
  const int nd = Gk * NL * K3;
  auto fd_off = [&](int i) {
    const int col2 = i / K3, u = i - col2 * K3;
    const int g = col2 / NL;  // candidate: its block starts at g * (NL * 2 * K3 + 1)
    return g * (NL * 2 * K3 + 1) + (col2 - g * NL) * 2 * K3 + u;
  };
  const bool fd2 = nd <= 2 * P;
  const int fdo0 = fd_off(min(tid, nd - 1)), fdo1 = fd_off(min(tid + P, nd - 1));
  const bool fdv0 = tid < nd, fdv1 = tid + P < nd;
  auto form_d = [&](int b) {
    double2* zz = z_s(b);
    if (fd2) {
      const double2 za0 = zz[fdo0], zr0 = zz[fdo0 + K3], za1 = zz[fdo1], zr1 = zz[fdo1 + K3];
      if (fdv0) zz[fdo0] = make_double2(dev::dsub(za0.x, zr0.x), dev::dsub(za0.y, zr0.y));
      if (fdv1) zz[fdo1] = make_double2(dev::dsub(za1.x, zr1.x), dev::dsub(za1.y, zr1.y));
      return;
    }
    for (int i = tid; i < nd; i += P) {
      double2* zc = zz + fd_off(i);
      const double2 za = zc[0], zr = zc[K3];
      zc[0] = make_double2(dev::dsub(za.x, zr.x), dev::dsub(za.y, zr.y));
    }
  };

  double smice = 0.0, mx = 0.0, cm = 0.0;
  unsigned rn[3];
#ifdef S3_TIMING  // tuning aid: per-phase cycle counts of CTA 0's warps
  long long tm_pro = clock64(), tm_wait = 0, tm_stage = 0, tm_rho = 0, tm_fd = 0, tm_comp = 0, tm_x;
#endif
  // prologue: tiles 0 and 1 in flight (two slots: tile 0), then wait for tile 0
  if (fst) {
    unsigned r0[3], r1[3];
    load_rho(0, r0);
    load_rho(1, r1);
    stage_fast(0, 0, r0);
    cp_async_commit();
    if (NS == 3) {
      if (ntiles > 1) stage_fast(1, 1, r1);
      cp_async_commit();
      load_rho(2, rn);
    } else {
#pragma unroll
      for (int q = 0; q < 3; ++q) rn[q] = r1[q];
    }
  } else {
    stage(0, 0);
    cp_async_commit();
    if (NS == 3) {
      if (ntiles > 1) stage(1, 1);
      cp_async_commit();
    }
  }
  if (NS == 3)
    cp_async_wait1();
  else
    asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  form_d(0);
#ifdef S3_TIMING
  tm_pro = clock64() - tm_pro;
#endif
  unsigned tflag_next = a.tplain[0];  // raw byte: tested one tile later
  for (int j = 0; j < ntiles; ++j) {
    const int b = j % NS;
    const bool tflag = tflag_next != 0u;
    if (j + 1 < ntiles) tflag_next = a.tplain[j + 1];
#ifdef S3_TIMING
    tm_x = clock64();
#endif
    if (NS == 3) asm volatile("cp.async.wait_group 0;\n" ::);  // tile j + 1 has landed
    __syncthreads();  // (two slots: tile j's D is formed, tile j - 1's slot is free)
#ifdef S3_TIMING
    tm_wait += clock64() - tm_x;
    tm_x = clock64();
#endif
    const int jn = j + NS - 1;  // the tile staged now
    if (fst) {
      if (jn < ntiles) stage_fast(jn, jn % NS, rn);
      cp_async_commit();
#ifdef S3_TIMING
      tm_stage += clock64() - tm_x;
      tm_x = clock64();
#endif
      load_rho(jn + 1, rn);  // consumed next iteration: latency hidden by this tile's compute
#ifdef S3_TIMING
      tm_rho += clock64() - tm_x;
      tm_x = clock64();
#endif
    } else {
      if (jn < ntiles) stage(jn, jn % NS);
      cp_async_commit();
    }
#ifdef S3_TIMING
    tm_stage += clock64() - tm_x;
    tm_x = clock64();
#endif
    if (NS == 3 && j + 1 < ntiles) form_d((j + 1) % 3);
#ifdef S3_TIMING
    tm_fd += clock64() - tm_x;
    tm_x = clock64();
#endif
    const int t0 = j * K3;
    const unsigned* tb = tab_s(b);
    const double2* bvp = bv_s(b) + size_t(ll);  // this thread's scenario: base at +0, bounds at +Ls per row
    const double2* zp = z_s(b) + size_t(gl) * (NL * 2 * K3 + 1);
    // whole plain tile (flag from the row-table builder) with no s or r row of
    // this warp's candidates: straight-line passes with the all-first fold;
    // any other tile: the same fast passes with per-row fixups and a
    // flag-driven fold
    // passes of 4 rows; round k, lane q computes pass k * S + q (S = 1: every
    // pass, in order); the owners then fold in pass order, handing (smice, cm)
    // on to the next lane of the pair's group
    const bool plain = tflag && !__any_sync(0xffffffffu, j == (ts0 >> 4) || j == (tr0 >> 4));
    constexpr int NP = K3 / 4;
    const int rounds = NP / S;
    if (plain) {
#pragma unroll 1
      for (int k = 0; k < rounds; ++k) {
        const int u0 = 4 * (k * S + myq);
        double em[4];
        s3_plain_em<NL, 4>(bvp, zp, RS, u0, cv, em);
        mx = s3max(mx, s3_tree_max(em));
        if (S == 1) {
          s3_fold_plain<4>(em, smice, cm);
        } else {
#pragma unroll 1
          for (int q = 0; q < S; ++q) {
            if (myq == q) s3_fold_plain<4>(em, smice, cm);
            s3_handoff(smice, cm, q, S);
          }
        }
      }
    } else {
#pragma unroll 1
      for (int k = 0; k < rounds; ++k) {
        const int u0 = 4 * (k * S + myq);
        double em[4];
        s3_rows_gen_em<NL, 4>(bvp, zp, RS, u0, t0, tb, cv, fx, em);
        mx = s3max(mx, s3_tree_max(em));
        if (S == 1) {
          s3_fold_gen<4>(em, tb, u0, smice, cm);
        } else {
#pragma unroll 1
          for (int q = 0; q < S; ++q) {
            if (myq == q) s3_fold_gen<4>(em, tb, u0, smice, cm);
            s3_handoff(smice, cm, q, S);
          }
        }
      }
    }
#ifdef S3_TIMING
    tm_comp += clock64() - tm_x;
#endif
    if (NS == 2 && j + 1 < ntiles) {  // two slots: tile j + 1 lands, then its D
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      form_d((j + 1) & 1);
    }
  }
  smice = dev::dadd(smice, cm);
  for (int o = 1; o < S; o <<= 1) mx = s3max(mx, __shfl_xor_sync(0xffffffffu, mx, o));  // order-free
#ifdef S3_TIMING
  if (blockIdx.x == 0 && (tid & 31) == 0 && a.st && (a.st->iter == 1 || a.st->iter == 100 || a.st->iter == 500 || a.st->iter == 850))
    printf("s3 timing iter %d warp %d NL %d tiles %d: prologue %lld wait+sync %lld stage %lld rho %lld form_d %lld compute %lld\n",
           a.st->iter, tid >> 5, NL, ntiles, tm_pro, tm_wait, tm_stage, tm_rho, tm_fd, tm_comp);
#endif
  if (valid) {
    const size_t o = size_t(l) * a.ldc + a.cand_idx[c];
    a.out_sm[o] = smice;
    a.out_mx[o] = mx;
  }
  // the last slice CTA of a candidate group reduces its candidates over the
  // scenarios (threadfence reduction: counters reset themselves)
  // (the CTA barrier orders every thread's stores before thread 0's
  // release-acquire add at device scope; the winner's barrier orders its
  // acquire before every thread's loads)
  __shared__ int s_last;
  __syncthreads();
  const int grp = (local / a.nsl) + g_base_group;
  if (tid == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.grp_done + grp) : "memory");
    s_last = old == a.nsl - 1;
    if (s_last) a.grp_done[grp] = 0;
  }
  __syncthreads();
  if (s_last) {
    // stage the group's per-pair results in shared memory (all threads, L2
    // reads), then one thread per candidate sums in scenario order
    double* ssm = smd;                       // [Gk][L]
    double* smx = smd + size_t(Gk) * L;      // [Gk][L]
    for (int i = tid; i < Gk * L; i += P) {
      const int g = i / L, ls = i - g * L;
      const int cgc = cgrp * Gk + g;
      if (cgc < g_count) {
        const size_t o = size_t(ls) * a.ldc + a.cand_idx[g_begin + cgc];
        ssm[i] = __ldcg(a.out_sm + o);  // written by other CTAs: read through L2
        smx[i] = __ldcg(a.out_mx + o);
      }
    }
    __syncthreads();
    const int cgc = cgrp * Gk + tid;
    if (tid < Gk && cgc < g_count) {
      double sum = 0.0;
      bool feasible = true;
      for (int ls = 0; ls < L; ++ls) {  // ((0 + s_0) + s_1) + ... (reduce.cpp:221-242)
        sum = dev::dadd(sum, ssm[tid * L + ls]);
        feasible = feasible && !(smx[tid * L + ls] > a.e_bar);
      }
      a.out_cand[a.cand_idx[g_begin + cgc]] = feasible ? sum : -1.0;
    }
  }
}

// lanes per pair for an iteration with `pairs` (candidate, scenario) pairs:
// the widest split that keeps pairs * S within `fill` threads (about one wave)
#ifndef S3_FILL2_16  // the S = 2 threshold as a fraction of the budget, in sixteenths
#define S3_FILL2_16 16
#endif
#ifndef S3_FILL4_16  // the S = 4 threshold as a fraction of the budget, in sixteenths
#define S3_FILL4_16 11
#endif
__host__ __device__ __forceinline__ int s3_lanes(long long pairs, long long fill, int force, int fill4_16 = S3_FILL4_16) {
  if (force == 1 || force == 2 || force == 4) return force;
  if (pairs * 4 * 16 <= fill * fill4_16) return 4;
  if (pairs * 2 * 16 <= fill * S3_FILL2_16) return 2;
  return 1;
}

// SF = 1: the one-lane-per-pair program compiled on its own (every split
// expression a constant); SF = 0: S lanes per pair at run time (2, 4).
template <int SF>
__global__ void __launch_bounds__(128, S3_MIN_BLOCKS) score3_kernel(S3Args a) {
  extern __shared__ double sm_dyn[];
  const int b = blockIdx.x;
  griddep_wait();
  int C = a.C, R = a.R;
  const int* gs = a.grp_start;
  const int* gc = a.grp_cta;
  if (a.st) {
    if (a.st->done) return;
    if (a.tdbg && b == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      a.tdbg[size_t(a.st->iter) * kTdbg + 6] = t;
    }
    C = a.st->Cl;  // this rank's candidates (all of them on one GPU)
    R = a.st->R;
    gs = a.st->grp_start;
    gc = a.st->grp_cta;
  }
  // with score1 taking the |phi(r)| = 1 candidates, the few multi-phase ones
  // run at their own split (latency-bound: one pass per lane per tile)
  const int S = SF ? 1 : (a.skip_nl1 ? a.s_multi : (a.st ? a.st->S : a.S));
  // work items (candidate group x scenario slice) strided over the grid: the
  // device loop launches a fixed, occupancy-sized grid for every iteration
  // (skip_nl1: the |phi(r)| = 1 items run in score1_kernel)
  for (int w = b + (a.skip_nl1 ? gc[1] : 0); w < gc[3]; w += gridDim.x) {
    // counter slot: global candidate-group index (every group range is a
    // whole number of nsl-slice items)
    if (w < gc[1])
      s3_body<1, 0, SF>(a, S, w, gs[1], gs[2] - gs[1], R, sm_dyn, 0);
    else if (w < gc[2])
      s3_body<2, 0, SF>(a, S, w - gc[1], gs[2], gs[3] - gs[2], R, sm_dyn, gc[1] / a.nsl);
    else
      s3_body<3, 0, SF>(a, S, w - gc[2], gs[3], C - gs[3], R, sm_dyn, gc[2] / a.nsl);
    __syncthreads();  // shared memory is reused by the next item
  }
  if (a.tdbg && a.st && threadIdx.x == 0) atomicMax(a.tdbg + size_t(a.st->iter) * kTdbg + 14, globaltimer_ns());
}

}  // namespace
}  // namespace kronred::b200
