// score1: the magnitude-objective scorer for candidates whose absorbed node r
// has a single present phase (|phi(r)| = 1: 995 of the 1,000 nodes of the C2
// benchmark feeder and most nodes of every generated feeder), compiled for
// one geometry so every shared-memory offset is an immediate:
//   16 Z-column slots per CTA (16 / S candidates), scenario slices of 8,
//   16-row tiles, S lanes per (candidate, scenario) pair (S = 1, 2, 4; one
//   kernel per S, selected per iteration by a switch node of the loop graph).
// Per pair the arithmetic and its order are score3's (kernels_score3.cuh,
// reduce.cpp:89-123, 194-244): Vc = base + c (Zs - Zr), |Vc| by the
// branch-free correctly rounded sqrt (with the __dsqrt_rn fallback), the
// exact cluster error max(m - min, max - m), the left-to-right SMICE fold
// (handed lane to lane with S > 1) and max_err. Candidates with
// |phi(r)| >= 2 run in score3_kernel at the same time (a second stream).
#pragma once

namespace kronred::b200 {
namespace {

constexpr int kS1K = 16;                  // rows per tile
constexpr int kS1Ls = 8;                  // scenarios per slice
constexpr int kS1G = 16;                  // Z-column slots per CTA at S = 1 (default item: 16 candidates)
constexpr int kS1CB = 2 * kS1K + 1;       // per-candidate staging block: Zs rows, Zr rows, one pad slot
constexpr int kS1TabE = kS1K / 4;         // table entries per tile, in double2 units
constexpr int kS1BvE = kS1K * 2 * kS1Ls;  // base + bounds of a tile's rows, one slice

// S lanes per pair, GK candidates per item: P = GK x 8 x S threads
template <int S, int GK_>
struct S1Geom {
  static constexpr int GK = GK_;                             // candidates per item
  static constexpr int P = GK * kS1Ls * S;                   // threads per CTA
  static constexpr int BUF = kS1TabE + kS1BvE + GK * kS1CB;  // one ring slot (double2)
  static constexpr int NZ = GK * 2 * kS1K;                   // Z chunks per tile
  static constexpr int ZPT = NZ / P;                         // per thread (4 / S)
  static constexpr int BVR = kS1K * 16 / P;                  // bv rows per thread (16 chunks per row)
  static constexpr int ND = GK * kS1K;                       // D elements per tile
};
// staging ring depth per split (tiles staged NS - 1 ahead): with S lanes per
// pair a tile's compute is S times shorter, and at S = 2 a fourth slot hides
// the copy latency (-0.8 us per mid-run iteration); S = 1 and S = 4 measure
// best with three (tools/ring_ab.sh)
#ifndef S1_NS1
#define S1_NS1 3
#endif
#ifndef S1_NS2
#define S1_NS2 4
#endif
#ifndef S1_NS4
#define S1_NS4 3
#endif
template <int S>
constexpr int s1_ns() { return S == 1 ? S1_NS1 : (S == 2 ? S1_NS2 : S1_NS4); }
// dynamic shared memory of every score1 variant: the ring plus the column table
template <int S, int GK>
constexpr size_t s1_smem_bytes() {
  return size_t(s1_ns<S>()) * S1Geom<S, GK>::BUF * sizeof(double2) + GK * 2 * sizeof(int) + 64;
}

// 4 plain rows at ring offsets u0..u0+3 (bvp: this pair's scenario column;
// rows 16 double2 apart, bounds 8 further; zp: this candidate's D)
template <int U0>
__device__ __forceinline__ void s1_plain4(const double2* __restrict__ bvp, const double2* __restrict__ zp, C2 cv,
                                          double (&em)[4]) {
  bool bad = false;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const double2 b0 = bvp[(U0 + v) * 16], b1 = bvp[(U0 + v) * 16 + 8];
    const double2 dz = zp[U0 + v];
    const double vx = dev::dadd(b0.x, dev::dsub(dev::dmul(cv.x, dz.x), dev::dmul(cv.y, dz.y)));
    const double vy = dev::dadd(b0.y, dev::dadd(dev::dmul(cv.x, dz.y), dev::dmul(cv.y, dz.x)));
    const double s2 = dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy));
    bad = bad || !sqrt_fast_ok(s2);
    const double m = sqrt_rn_fast(s2);
    em[v] = s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
  }
  if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double2 b0 = bvp[(U0 + v) * 16], b1 = bvp[(U0 + v) * 16 + 8];
      const double2 dz = zp[U0 + v];
      const double vx = dev::dadd(b0.x, dev::dsub(dev::dmul(cv.x, dz.x), dev::dmul(cv.y, dz.y)));
      const double vy = dev::dadd(b0.y, dev::dadd(dev::dmul(cv.x, dz.y), dev::dmul(cv.y, dz.x)));
      const double m = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
      em[v] = s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
    }
  }
}

// 4 general rows: r's row and padding rows contribute nothing; the s row of
// r's phase merges r's member bounds (exact: rounded subtraction is monotone)
struct S1Fix {
  int ts0, ts1, tr0;
  unsigned rph;  // r's phase
  double rlo, rhi;
};
template <int U0>
__device__ __forceinline__ void s1_gen4(const double2* __restrict__ bvp, const double2* __restrict__ zp, C2 cv,
                                        const unsigned* tb, int t0, const S1Fix& f, double (&em)[4]) {
  bool bad = false;
  double m4[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const double2 b0 = bvp[(U0 + v) * 16], b1 = bvp[(U0 + v) * 16 + 8];
    const double2 dz = zp[U0 + v];
    const double vx = dev::dadd(b0.x, dev::dsub(dev::dmul(cv.x, dz.x), dev::dmul(cv.y, dz.y)));
    const double vy = dev::dadd(b0.y, dev::dadd(dev::dmul(cv.x, dz.y), dev::dmul(cv.y, dz.x)));
    const double s2 = dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy));
    bad = bad || !sqrt_fast_ok(s2);
    m4[v] = sqrt_rn_fast(s2);
  }
  if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double2 b0 = bvp[(U0 + v) * 16];
      const double2 dz = zp[U0 + v];
      const double vx = dev::dadd(b0.x, dev::dsub(dev::dmul(cv.x, dz.x), dev::dmul(cv.y, dz.y)));
      const double vy = dev::dadd(b0.y, dev::dadd(dev::dmul(cv.x, dz.y), dev::dmul(cv.y, dz.x)));
      m4[v] = dev::dsqrt(dev::dadd(dev::dmul(vx, vx), dev::dmul(vy, vy)));
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const double2 b1 = bvp[(U0 + v) * 16 + 8];
    const double m = m4[v];
    double e = s3max(dev::dsub(m, b1.x), dev::dsub(b1.y, m));
    const int t = t0 + U0 + v;
    const unsigned ph = tb[U0 + v] & 3u;
    if (t >= f.ts0 && t < f.ts1 && ph == f.rph) e = s3max(e, s3max(dev::dsub(m, f.rlo), dev::dsub(f.rhi, m)));
    em[v] = (t == f.tr0 || ph == 3u) ? 0.0 : e;
  }
}

template <int S, int GK_>
__device__ __forceinline__ void s1_item(const S3Args& a, int local, int g_count, int R, double* smd) {
  using Geo = S1Geom<S, GK_>;
  constexpr int GK = Geo::GK, P = Geo::P;
  const int L = a.L;
  const int tid = threadIdx.x;
  const int pr = tid / S, myq = tid % S;  // pair slot, lane in the pair's group
  const int nsl = a.nsl;
  const int cgrp = local / nsl, sl = local - cgrp * nsl;
  const int gl = pr / kS1Ls, ll = pr % kS1Ls;
  const int l = min(sl * kS1Ls + ll, L - 1);
  const int cg = cgrp * GK + gl;
  const bool valid = cg < g_count && sl * kS1Ls + ll < L && myq == 0;
  const int c = min(cg, g_count - 1);  // the |phi(r)| = 1 group starts at candidate slot 0
  double2* base2 = reinterpret_cast<double2*>(smd);
  constexpr int NS = s1_ns<S>();
  int* zcol = reinterpret_cast<int*>(base2 + NS * Geo::BUF);  // [GK][2]: Z columns of s and r

  const int4 cd = a.cand[c];
  const int s = cd.x, r = cd.y;
  const unsigned ms = a.mask[s], mr = a.mask[r];
  const unsigned rph = unsigned(__ffs(int(mr)) - 1);
  const int rr = a.prow_off[r];
  const double2 rb = a.bv[bv_bnd(size_t(rr), L, l)];
  const C2 cv = ld2(a.iagg + (size_t(r) * L + l) * 3 + rph);
  const S1Fix fx{cd.z, cd.z + __popc(ms), cd.w, rph, rb.x, rb.y};
  if (ll == 0 && myq == 0) {
    zcol[gl * 2 + 0] = a.prow_off[s] + popc_below(ms, int(rph));
    zcol[gl * 2 + 1] = rr;
  }
  __syncthreads();
  const size_t nphi = size_t(a.nphi);
  const int ntiles = (R + kS1K - 1) / kS1K;
  // staging roles (fixed for the item): BVR bv rows per thread (16-byte chunk
  // bv_ch of each), one table row of the Z block and ZPT Z columns
  const int bv_ch = tid % 16, u_a = tid / 16, u_z = tid % 16;
  const bool bv_in = sl * kS1Ls + (bv_ch % kS1Ls) < L;
  const size_t bv_off = size_t(bv_ch / kS1Ls) * L + size_t(sl) * kS1Ls + size_t(bv_ch % kS1Ls);
  constexpr int ZN = Geo::ZPT > 0 ? Geo::ZPT : 1;
  const double2* zsrc[ZN];
  int zdst[ZN];
  bool zon[ZN];
#pragma unroll
  for (int q = 0; q < ZN; ++q) {
    const int i = tid + q * P;  // chunk: column i / 16, row u_z
    const int col = min(i / kS1K, 2 * GK - 1);
    zon[q] = i < Geo::NZ;
    zsrc[q] = a.Z + size_t(zcol[col]) * nphi;
    zdst[q] = (col / 2) * kS1CB + (col % 2) * kS1K + u_z;
  }
  const unsigned long long zpol = l2_evict_first_policy();
  auto slot = [&](int b) { return base2 + b * Geo::BUF; };
  auto load_rho = [&](int j, unsigned (&rr3)[Geo::BVR + 1]) {  // raw table entries: (rho << 3) | flags
    const int t0 = j * kS1K;
    const bool in = j < ntiles;
#pragma unroll
    for (int k = 0; k < Geo::BVR; ++k) rr3[k] = in ? __ldg(a.tab + t0 + u_a + k * (P / 16)) : 0u;
    rr3[Geo::BVR] = in ? __ldg(a.tab + t0 + u_z) : 0u;
  };
  auto stage = [&](int j, int b, const unsigned (&rr3)[Geo::BVR + 1]) {
    double2* sb = slot(b);
    const int t0 = j * kS1K;
    if (tid < kS1TabE) cp_async16(sb + tid, a.tab + t0 + 4 * tid);
    if (bv_in) {
#pragma unroll
      for (int k = 0; k < Geo::BVR; ++k)
        cp_async16(sb + kS1TabE + (u_a + k * (P / 16)) * 16 + bv_ch, a.bv + size_t(rr3[k] >> 3) * 2 * L + bv_off);
    }
    const size_t rz = rr3[Geo::BVR] >> 3;
#pragma unroll
    for (int q = 0; q < ZN; ++q)
      if (zon[q]) cp_async16_hint(sb + kS1TabE + kS1BvE + zdst[q], zsrc[q] + rz, zpol);
  };
  // D = Zs - Zr (scalar.cpp:16-17) once per (candidate, row)
  auto form_d = [&](int b) {
    double2* zz = slot(b) + kS1TabE + kS1BvE;
#pragma unroll
    for (int e = tid; e < Geo::ND; e += P) {
      double2* zc = zz + (e / kS1K) * kS1CB + (e % kS1K);
      const double2 za = zc[0], zb = zc[kS1K];
      zc[0] = make_double2(dev::dsub(za.x, zb.x), dev::dsub(za.y, zb.y));
    }
  };

  double smice = 0.0, mx = 0.0, cm = 0.0;
  unsigned rn[Geo::BVR + 1];
  // prologue: tiles 0 .. NS - 2 in flight, then wait for tile 0
#pragma unroll
  for (int t = 0; t < NS - 1; ++t) {
    load_rho(t, rn);
    if (t < ntiles) stage(t, t, rn);
    cp_async_commit();
  }
  load_rho(NS - 1, rn);
  cp_async_wait_pending(NS - 2);
  __syncthreads();
  form_d(0);
  unsigned tflag_next = a.tplain[0];
  for (int j = 0; j < ntiles; ++j) {
    const int b = j % NS;
    const bool tflag = tflag_next != 0u;
    if (j + 1 < ntiles) tflag_next = a.tplain[j + 1];
    cp_async_wait_pending(NS - 3);  // tile j + 1 has landed
    __syncthreads();
    if (j + NS - 1 < ntiles) stage(j + NS - 1, (j + NS - 1) % NS, rn);
    cp_async_commit();
    load_rho(j + NS, rn);
    if (j + 1 < ntiles) form_d((j + 1) % NS);
    const double2* sb = slot(b);
    const unsigned* tb = reinterpret_cast<const unsigned*>(sb);
    const double2* bvp = sb + kS1TabE + ll + 4 * myq * 16;      // this lane's first pass
    const double2* zp = sb + kS1TabE + kS1BvE + gl * kS1CB + 4 * myq;
    const bool plain = tflag && !__any_sync(0xffffffffu, j == (fx.ts0 >> 4) || j == (fx.tr0 >> 4));
    const int t0 = j * kS1K + 4 * myq;
    const unsigned* tq = tb + 4 * myq;
    // round k: this lane's pass k * S + myq (rows 4 (k S + myq) .. + 3)
#pragma unroll
    for (int k = 0; k < 4 / S; ++k) {
      double em[4];
      if (plain)
        s1_plain4<0>(bvp + 4 * S * k * 16, zp + 4 * S * k, cv, em);
      else
        s1_gen4<0>(bvp + 4 * S * k * 16, zp + 4 * S * k, cv, tq + 4 * S * k, t0 + 4 * S * k, fx, em);
      mx = s3max(mx, s3_tree_max(em));
#pragma unroll
      for (int q = 0; q < S; ++q) {
        if (myq == q) {
          if (plain) {
            s3_fold_plain<4>(em, smice, cm);
          } else {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (tq[4 * S * k + v] & 4u) {
                smice = dev::dadd(smice, cm);
                cm = 0.0;
              }
              cm = s3max(cm, em[v]);
            }
          }
        }
        if (S > 1) s3_handoff(smice, cm, q, S);
      }
    }
  }
  smice = dev::dadd(smice, cm);
#pragma unroll
  for (int o = 1; o < S; o <<= 1) mx = s3max(mx, __shfl_xor_sync(0xffffffffu, mx, o));  // order-free
  if (valid) {
    const size_t o = size_t(l) * a.ldc + a.cand_idx[c];
    a.out_sm[o] = smice;
    a.out_mx[o] = mx;
  }
  // the last slice CTA of a candidate group sums its candidates over the
  // scenarios (as score3: self-resetting counters, release/acquire at gpu scope)
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.grp_done + cgrp) : "memory");
    s_last = old == nsl - 1;
    if (s_last) a.grp_done[cgrp] = 0;
  }
  __syncthreads();
  if (s_last) {
    double* ssm = smd;                 // [GK][L]
    double* smx = smd + size_t(GK) * L;
    for (int i = tid; i < GK * L; i += P) {
      const int g = i / L, ls = i - g * L;
      const int cgc = cgrp * GK + g;
      if (cgc < g_count) {
        const size_t o = size_t(ls) * a.ldc + a.cand_idx[cgc];
        ssm[i] = __ldcg(a.out_sm + o);
        smx[i] = __ldcg(a.out_mx + o);
      }
    }
    __syncthreads();
    const int cgc = cgrp * GK + tid;
    if (tid < GK && cgc < g_count) {
      double sum = 0.0;
      bool feasible = true;
      for (int ls = 0; ls < L; ++ls) {  // ((0 + s_0) + s_1) + ... (reduce.cpp:221-242)
        sum = dev::dadd(sum, ssm[tid * L + ls]);
        feasible = feasible && !(smx[tid * L + ls] > a.e_bar);
      }
      a.out_cand[a.cand_idx[cgc]] = feasible ? sum : -1.0;
    }
  }
}

// work items of the |phi(r)| = 1 group: [0, grp_cta[1]) (candidate groups of
// GK x scenario slices), strided over a persistent grid
constexpr int s1_min_blocks(int P) { return P >= 256 ? 2 : 384 / P; }  // register budget: <= 170
template <int S, int GK>
__global__ void __launch_bounds__(S1Geom<S, GK>::P, s1_min_blocks(S1Geom<S, GK>::P)) score1_kernel(S3Args a) {
  extern __shared__ double sm_dyn[];
  int R = a.R, n1 = a.grp_start[2] - a.grp_start[1], items = a.grp_cta[1];
  if (a.st) {
    if (a.st->done) return;
    R = a.st->R;
    n1 = a.st->grp_start[2] - a.st->grp_start[1];
    items = a.st->grp_cta[1];
  }
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    s1_item<S, GK>(a, w, n1, R, sm_dyn);
    __syncthreads();  // shared memory is reused by the next item
  }
  if (a.tdbg && a.st && threadIdx.x == 0) atomicMax(a.tdbg + size_t(a.st->iter) * kTdbg + 15, globaltimer_ns());
}

}  // namespace
}  // namespace kronred::b200
