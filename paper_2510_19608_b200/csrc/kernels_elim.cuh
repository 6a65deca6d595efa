// K1f: level-scheduled block elimination executor and the 3x3 complex block
// arithmetic it needs (complex3.hpp:76-90, complex3.cpp:9-61, solver.cpp:20-117).
#pragma once

namespace kronred::b200 {
namespace {

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

// masked_inverse (complex3.cpp:9-61): Gauss-Jordan with partial pivoting on
// the K x K present-phase submatrix, compiled per K so the work arrays stay in
// registers (the row swap is a predicated exchange with every candidate row).
// Pivot magnitudes use hypot (glibc cabs on the host); they only select
// pivots / gate singularity. Divisions are the __divdc3 replica.
template <unsigned MASK>
__device__ __forceinline__ bool masked_inverse_k(const C2 in[9], C2 out[9], double tol, double& smallest) {
  constexpr int K = int((MASK & 1u) + ((MASK >> 1) & 1u) + ((MASK >> 2) & 1u));
  // present phases, ascending (compile-time: every index below is static)
  constexpr int i0 = (MASK & 1u) ? 0 : ((MASK & 2u) ? 1 : 2);
  constexpr int i1 = K < 2 ? 0 : ((MASK & 1u) ? ((MASK & 2u) ? 1 : 2) : 2);
  constexpr int idx[3] = {i0, i1, 2};
  C2 a[K][K], inv[K][K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      a[i][j] = in[idx[i] * 3 + idx[j]];
      inv[i][j] = i == j ? C2{1.0, 0.0} : C2{0.0, 0.0};
    }
  smallest = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
  for (int col = 0; col < K; ++col) {
    int piv = col;
    double best = cabs_dev(a[col][col]);
#pragma unroll
    for (int r = col + 1; r < K; ++r) {
      const double m = cabs_dev(a[r][col]);
      if (m > best) {
        best = m;
        piv = r;
      }
    }
    smallest = fmin(smallest, best);
    if (best <= tol) return false;
#pragma unroll
    for (int r = col + 1; r < K; ++r)
      if (piv == r)
#pragma unroll
        for (int j = 0; j < K; ++j) {
          C2 t = a[r][j];
          a[r][j] = a[col][j];
          a[col][j] = t;
          t = inv[r][j];
          inv[r][j] = inv[col][j];
          inv[col][j] = t;
        }
    const C2 d = a[col][col];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      a[col][j] = dev::cdiv(a[col][j], d);
      inv[col][j] = dev::cdiv(inv[col][j], d);
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (r == col) continue;
      const C2 f = a[r][col];
      if (dev::cis0(f)) continue;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        a[r][j] = dev::csub(a[r][j], dev::cmul(f, a[col][j]));
        inv[r][j] = dev::csub(inv[r][j], dev::cmul(f, inv[col][j]));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) out[idx[i] * 3 + idx[j]] = inv[i][j];
  return true;
}

__device__ bool masked_inverse(const C2 in[9], unsigned mask, C2 out[9], double tol, double& smallest) {
#pragma unroll
  for (int e = 0; e < 9; ++e) out[e] = {0.0, 0.0};
  smallest = 0.0;
  switch (mask & 7u) {
    case 1: return masked_inverse_k<1>(in, out, tol, smallest);
    case 2: return masked_inverse_k<2>(in, out, tol, smallest);
    case 3: return masked_inverse_k<3>(in, out, tol, smallest);
    case 4: return masked_inverse_k<4>(in, out, tol, smallest);
    case 5: return masked_inverse_k<5>(in, out, tol, smallest);
    case 6: return masked_inverse_k<6>(in, out, tol, smallest);
    case 7: return masked_inverse_k<7>(in, out, tol, smallest);
    default: return true;  // nothing present: the pseudo-inverse of 0 is 0
  }
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

#ifndef ELIM_THREADS  // threads of the single-CTA level executor (register budget 65536 / ELIM_THREADS)
#define ELIM_THREADS 256
#endif
__global__ void __launch_bounds__(ELIM_THREADS) elim_factor_kernel(ElimDev e) {
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
}  // namespace
}  // namespace kronred::b200
