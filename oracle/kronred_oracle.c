/*
 * kronred_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the
 * product). Plain-C restatement of the reference's exhaustive-search network
 * reduction (Opti-KRON `kronred`, /root/reference/proj/src), written from the
 * reference's behaviour so the GPU path can be checked without the reference
 * build. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.
 *
 * Complex arithmetic uses C99 `double _Complex`, which GCC lowers exactly like
 * libstdc++'s std::complex<double>: products inline as (ac-bd, ad+bc),
 * quotients through libgcc __divdc3, |z| through cabs (= hypot). Compile with
 * -ffp-contract=off (no FMA contraction), as the reference's x86-64 build has
 * no FMA either. Parity is pinned bit-for-bit against the golden vectors the
 * unmodified reference wrote (tests/test_oracle.py).
 */
#include "kronred_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cx;

enum { E_SINGULAR = -1, E_VALIDATION = -2, E_NOMEM = -3 };

static int has(uint8_t m, int p) { return (m >> p) & 1; }

/* ---- 3x3 complex blocks (complex3.hpp:102-187) ---------------------------- */

typedef struct { cx m[9]; } mat3;
typedef struct { cx v[3]; } vec3;

/* Mat3c * Mat3c with the zero-skip of complex3.hpp:138-147. */
static mat3 mat_mul(const mat3* a, const mat3* b) {
  mat3 r;
  memset(&r, 0, sizeof r);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      const cx aik = a->m[i * 3 + k];
      if (aik == 0) continue;
      for (int j = 0; j < 3; ++j) r.m[i * 3 + j] += aik * b->m[k * 3 + j];
    }
  return r;
}

/* Mat3c * Vec3c, accumulation from +0 (complex3.hpp:148-153). */
static vec3 mat_vec(const mat3* a, const vec3* x) {
  vec3 r;
  memset(&r, 0, sizeof r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.v[i] += a->m[i * 3 + j] * x->v[j];
  return r;
}

static int mat_is_zero(const mat3* a) {
  for (int i = 0; i < 9; ++i)
    if (a->m[i] != 0) return 0;
  return 1;
}

static double mat_max_abs(const mat3* a) {
  double r = 0;
  for (int i = 0; i < 9; ++i) {
    const double v = cabs(a->m[i]);
    if (r < v) r = v; /* std::max(r, v) */
  }
  return r;
}

/* masked_inverse (complex3.cpp:9-61): Gauss-Jordan with partial pivoting on
 * the present-phase submatrix; |.| is cabs, ties keep the upper row. */
static int masked_inverse(const mat3* in, uint8_t mask, mat3* out, double* smallest,
                          double pivot_tol) {
  memset(out, 0, sizeof *out);
  *smallest = 0.0;
  int idx[3], k = 0;
  for (int p = 0; p < 3; ++p)
    if (has(mask, p)) idx[k++] = p;
  if (k == 0) return 1;
  cx a[3][3], inv[3][3];
  memset(inv, 0, sizeof inv);
  for (int i = 0; i < k; ++i) {
    inv[i][i] = 1.0;
    for (int j = 0; j < k; ++j) a[i][j] = in->m[idx[i] * 3 + idx[j]];
  }
  *smallest = INFINITY;
  for (int col = 0; col < k; ++col) {
    int piv = col;
    double best = cabs(a[col][col]);
    for (int r = col + 1; r < k; ++r) {
      const double m = cabs(a[r][col]);
      if (m > best) {
        best = m;
        piv = r;
      }
    }
    if (best < *smallest) *smallest = best;
    if (best <= pivot_tol) return 0;
    if (piv != col) {
      cx t[3];
      memcpy(t, a[piv], sizeof t);
      memcpy(a[piv], a[col], sizeof t);
      memcpy(a[col], t, sizeof t);
      memcpy(t, inv[piv], sizeof t);
      memcpy(inv[piv], inv[col], sizeof t);
      memcpy(inv[col], t, sizeof t);
    }
    const cx d = a[col][col];
    for (int j = 0; j < k; ++j) {
      a[col][j] /= d;
      inv[col][j] /= d;
    }
    for (int r = 0; r < k; ++r) {
      if (r == col) continue;
      const cx f = a[r][col];
      if (f == 0) continue;
      for (int j = 0; j < k; ++j) {
        a[r][j] -= f * a[col][j];
        inv[r][j] -= f * inv[col][j];
      }
    }
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) out->m[idx[i] * 3 + idx[j]] = inv[i][j];
  return 1;
}

/* ---- node-indexed block-sparse matrix (block_matrix.hpp:47-92) ------------ */
/* Dense table of block pointers; a row is visited in ascending column order,
 * which is std::map's iteration order in the reference. */

typedef struct {
  int n;
  mat3** b; /* [n*n], NULL = structurally absent */
} bmat;

static int bm_init(bmat* y, int n) {
  y->n = n;
  y->b = (mat3**)calloc((size_t)n * (size_t)n, sizeof(mat3*));
  return y->b ? 0 : E_NOMEM;
}

static void bm_free(bmat* y) {
  if (!y->b) return;
  for (size_t i = 0; i < (size_t)y->n * (size_t)y->n; ++i) free(y->b[i]);
  free(y->b);
  y->b = NULL;
}

/* block(i, j): created zero on first access. */
static mat3* bm_block(bmat* y, int i, int j) {
  mat3** p = &y->b[(size_t)i * (size_t)y->n + (size_t)j];
  if (!*p) *p = (mat3*)calloc(1, sizeof(mat3));
  return *p;
}

static const mat3* bm_find(const bmat* y, int i, int j) {
  return y->b[(size_t)i * (size_t)y->n + (size_t)j];
}

static void bm_erase(bmat* y, int i, int j) {
  mat3** p = &y->b[(size_t)i * (size_t)y->n + (size_t)j];
  free(*p);
  *p = NULL;
}

static int bm_copy(const bmat* src, bmat* dst) {
  if (bm_init(dst, src->n)) return E_NOMEM;
  for (size_t i = 0; i < (size_t)src->n * (size_t)src->n; ++i)
    if (src->b[i]) {
      dst->b[i] = (mat3*)malloc(sizeof(mat3));
      *dst->b[i] = *src->b[i];
    }
  return 0;
}

static double bm_max_abs(const bmat* y) {
  double m = 0;
  for (size_t i = 0; i < (size_t)y->n * (size_t)y->n; ++i)
    if (y->b[i]) {
      const double v = mat_max_abs(y->b[i]);
      if (m < v) m = v;
    }
  return m;
}

/* ---- admittance assembly (grid_model.cpp:215-272, io.cpp:138-165) --------- */

static mat3 masked(const mat3* a, uint8_t mr, uint8_t mc) {
  mat3 r;
  memset(&r, 0, sizeof r);
  for (int i = 0; i < 3; ++i) {
    if (!has(mr, i)) continue;
    for (int j = 0; j < 3; ++j)
      if (has(mc, j)) r.m[i * 3 + j] = a->m[i * 3 + j];
  }
  return r;
}

static mat3 load_block(const double* p) {
  mat3 r;
  for (int k = 0; k < 9; ++k) r.m[k] = CMPLX(p[2 * k], p[2 * k + 1]);
  return r;
}

static mat3 transpose(const mat3* a) {
  mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i * 3 + j] = a->m[j * 3 + i];
  return r;
}

static int assemble(const oracle_net* net, bmat* y) {
  const int n = net->n;
  if (bm_init(y, n)) return E_NOMEM;
  uint8_t* seen = (uint8_t*)calloc((size_t)n * (size_t)n, 1);
  if (!seen) return E_NOMEM;
  for (int b = 0; b < net->nb; ++b) {
    const int f = net->from[b], t = net->to[b];
    if (f < 0 || f >= n || t < 0 || t >= n) {
      free(seen);
      return E_VALIDATION;
    }
    const int lo = f < t ? f : t, hi = f < t ? t : f;
    if (seen[(size_t)lo * n + hi]) {
      free(seen);
      return E_VALIDATION; /* duplicate branch */
    }
    seen[(size_t)lo * n + hi] = 1;
    /* branch parse: y_block masked to the common phases, or masked z_block
     * inverted by masked_inverse (io.cpp:151-160); shunts masked to the
     * endpoint phases (io.cpp:161-164). */
    const uint8_t common = net->phases[f] & net->phases[t];
    mat3 raw = load_block(net->y + (size_t)b * 18);
    mat3 ys = masked(&raw, common, common);
    if (net->is_z && net->is_z[b]) {
      mat3 inv;
      double piv;
      if (!masked_inverse(&ys, common, &inv, &piv, 1e-13)) {
        free(seen);
        return E_VALIDATION;
      }
      ys = inv;
    }
    mat3 shf, sht;
    memset(&shf, 0, sizeof shf);
    memset(&sht, 0, sizeof sht);
    if (net->sh_from) {
      raw = load_block(net->sh_from + (size_t)b * 18);
      shf = masked(&raw, net->phases[f], net->phases[f]);
    }
    if (net->sh_to) {
      raw = load_block(net->sh_to + (size_t)b * 18);
      sht = masked(&raw, net->phases[t], net->phases[t]);
    }
    const mat3 yt = transpose(&ys);
    mat3* p;
    p = bm_block(y, f, t);
    for (int k = 0; k < 9; ++k) p->m[k] -= ys.m[k];
    p = bm_block(y, t, f);
    for (int k = 0; k < 9; ++k) p->m[k] -= yt.m[k];
    p = bm_block(y, f, f);
    for (int k = 0; k < 9; ++k) p->m[k] += ys.m[k];
    p = bm_block(y, t, t);
    for (int k = 0; k < 9; ++k) p->m[k] += yt.m[k];
    p = bm_block(y, f, f);
    for (int k = 0; k < 9; ++k) p->m[k] += shf.m[k];
    p = bm_block(y, t, t);
    for (int k = 0; k < 9; ++k) p->m[k] += sht.m[k];
  }
  free(seen);
  /* confine blocks to present phases */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      mat3* p = y->b[(size_t)i * n + j];
      if (p) *p = masked(p, net->phases[i], net->phases[j]);
    }
  /* a present non-slack phase needs a nonzero admittance row */
  for (int i = 0; i < n; ++i) {
    if (i == net->slack) continue;
    for (int ph = 0; ph < 3; ++ph) {
      if (!has(net->phases[i], ph)) continue;
      int nonzero = 0;
      for (int j = 0; j < n && !nonzero; ++j) {
        const mat3* p = bm_find(y, i, j);
        if (!p) continue;
        for (int c = 0; c < 3; ++c)
          if (p->m[ph * 3 + c] != 0) nonzero = 1;
      }
      if (!nonzero) return E_VALIDATION;
    }
  }
  /* prune_zero_blocks (block_matrix.cpp:21-30) */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const mat3* p = bm_find(y, i, j);
      if (p && mat_is_zero(p)) bm_erase(y, i, j);
    }
  return 0;
}

/* ---- block elimination (solver.cpp:20-118) -------------------------------- */

typedef struct {
  int node;
  mat3 from_elim; /* A[node][k] */
  mat3 to_elim;   /* A[k][node] */
} coupling;

typedef struct {
  int node;
  mat3 pinv;
  int ncoup;
  coupling* coup;
} step;

typedef struct {
  int n;
  int nsteps;
  step* steps;
  uint8_t* eliminated;
  bmat rem; /* remaining (Schur complement) rows */
} elim;

static void elim_free(elim* e) {
  for (int s = 0; s < e->nsteps; ++s) free(e->steps[s].coup);
  free(e->steps);
  free(e->eliminated);
  bm_free(&e->rem);
  memset(e, 0, sizeof *e);
}

/* Greedy minimum-degree (lowest id on ties) elimination of the flagged nodes,
 * Schur updates on every active neighbour pair. Returns 0, or -(k+1)-16 for a
 * singular present-phase pivot at node k. */
static int eliminate(const bmat* y, const uint8_t* phases, const uint8_t* to_elim, elim* e) {
  const int n = y->n;
  memset(e, 0, sizeof *e);
  e->n = n;
  if (bm_copy(y, &e->rem)) return E_NOMEM;
  bmat* w = &e->rem;
  e->eliminated = (uint8_t*)calloc((size_t)n, 1);
  int remaining = 0;
  for (int i = 0; i < n; ++i) remaining += to_elim[i] ? 1 : 0;
  e->steps = (step*)calloc((size_t)(remaining > 0 ? remaining : 1), sizeof(step));
  int* degree = (int*)calloc((size_t)n, sizeof(int));
  int* nb = (int*)malloc(sizeof(int) * (size_t)n);
  if (!e->eliminated || !e->steps || !degree || !nb) {
    free(degree);
    free(nb);
    return E_NOMEM;
  }
  for (int i = 0; i < n; ++i) {
    int d = 0;
    for (int j = 0; j < n; ++j)
      if (j != i && bm_find(w, i, j)) ++d;
    degree[i] = d;
  }
  double scale = bm_max_abs(y);
  if (scale < 1.0) scale = 1.0;
  const double pivot_floor = 1e-12 * scale;

  while (remaining > 0) {
    int k = -1, best = 0x7fffffff;
    for (int i = 0; i < n; ++i) {
      if (!to_elim[i] || e->eliminated[i]) continue;
      if (degree[i] < best) {
        best = degree[i];
        k = i;
      }
    }
    mat3 diag;
    memset(&diag, 0, sizeof diag);
    if (bm_find(w, k, k)) diag = *bm_find(w, k, k);
    step* st = &e->steps[e->nsteps];
    st->node = k;
    double pivot = 0;
    if (!masked_inverse(&diag, phases[k], &st->pinv, &pivot, pivot_floor)) {
      free(degree);
      free(nb);
      return -(k + 1) - 16;
    }
    int nc = 0;
    for (int j = 0; j < n; ++j)
      if (j != k && bm_find(w, k, j) && !e->eliminated[j]) nb[nc++] = j;
    st->coup = (coupling*)malloc(sizeof(coupling) * (size_t)(nc > 0 ? nc : 1));
    st->ncoup = nc;
    for (int c = 0; c < nc; ++c) {
      const int j = nb[c];
      st->coup[c].node = j;
      st->coup[c].to_elim = *bm_find(w, k, j);
      st->coup[c].from_elim = *bm_block(w, j, k);
    }
    for (int a = 0; a < nc; ++a) {
      const coupling* ci = &st->coup[a];
      const mat3 t = mat_mul(&ci->from_elim, &st->pinv);
      for (int b = 0; b < nc; ++b) {
        const coupling* cj = &st->coup[b];
        const int inserted = bm_find(w, ci->node, cj->node) == NULL;
        mat3* blk = bm_block(w, ci->node, cj->node);
        const mat3 upd = mat_mul(&t, &cj->to_elim);
        for (int q = 0; q < 9; ++q) blk->m[q] -= upd.m[q];
        if (inserted && ci->node != cj->node) ++degree[ci->node];
      }
      bm_erase(w, ci->node, k);
      --degree[ci->node];
    }
    for (int j = 0; j < n; ++j) bm_erase(w, k, j);
    e->eliminated[k] = 1;
    e->nsteps++;
    --remaining;
  }
  free(degree);
  free(nb);
  return 0;
}

/* solve_interior (solver.cpp:100-129): forward push, backward resolve. */
static void solve_interior(const elim* e, const cx* b, cx* x, cx* rhs, vec3* t) {
  const int n = e->n;
  memcpy(rhs, b, sizeof(cx) * 3 * (size_t)n);
  memset(t, 0, sizeof(vec3) * (size_t)n);
  for (int s = 0; s < e->nsteps; ++s) {
    const step* st = &e->steps[s];
    vec3 bk;
    for (int p = 0; p < 3; ++p) bk.v[p] = rhs[3 * st->node + p];
    const vec3 tk = mat_vec(&st->pinv, &bk);
    t[st->node] = tk;
    for (int c = 0; c < st->ncoup; ++c) {
      const vec3 upd = mat_vec(&st->coup[c].from_elim, &tk);
      for (int p = 0; p < 3; ++p) rhs[3 * st->coup[c].node + p] -= upd.v[p];
    }
  }
  for (int s = e->nsteps - 1; s >= 0; --s) {
    const step* st = &e->steps[s];
    vec3 acc;
    memset(&acc, 0, sizeof acc);
    for (int c = 0; c < st->ncoup; ++c) {
      vec3 xj;
      for (int p = 0; p < 3; ++p) xj.v[p] = x[3 * st->coup[c].node + p];
      const vec3 r = mat_vec(&st->coup[c].to_elim, &xj);
      for (int p = 0; p < 3; ++p) acc.v[p] += r.v[p];
    }
    const vec3 corr = mat_vec(&st->pinv, &acc);
    for (int p = 0; p < 3; ++p) x[3 * st->node + p] = t[st->node].v[p] - corr.v[p];
  }
}

/* ---- anchored solver (solver.cpp:149-167) --------------------------------- */

typedef struct {
  int n, slack;
  cx vs[3];
  elim e;
  cx* rhs;
  vec3* t;
  cx* v_zero;
} anchored;

static void anchored_free(anchored* a) {
  elim_free(&a->e);
  free(a->rhs);
  free(a->t);
  free(a->v_zero);
}

static void anchored_solve(const anchored* a, const cx* inj, cx* x) {
  memset(x, 0, sizeof(cx) * 3 * (size_t)a->n);
  for (int p = 0; p < 3; ++p) x[3 * a->slack + p] = a->vs[p];
  solve_interior(&a->e, inj, x, a->rhs, a->t);
}

static int anchored_init(anchored* a, const bmat* y, const uint8_t* phases, int slack,
                         const cx* vs) {
  memset(a, 0, sizeof *a);
  const int n = y->n;
  a->n = n;
  a->slack = slack;
  for (int p = 0; p < 3; ++p) a->vs[p] = vs[p];
  if (slack < 0 || slack >= n) return E_VALIDATION;
  uint8_t* te = (uint8_t*)malloc((size_t)n);
  for (int i = 0; i < n; ++i) te[i] = i != slack;
  int rc = eliminate(y, phases, te, &a->e);
  free(te);
  if (rc) return rc;
  a->rhs = (cx*)malloc(sizeof(cx) * 3 * (size_t)n);
  a->t = (vec3*)malloc(sizeof(vec3) * (size_t)n);
  a->v_zero = (cx*)malloc(sizeof(cx) * 3 * (size_t)n);
  cx* zero = (cx*)calloc(3 * (size_t)n, sizeof(cx));
  if (!a->rhs || !a->t || !a->v_zero || !zero) return E_NOMEM;
  anchored_solve(a, zero, a->v_zero);
  free(zero);
  return 0;
}

static void net_slack_voltage(const oracle_net* net, cx* vs) {
  for (int p = 0; p < 3; ++p) vs[p] = CMPLX(net->slack_v[2 * p], net->slack_v[2 * p + 1]);
}

int oracle_solve(const oracle_net* net, const double* inj, int32_t nrhs, double* out) {
  bmat y;
  int rc = assemble(net, &y);
  if (rc) {
    bm_free(&y);
    return rc;
  }
  anchored a;
  cx vs[3];
  net_slack_voltage(net, vs);
  rc = anchored_init(&a, &y, net->phases, net->slack, vs);
  if (rc == 0) {
    const size_t dim = 3 * (size_t)net->n;
    cx* b = (cx*)malloc(sizeof(cx) * dim);
    cx* x = (cx*)malloc(sizeof(cx) * dim);
    for (int r = 0; r < nrhs; ++r) {
      for (size_t t = 0; t < dim; ++t)
        b[t] = CMPLX(inj[(r * dim + t) * 2], inj[(r * dim + t) * 2 + 1]);
      anchored_solve(&a, b, x);
      for (size_t t = 0; t < dim; ++t) {
        out[(r * dim + t) * 2] = creal(x[t]);
        out[(r * dim + t) * 2 + 1] = cimag(x[t]);
      }
    }
    free(b);
    free(x);
  }
  anchored_free(&a);
  bm_free(&y);
  return rc;
}

/* ---- Kron reduction (kron.cpp:34-46, solver.cpp:131-147) ------------------ */

/* Eliminate `reduce` from Y; the Schur complement over the kept nodes (dense
 * compact table, ascending original ids) goes to *out. */
static int kron(const bmat* y, const uint8_t* phases, int nred, const int32_t* reduce,
                bmat* out, int32_t* kept_ids, int* nk) {
  const int n = y->n;
  uint8_t* te = (uint8_t*)calloc((size_t)n, 1);
  for (int i = 0; i < nred; ++i) {
    if (reduce[i] < 0 || reduce[i] >= n || te[reduce[i]]) {
      free(te);
      return E_VALIDATION;
    }
    te[reduce[i]] = 1;
  }
  elim e;
  int rc = eliminate(y, phases, te, &e);
  free(te);
  if (rc) {
    elim_free(&e);
    return rc;
  }
  int* pos = (int*)malloc(sizeof(int) * (size_t)n);
  int k = 0;
  for (int i = 0; i < n; ++i) {
    pos[i] = -1;
    if (!e.eliminated[i]) {
      pos[i] = k;
      kept_ids[k++] = i;
    }
  }
  *nk = k;
  bm_init(out, k);
  for (int i = 0; i < n; ++i) {
    if (e.eliminated[i]) continue;
    for (int j = 0; j < n; ++j) {
      const mat3* blk = bm_find(&e.rem, i, j);
      if (!blk || mat_is_zero(blk)) continue;
      *bm_block(out, pos[i], pos[j]) = *blk;
    }
  }
  free(pos);
  elim_free(&e);
  return 0;
}

int oracle_kron(const oracle_net* net, int32_t nred, const int32_t* reduce, int32_t* kept_ids,
                double* blocks, uint8_t* present) {
  bmat y, yk;
  memset(&yk, 0, sizeof yk);
  int rc = assemble(net, &y);
  int nk = 0;
  if (rc == 0) rc = kron(&y, net->phases, nred, reduce, &yk, kept_ids, &nk);
  if (rc == 0) {
    for (int i = 0; i < nk; ++i)
      for (int j = 0; j < nk; ++j) {
        const mat3* b = bm_find(&yk, i, j);
        present[(size_t)i * nk + j] = b != NULL;
        double* o = blocks + ((size_t)i * nk + j) * 18;
        for (int q = 0; q < 9; ++q) {
          o[2 * q] = b ? creal(b->m[q]) : 0.0;
          o[2 * q + 1] = b ? cimag(b->m[q]) : 0.0;
        }
      }
  }
  bm_free(&yk);
  bm_free(&y);
  return rc ? rc : nk;
}

/* ---- reduction loop (reduce.cpp:39-123, 194-451) -------------------------- */

typedef struct {
  int n, slack, L;
  int nsup;
  int* supernodes; /* ascending */
  int* sup;
  int* head; /* member list per super-node, insertion order */
  int* tail;
  int* next;
  uint8_t* lam; /* super-node adjacency, dense n*n */
  cx* iagg;     /* [L][3n] */
} state;

static void state_free(state* s) {
  free(s->supernodes);
  free(s->sup);
  free(s->head);
  free(s->tail);
  free(s->next);
  free(s->lam);
  free(s->iagg);
}

/* init_state (reduce.cpp:39-61) */
static int state_init(state* s, const oracle_net* net, int L, const cx* inj) {
  const int n = net->n;
  memset(s, 0, sizeof *s);
  s->n = n;
  s->slack = net->slack;
  s->L = L;
  s->nsup = n;
  s->supernodes = (int*)malloc(sizeof(int) * (size_t)n);
  s->sup = (int*)malloc(sizeof(int) * (size_t)n);
  s->head = (int*)malloc(sizeof(int) * (size_t)n);
  s->tail = (int*)malloc(sizeof(int) * (size_t)n);
  s->next = (int*)malloc(sizeof(int) * (size_t)n);
  s->lam = (uint8_t*)calloc((size_t)n * (size_t)n, 1);
  s->iagg = (cx*)malloc(sizeof(cx) * 3 * (size_t)n * (size_t)L);
  if (!s->supernodes || !s->sup || !s->head || !s->tail || !s->next || !s->lam || !s->iagg)
    return E_NOMEM;
  for (int i = 0; i < n; ++i) {
    s->supernodes[i] = i;
    s->sup[i] = i;
    s->head[i] = s->tail[i] = i;
    s->next[i] = -1;
  }
  for (int b = 0; b < net->nb; ++b) {
    const int f = net->from[b], t = net->to[b];
    s->lam[(size_t)f * n + t] = 1;
    s->lam[(size_t)t * n + f] = 1;
  }
  memcpy(s->iagg, inj, sizeof(cx) * 3 * (size_t)n * (size_t)L);
  return 0;
}

/* enumerate_candidates (reduce.cpp:63-73): super-nodes ascending, their
 * super-node neighbours ascending, r != slack, mask(r) subset of mask(s). */
static int enumerate(const state* st, const uint8_t* masks, int* cs, int* cr) {
  const int n = st->n;
  int c = 0;
  for (int a = 0; a < st->nsup; ++a) {
    const int s = st->supernodes[a];
    for (int r = 0; r < n; ++r) {
      if (!st->lam[(size_t)s * n + r] || r == st->slack) continue;
      if ((masks[r] & ~masks[s]) == 0) {
        cs[c] = s;
        cr[c] = r;
        ++c;
      }
    }
  }
  return c;
}

/* commit (reduce.cpp:299-344) */
static void commit(state* st, int s, int r) {
  const int n = st->n;
  for (int j = st->head[r]; j >= 0; j = st->next[j]) st->sup[j] = s;
  st->next[st->tail[s]] = st->head[r];
  st->tail[s] = st->tail[r];
  st->head[r] = st->tail[r] = -1;
  int a = 0;
  while (st->supernodes[a] != r) ++a;
  memmove(st->supernodes + a, st->supernodes + a + 1, sizeof(int) * (size_t)(st->nsup - a - 1));
  st->nsup--;
  st->lam[(size_t)s * n + r] = 0;
  for (int t = 0; t < n; ++t) {
    if (!st->lam[(size_t)r * n + t] || t == s) continue;
    st->lam[(size_t)t * n + r] = 0;
    st->lam[(size_t)t * n + s] = 1;
    st->lam[(size_t)s * n + t] = 1;
  }
  memset(st->lam + (size_t)r * n, 0, (size_t)n);
  for (int l = 0; l < st->L; ++l) {
    cx* inj = st->iagg + (size_t)l * 3 * n;
    for (int p = 0; p < 3; ++p) {
      inj[3 * s + p] += inj[3 * r + p];
      inj[3 * r + p] = 0;
    }
  }
}

typedef struct {
  double max_err, smice;
  int feasible;
} scen_score;

/* score_scenario (reduce.cpp:89-123): super-node voltages distributed to
 * cluster members; feasibility gated on the magnitude error; early exit. */
static scen_score score_scenario(const state* st, int s, int r, const double* vre,
                                 const double* vim, const double* mag, const double* hre,
                                 const double* him, const double* hmag, const uint8_t* masks,
                                 double e_bar, int complex_obj) {
  scen_score out = {0.0, 0.0, 1};
  for (int a = 0; a < st->nsup; ++a) {
    const int i = st->supernodes[a];
    if (i == r) continue;
    double cmax = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int cl = pass == 0 ? i : r;
      if (pass == 1 && i != s) break;
      for (int j = st->head[cl]; j >= 0; j = st->next[j]) {
        for (int p = 0; p < 3; ++p) {
          if (!has(masks[j], p)) continue;
          const size_t si = (size_t)(3 * i + p), sj = (size_t)(3 * j + p);
          const double em = fabs(mag[si] - hmag[sj]);
          if (em > out.max_err) out.max_err = em;
          double eo = em;
          if (complex_obj) {
            const double dr = vre[si] - hre[sj];
            const double di = vim[si] - him[sj];
            eo = sqrt(dr * dr + di * di);
          }
          if (eo > cmax) cmax = eo;
        }
      }
    }
    if (out.max_err > e_bar) {
      out.feasible = 0;
      return out;
    }
    out.smice += cmax;
  }
  return out;
}

typedef struct {
  double *re, *im;
} planar;

/* model_max_errors (reduce.cpp:490-550) for the clusters of `st`. */
static int model_errors(const bmat* y, const oracle_net* net, const state* st, int L,
                        const cx* inj0, const cx* volt, double* out) {
  const int n = net->n;
  int32_t* reduce = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* kept = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int nred = 0;
  for (int i = 0; i < n; ++i)
    if (st->sup[i] != i) reduce[nred++] = i;
  bmat yk;
  memset(&yk, 0, sizeof yk);
  int nk = 0;
  int rc = kron(y, net->phases, nred, reduce, &yk, kept, &nk);
  if (rc) {
    free(reduce);
    free(kept);
    bm_free(&yk);
    return rc;
  }
  int* pos = (int*)malloc(sizeof(int) * (size_t)n);
  uint8_t* kph = (uint8_t*)malloc((size_t)nk);
  for (int i = 0; i < n; ++i) pos[i] = -1;
  for (int p = 0; p < nk; ++p) {
    pos[kept[p]] = p;
    kph[p] = net->phases[kept[p]];
  }
  cx vs[3];
  net_slack_voltage(net, vs);
  anchored a;
  rc = anchored_init(&a, &yk, kph, pos[net->slack], vs);
  if (rc == 0) {
    /* clusters: super-nodes ascending, members sorted ascending */
    int* assigned = (int*)malloc(sizeof(int) * (size_t)n);
    for (int j = 0; j < n; ++j) assigned[j] = pos[st->sup[j]];
    cx* ik = (cx*)malloc(sizeof(cx) * 3 * (size_t)nk);
    cx* vk = (cx*)malloc(sizeof(cx) * 3 * (size_t)nk);
    for (int l = 0; l < L; ++l) {
      const cx* sc = inj0 + (size_t)l * 3 * n;
      const cx* vv = volt + (size_t)l * 3 * n;
      memset(ik, 0, sizeof(cx) * 3 * (size_t)nk);
      for (int q = 0; q < nk; ++q) {
        const int i = kept[q];
        for (int j = 0; j < n; ++j) {
          if (st->sup[j] != i) continue;
          for (int p = 0; p < 3; ++p) ik[3 * q + p] += sc[3 * j + p];
        }
      }
      anchored_solve(&a, ik, vk);
      double err = 0;
      for (int j = 0; j < n; ++j) {
        const int pj = assigned[j];
        for (int p = 0; p < 3; ++p) {
          if (!has(net->phases[j], p)) continue;
          const double e = fabs(cabs(vk[3 * pj + p]) - cabs(vv[3 * j + p]));
          if (err < e) err = e;
        }
      }
      out[l] = err;
    }
    free(assigned);
    free(ik);
    free(vk);
  }
  anchored_free(&a);
  free(pos);
  free(kph);
  free(reduce);
  free(kept);
  bm_free(&yk);
  return rc;
}

int oracle_run(const oracle_net* net, int32_t L, const double* inj_in, double e_bar,
               int32_t objective, double target, int32_t has_target, int32_t cap, int32_t* out_s,
               int32_t* out_r, double* out_smice, double* out_maxerr, int32_t* out_nsup,
               int32_t* out_cands, double* out_final, int32_t score_iters, int32_t score_cap,
               int32_t* sc_iter, int32_t* sc_s, int32_t* sc_r, int32_t* sc_feas, double* sc_smice,
               double* sc_maxerr, int32_t* nscores) {
  const int n = net->n;
  const size_t dim = 3 * (size_t)n;
  if (!(e_bar >= 0)) return E_VALIDATION;
  if (has_target && !(target >= 0 && target <= 1)) return E_VALIDATION;
  if (L <= 0) return E_VALIDATION;
  if (nscores) *nscores = 0;
  bmat y;
  int rc = assemble(net, &y);
  if (rc) {
    bm_free(&y);
    return rc;
  }
  cx vs[3];
  net_slack_voltage(net, vs);
  anchored a;
  rc = anchored_init(&a, &y, net->phases, net->slack, vs);
  if (rc) {
    anchored_free(&a);
    bm_free(&y);
    return rc;
  }
  /* scenario_from_currents (scenario.cpp:22-50): slack rows and absent phases
   * zeroed, voltages = anchored solve */
  cx* inj = (cx*)malloc(sizeof(cx) * dim * (size_t)L);
  cx* volt = (cx*)malloc(sizeof(cx) * dim * (size_t)L);
  for (int l = 0; l < L; ++l) {
    for (size_t t = 0; t < dim; ++t) {
      const int node = (int)(t / 3), p = (int)(t % 3);
      cx v = CMPLX(inj_in[(l * dim + t) * 2], inj_in[(l * dim + t) * 2 + 1]);
      if (node == net->slack || !has(net->phases[node], p)) v = 0;
      inj[l * dim + t] = v;
    }
    anchored_solve(&a, inj + l * dim, volt + l * dim);
  }
  /* DeltaCache (reduce.cpp:249-294): V-hat planar + magnitude, base, Z */
  double* hre = (double*)malloc(sizeof(double) * dim * (size_t)L);
  double* him = (double*)malloc(sizeof(double) * dim * (size_t)L);
  double* hmag = (double*)malloc(sizeof(double) * dim * (size_t)L);
  double* bre = (double*)malloc(sizeof(double) * dim * (size_t)L);
  double* bim = (double*)malloc(sizeof(double) * dim * (size_t)L);
  for (size_t t = 0; t < dim * (size_t)L; ++t) {
    hre[t] = creal(volt[t]);
    him[t] = cimag(volt[t]);
    hmag[t] = sqrt(hre[t] * hre[t] + him[t] * him[t]);
  }
  planar* z = (planar*)calloc(dim, sizeof(planar)); /* [node*3+p] */
  cx* unit = (cx*)calloc(dim, sizeof(cx));
  cx* resp = (cx*)malloc(sizeof(cx) * dim);
  cx* xb = (cx*)malloc(sizeof(cx) * dim);
  double* vre = (double*)malloc(sizeof(double) * dim);
  double* vim = (double*)malloc(sizeof(double) * dim);
  double* mag = (double*)malloc(sizeof(double) * dim);
  int* cs = (int*)malloc(sizeof(int) * (size_t)n * (size_t)n);
  int* cr = (int*)malloc(sizeof(int) * (size_t)n * (size_t)n);
  double* cand_smice = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  double* cand_err = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n * (size_t)L);
  uint8_t* cand_feas = (uint8_t*)malloc((size_t)n * (size_t)n);
  state st;
  rc = state_init(&st, net, L, inj);

  /* refresh_base (reduce.cpp:265-268) */
#define REFRESH_BASE()                                                  \
  for (int l = 0; l < L; ++l) {                                         \
    anchored_solve(&a, st.iagg + l * dim, xb);                          \
    for (size_t t = 0; t < dim; ++t) {                                  \
      bre[l * dim + t] = creal(xb[t]);                                  \
      bim[l * dim + t] = cimag(xb[t]);                                  \
    }                                                                   \
  }
  if (rc == 0) {
    REFRESH_BASE();
  }
  int iteration = 0;
  while (rc == 0) {
    if (has_target && (double)(n - st.nsup) / (double)n >= target) break;
    const int nc = enumerate(&st, net->phases, cs, cr);
    if (nc == 0) break;
    /* ensure_columns (reduce.cpp:270-289): unit response minus v0; columns
     * are deterministic, so each is computed once and kept */
    for (int c = 0; c < nc; ++c)
      for (int e = 0; e < 2; ++e) {
        const int node = e ? cr[c] : cs[c];
        for (int p = 0; p < 3; ++p) {
          if (!has(net->phases[node], p) || z[3 * node + p].re) continue;
          unit[3 * node + p] = 1.0;
          anchored_solve(&a, unit, resp);
          unit[3 * node + p] = 0;
          planar* col = &z[3 * node + p];
          col->re = (double*)malloc(sizeof(double) * dim);
          col->im = (double*)malloc(sizeof(double) * dim);
          for (size_t t = 0; t < dim; ++t) {
            const cx d = resp[t] - a.v_zero[t];
            col->re[t] = creal(d);
            col->im[t] = cimag(d);
          }
        }
      }
    /* evaluate_candidate_delta (reduce.cpp:194-244) */
    for (int c = 0; c < nc; ++c) {
      const int s = cs[c], r = cr[c];
      double* merr = cand_err + (size_t)c * L;
      for (int l = 0; l < L; ++l) merr[l] = 0.0;
      int feasible = 1;
      double smice = 0;
      for (int l = 0; l < L && feasible; ++l) {
        memcpy(vre, bre + l * dim, sizeof(double) * dim);
        memcpy(vim, bim + l * dim, sizeof(double) * dim);
        for (int p = 0; p < 3; ++p) {
          const cx cc = st.iagg[l * dim + 3 * r + p];
          if (cc == 0) continue;
          const planar* zs = &z[3 * s + p];
          const planar* zr = &z[3 * r + p];
          if (!zs->re || !zr->re) {
            rc = E_VALIDATION; /* missing response column for a loaded phase */
            break;
          }
          const double cre = creal(cc), cim = cimag(cc);
          /* axpy_diff (kernels/scalar.cpp): out += c * (p - q) */
          for (size_t t = 0; t < dim; ++t) {
            const double dr = zs->re[t] - zr->re[t];
            const double di = zs->im[t] - zr->im[t];
            vre[t] += cre * dr - cim * di;
            vim[t] += cre * di + cim * dr;
          }
        }
        if (rc) break;
        for (size_t t = 0; t < dim; ++t) mag[t] = sqrt(vre[t] * vre[t] + vim[t] * vim[t]);
        const scen_score ss =
            score_scenario(&st, s, r, vre, vim, mag, hre + l * dim, him + l * dim,
                           hmag + l * dim, net->phases, e_bar, objective == 1);
        merr[l] = ss.max_err;
        feasible = ss.feasible;
        smice += ss.smice;
      }
      if (rc) break;
      cand_feas[c] = (uint8_t)feasible;
      cand_smice[c] = feasible ? smice : INFINITY;
      if (iteration < score_iters && nscores && *nscores < score_cap) {
        const int k = (*nscores)++;
        sc_iter[k] = iteration + 1;
        sc_s[k] = s;
        sc_r[k] = r;
        sc_feas[k] = feasible;
        sc_smice[k] = cand_smice[c];
        for (int l = 0; l < L; ++l) sc_maxerr[(size_t)k * L + l] = merr[l];
      }
    }
    if (rc) break;
    /* strict < keeps the first minimum (reduce.cpp:397-404) */
    int best = -1;
    for (int c = 0; c < nc; ++c) {
      if (!cand_feas[c]) continue;
      if (best < 0 || cand_smice[c] < cand_smice[best]) best = c;
    }
    if (best < 0) break;
    commit(&st, cs[best], cr[best]);
    REFRESH_BASE();
    if (iteration < cap) {
      out_s[iteration] = cs[best];
      out_r[iteration] = cr[best];
      out_smice[iteration] = cand_smice[best];
      for (int l = 0; l < L; ++l) out_maxerr[(size_t)iteration * L + l] = cand_err[(size_t)best * L + l];
      out_nsup[iteration] = st.nsup;
      out_cands[iteration] = nc;
    }
    ++iteration;
  }
#undef REFRESH_BASE
  if (rc == 0 && out_final) rc = model_errors(&y, net, &st, L, inj, volt, out_final);

  for (size_t t = 0; t < dim; ++t) {
    free(z[t].re);
    free(z[t].im);
  }
  free(z);
  free(unit);
  free(resp);
  free(xb);
  free(vre);
  free(vim);
  free(mag);
  free(cs);
  free(cr);
  free(cand_smice);
  free(cand_err);
  free(cand_feas);
  free(hre);
  free(him);
  free(hmag);
  free(bre);
  free(bim);
  free(inj);
  free(volt);
  state_free(&st);
  anchored_free(&a);
  bm_free(&y);
  return rc ? rc : iteration;
}

void oracle_cdiv(const double* in, int32_t N, double* out) {
  for (int32_t i = 0; i < N; ++i) {
    const cx a = CMPLX(in[4 * i], in[4 * i + 1]);
    const cx b = CMPLX(in[4 * i + 2], in[4 * i + 3]);
    const cx q = a / b;
    out[2 * i] = creal(q);
    out[2 * i + 1] = cimag(q);
  }
}
