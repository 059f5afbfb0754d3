/*
 * tdw_oracle.c -- CPU restatement of the reference MOT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the CUDA
 * product path and the CPU baseline timed by bench.py (cpu_baseline, --impl
 * reference).  It is never linked into or called by paper_2111_05205_b200/.
 *
 * It restates, line for line in behaviour (not in code), the reference files:
 *   retarded_coeff_table      pkg/src/tdwavebem/elemint.py:89-186
 *     _edge_frames            elemint.py:36-57
 *     _clip_limits            elemint.py:60-76
 *     _masked_forms           elemint.py:79-86
 *     closed-form bundles     _closed_forms.py (re-derived: oracle/closed_forms.h)
 *   mesh_stats / radii        mesh.py:64-75, 85-107
 *   compute_gamma_star        marching.py:67-69
 *   _arrival_sorted_pairs     marching.py:93-129
 *   build_retarded_matrices   marching.py:132-181  (lag CSR, no upper cutoff)
 *   TimeHistory sums          marching.py:205-242
 *   build_step_matrix + march marching.py:279-338  (sigma/tau form)
 * The sparse LU (scipy SuperLU) of the reference is replaced by Gauss-Seidel
 * iterated to round-off on the strictly diagonally dominant step matrix
 * (cond(A) <= 1.51), followed by the reference's residual test.
 *
 * Parity is pinned against tests/golden/*.npz produced by running the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "closed_forms.h"

#define OR_OK 0
#define OR_INVALID 1
#define OR_SINGULAR 2
#define OR_RESIDUAL 3
#define OR_NOMEM 4

static const double Y_TOL = 1e-12; /* elemint.py:33 */

typedef void (*bundle_fn)(double, double, double, double, double*);

static bundle_fn uw_fn(int d) {
  return d == 1 ? tdw_uw_d1 : d == 2 ? tdw_uw_d2 : d == 3 ? tdw_uw_d3 : 0;
}
static bundle_fn bm_fn(int d) {
  return d == 1 ? tdw_bm_d1 : d == 2 ? tdw_bm_d2 : d == 3 ? tdw_bm_d3 : 0;
}

static inline double ipow(double v, int e) {
  double r = 1.0;
  for (int k = 0; k < e; ++k) r *= v;
  return r;
}

static inline double clipd(double a, double lo, double hi) {
  /* np.clip(a, lo, hi) == minimum(maximum(a, lo), hi) */
  double t = a > lo ? a : lo;
  return t < hi ? t : hi;
}

/* One (P, triangle ABC, s) triple -> (U, W) or (Ubar, Wbar).
 * kind 0 = "uw", 1 = "bm".  Follows elemint.py:116-186. */
static void coeff_one(const double* P, const double* A, const double* B, const double* C,
                      const double* ez, double s, int d, double K, int kind,
                      const double* nx, double* out0, double* out1) {
  const double* V1[3] = {A, B, C};
  const double* V2[3] = {B, C, A};
  double zs = (P[0] - A[0]) * ez[0] + (P[1] - A[1]) * ez[1] + (P[2] - A[2]) * ez[2];
  double O[3] = {P[0] - zs * ez[0], P[1] - zs * ez[1], P[2] - zs * ez[2]};
  double x1[3], x2[3], y[3], elen[3], xh[3][3], yh[3][3];
  for (int e = 0; e < 3; ++e) {
    double ev[3] = {V2[e][0] - V1[e][0], V2[e][1] - V1[e][1], V2[e][2] - V1[e][2]};
    elen[e] = sqrt(ev[0] * ev[0] + ev[1] * ev[1] + ev[2] * ev[2]);
    for (int k = 0; k < 3; ++k) xh[e][k] = ev[k] / elen[e];
    yh[e][0] = ez[1] * xh[e][2] - ez[2] * xh[e][1];
    yh[e][1] = ez[2] * xh[e][0] - ez[0] * xh[e][2];
    yh[e][2] = ez[0] * xh[e][1] - ez[1] * xh[e][0];
    double rel[3] = {V1[e][0] - O[0], V1[e][1] - O[1], V1[e][2] - O[2]};
    x1[e] = rel[0] * xh[e][0] + rel[1] * xh[e][1] + rel[2] * xh[e][2];
    x2[e] = x1[e] + elen[e];
    y[e] = rel[0] * yh[e][0] + rel[1] * yh[e][1] + rel[2] * yh[e][2];
  }
  double za = fabs(zs);
  double emax = elen[0];
  if (elen[1] > emax) emax = elen[1];
  if (elen[2] > emax) emax = elen[2];
  double zscale = emax + fabs(zs);
  double sgn = zs > 1e-12 * zscale ? 1.0 : -1.0;
  double nx3 = 0.0;
  if (kind == 1) nx3 = nx[0] * ez[0] + nx[1] * ez[1] + nx[2] * ez[2];

  double acc0 = 0.0, acc1 = 0.0;
  for (int e = 0; e < 3; ++e) {
    double scale = elen[e] + za;
    int alive = (fabs(y[e]) > Y_TOL * scale) && (s > za);
    double xc2 = s * s - y[e] * y[e] - za * za;
    int has = xc2 > 0.0;
    double xc = sqrt(has ? xc2 : 0.0);
    double xlo = clipd(x1[e], -xc, xc), xhi = clipd(x2[e], -xc, xc);
    int fmask = has && (xhi > xlo) && alive;
    int m1 = fmask && (x1[e] > -xc) && (x1[e] < xc);
    int m2 = fmask && (x2[e] > -xc) && (x2[e] < xc);
    double datan = 0.0, pw = 0.0;
    if (alive) {
      datan = atan(x2[e] / y[e]) - atan(x1[e] / y[e]);
      pw = s - za;
    }
    double t0, t1;
    if (kind == 0) {
      double lo[2] = {0, 0}, hi[2] = {0, 0};
      if (fmask) {
        uw_fn(d)(xlo, y[e], za, s, lo);
        uw_fn(d)(xhi, y[e], za, s, hi);
      }
      double a0 = -ipow(pw, d + 1) / (d + 1) * datan;
      double az = sgn * ipow(pw, d) * datan;
      t0 = a0 + hi[0] - lo[0];
      t1 = az + sgn * (hi[1] - lo[1]);
    } else {
      double lo[8] = {0}, hi[8] = {0};
      if (fmask) {
        bm_fn(d)(xlo, y[e], za, s, lo);
        bm_fn(d)(xhi, y[e], za, s, hi);
      }
      if (!m1) { lo[0] = 0.0; lo[1] = 0.0; }
      if (!m2) { hi[0] = 0.0; hi[1] = 0.0; }
      double n1 = nx[0] * xh[e][0] + nx[1] * xh[e][1] + nx[2] * xh[e][2];
      double n2 = nx[0] * yh[e][0] + nx[1] * yh[e][1] + nx[2] * yh[e][2];
      double pwd = ipow(pw, d);
      double az = sgn * pwd * datan;
      double as = -pwd * datan;
      double azz = d > 1 ? -d * ipow(pw, d - 1) * datan : -(pw > 0.0 ? 1.0 : 0.0) * datan;
      double azs = -sgn * azz;
      double dPx = lo[0] - hi[0];
      double dPy = -(hi[2] - lo[2]);
      double dz = az + sgn * (hi[3] - lo[3]);
      double ds = as + hi[4] - lo[4];
      double dzPx = sgn * (lo[1] - hi[1]);
      double dzPy = -sgn * (hi[5] - lo[5]);
      double dzz = azz + hi[6] - lo[6];
      double dzs = azs + sgn * (hi[7] - lo[7]);
      t0 = n1 * dPx + n2 * dPy + nx3 * dz - ds;
      t1 = n1 * dzPx + n2 * dzPy + nx3 * dzz - dzs;
    }
    acc0 += t0;
    acc1 += t1;
  }
  if (kind == 0) {
    *out0 = K * acc0;
    *out1 = -K * acc1;
  } else {
    *out0 = K * acc0;
    *out1 = -K * acc1;
  }
}

static double kfac(int d, double c, double dt) {
  double cd = c * dt, p = 1.0;
  for (int k = 0; k < d; ++k) p *= cd;
  return 1.0 / (4.0 * M_PI * p);
}

/* retarded_coeff_table (elemint.py:89).  Arrays are C-contiguous (n,3) / (n,). */
int oracle_coeff_table(int64_t n, const double* P, const double* A, const double* B,
                       const double* C, const double* ez, const double* s, int d, double c,
                       double dt, int kind, const double* nx, double* out0, double* out1) {
  if (d < 1 || d > 3) return OR_INVALID;
  if (kind != 0 && kind != 1) return OR_INVALID;
  if (kind == 1 && !nx) return OR_INVALID;
  double K = kfac(d, c, dt);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    coeff_one(P + 3 * t, A + 3 * t, B + 3 * t, C + 3 * t, ez + 3 * t, s[t], d, K, kind,
              kind == 1 ? nx + 3 * t : 0, out0 + t, out1 + t);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* mesh-derived quantities (mesh.py:42-75)                                    */
typedef struct {
  int ns;
  const double* verts;
  const int64_t* tris;
  double *v0, *v1, *v2, *nrm, *cen, *rad;
} omesh;

static int mesh_build(omesh* m, int ns, const double* verts, const int64_t* tris) {
  m->ns = ns;
  m->verts = verts;
  m->tris = tris;
  m->v0 = malloc(sizeof(double) * 3 * ns);
  m->v1 = malloc(sizeof(double) * 3 * ns);
  m->v2 = malloc(sizeof(double) * 3 * ns);
  m->nrm = malloc(sizeof(double) * 3 * ns);
  m->cen = malloc(sizeof(double) * 3 * ns);
  m->rad = malloc(sizeof(double) * ns);
  if (!m->v0 || !m->v1 || !m->v2 || !m->nrm || !m->cen || !m->rad) return OR_NOMEM;
  for (int e = 0; e < ns; ++e) {
    const double* a = verts + 3 * tris[3 * e];
    const double* b = verts + 3 * tris[3 * e + 1];
    const double* cc = verts + 3 * tris[3 * e + 2];
    double u[3], w[3], cr[3];
    for (int k = 0; k < 3; ++k) {
      m->v0[3 * e + k] = a[k];
      m->v1[3 * e + k] = b[k];
      m->v2[3 * e + k] = cc[k];
      u[k] = b[k] - a[k];
      w[k] = cc[k] - a[k];
    }
    cr[0] = u[1] * w[2] - u[2] * w[1];
    cr[1] = u[2] * w[0] - u[0] * w[2];
    cr[2] = u[0] * w[1] - u[1] * w[0];
    double nn = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    double r = 0.0;
    for (int k = 0; k < 3; ++k) {
      m->nrm[3 * e + k] = cr[k] / nn;
      m->cen[3 * e + k] = (a[k] + b[k] + cc[k]) / 3.0;
    }
    const double* vv[3] = {a, b, cc};
    for (int q = 0; q < 3; ++q) {
      double dx = vv[q][0] - m->cen[3 * e], dy = vv[q][1] - m->cen[3 * e + 1],
             dz = vv[q][2] - m->cen[3 * e + 2];
      double dd = sqrt(dx * dx + dy * dy + dz * dz);
      if (dd > r) r = dd;
    }
    m->rad[e] = r;
  }
  return OR_OK;
}

static void mesh_free(omesh* m) {
  free(m->v0); free(m->v1); free(m->v2); free(m->nrm); free(m->cen); free(m->rad);
}

/* max vertex diameter over used vertices (mesh.py:85-107) */
double oracle_max_diameter(int nv, const double* verts, int ns, const int64_t* tris) {
  char* used = calloc(nv, 1);
  for (int64_t k = 0; k < 3 * (int64_t)ns; ++k) used[tris[k]] = 1;
  double dmax = 0.0;
#pragma omp parallel for reduction(max : dmax) schedule(dynamic, 16)
  for (int i = 0; i < nv; ++i) {
    if (!used[i]) continue;
    for (int j = 0; j < nv; ++j) {
      if (!used[j]) continue;
      double dx = verts[3 * i] - verts[3 * j], dy = verts[3 * i + 1] - verts[3 * j + 1],
             dz = verts[3 * i + 2] - verts[3 * j + 2];
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 > dmax) dmax = d2;
    }
  }
  free(used);
  return sqrt(dmax);
}

int oracle_gamma_star(int nv, const double* verts, int ns, const int64_t* tris, int d, double c,
                      double dt) {
  double diam = oracle_max_diameter(nv, verts, ns, tris);
  return (int)ceil(diam / (c * dt)) + d + 1;
}

/* ------------------------------------------------------------------------ */
/* Lag CSR store, the reference's RetardedMatrixSet (marching.py:72-90, 132-181):
 * for each lag g = 1..G a CSR matrix over the stored rows holding U^(g), W^(g)
 * of every pair already arrived by g (arrival a_ij <= g, marching.py:108-110),
 * columns increasing within a row, no upper cutoff. */
typedef struct {
  int nr, G;
  int64_t** rowptr; /* [G][nr+1] */
  int32_t** col;    /* [G][nnz_g] */
  double **U, **W;  /* [G][nnz_g] */
  int64_t nvals;
} lagstore;

static int arrival_of(const omesh* m, int i, int j, double c, double dt) {
  double dx = m->cen[3 * i] - m->cen[3 * j], dy = m->cen[3 * i + 1] - m->cen[3 * j + 1],
         dz = m->cen[3 * i + 2] - m->cen[3 * j + 2];
  double dist = sqrt(dx * dx + dy * dy + dz * dz);
  dist = dist - m->rad[j];
  if (dist < 0.0) dist = 0.0;
  int a = (int)ceil(dist / (c * dt)) - 1;
  return a > 1 ? a : 1;
}

static void lag_free(lagstore* L) {
  for (int g = 0; g < L->G; ++g) {
    if (L->rowptr) free(L->rowptr[g]);
    if (L->col) free(L->col[g]);
    if (L->U) free(L->U[g]);
    if (L->W) free(L->W[g]);
  }
  free(L->rowptr); free(L->col); free(L->U); free(L->W);
}

static int lag_build_list(lagstore* L, const omesh* m, int row_lo, int row_hi,
                          const int* rowlist, int G, int bie, int d, double c, double dt) {
  int nr = row_hi - row_lo, ns = m->ns;
#define ROW_OF(r) (rowlist ? rowlist[r] : row_lo + (r))
  L->nr = nr;
  L->G = G;
  L->nvals = 0;
  L->rowptr = calloc(G, sizeof(int64_t*));
  L->col = calloc(G, sizeof(int32_t*));
  L->U = calloc(G, sizeof(double*));
  L->W = calloc(G, sizeof(double*));
  if (!L->rowptr || !L->col || !L->U || !L->W) return OR_NOMEM;
  /* per row: arrivals of all columns (int8 would do; int keeps it simple) */
  int* arr = malloc(sizeof(int) * (size_t)nr * ns);
  if (!arr) return OR_NOMEM;
#pragma omp parallel for schedule(dynamic, 8)
  for (int r = 0; r < nr; ++r)
    for (int j = 0; j < ns; ++j) arr[(size_t)r * ns + j] = arrival_of(m, ROW_OF(r), j, c, dt);
  for (int g = 1; g <= G; ++g) {
    int64_t* rp = calloc(nr + 1, sizeof(int64_t));
    if (!rp) { free(arr); return OR_NOMEM; }
#pragma omp parallel for schedule(static)
    for (int r = 0; r < nr; ++r) {
      int64_t k = 0;
      for (int j = 0; j < ns; ++j) k += arr[(size_t)r * ns + j] <= g;
      rp[r + 1] = k;
    }
    for (int r = 0; r < nr; ++r) rp[r + 1] += rp[r];
    L->rowptr[g - 1] = rp;
    L->col[g - 1] = malloc(sizeof(int32_t) * (rp[nr] ? rp[nr] : 1));
    L->U[g - 1] = malloc(sizeof(double) * (rp[nr] ? rp[nr] : 1));
    L->W[g - 1] = malloc(sizeof(double) * (rp[nr] ? rp[nr] : 1));
    if (!L->col[g - 1] || !L->U[g - 1] || !L->W[g - 1]) { free(arr); return OR_NOMEM; }
    L->nvals += rp[nr];
  }
  double K = kfac(d, c, dt);
  int kind = bie == 1 ? 1 : 0;
#pragma omp parallel for schedule(dynamic, 4)
  for (int r = 0; r < nr; ++r) {
    int i = ROW_OF(r);
    double nxi[3] = {-m->nrm[3 * i], -m->nrm[3 * i + 1], -m->nrm[3 * i + 2]};
    int64_t* pos = malloc(sizeof(int64_t) * G);
    for (int g = 0; g < G; ++g) pos[g] = L->rowptr[g][r];
    for (int j = 0; j < ns; ++j) {
      int a = arr[(size_t)r * ns + j];
      for (int g = a; g <= G; ++g) {
        double s = (double)g * c * dt;
        int64_t q = pos[g - 1]++;
        L->col[g - 1][q] = j;
        coeff_one(m->cen + 3 * i, m->v0 + 3 * j, m->v1 + 3 * j, m->v2 + 3 * j, m->nrm + 3 * j, s,
                  d, K, kind, nxi, L->U[g - 1] + q, L->W[g - 1] + q);
      }
    }
    free(pos);
  }
  free(arr);
  return OR_OK;
#undef ROW_OF
}

static int lag_build(lagstore* L, const omesh* m, int row_lo, int row_hi, int G, int bie, int d,
                     double c, double dt) {
  return lag_build_list(L, m, row_lo, row_hi, 0, G, bie, d, c, dt);
}

/* b_r (+)= U_g tau - W_g sigma over the stored rows (one lag): the reference's
 * b += U[g-1] @ tau - W[g-1] @ sig (marching.py:320-327). */
static void lag_apply(const lagstore* L, int g, const double* tau, const double* sig, double* b,
                      int first) {
  const int nr = L->nr;
  const int64_t* rp = L->rowptr[g - 1];
  const int32_t* col = L->col[g - 1];
  const double* U = L->U[g - 1];
  const double* W = L->W[g - 1];
#pragma omp parallel for schedule(static) if (rp[nr] >= 32768)
  for (int r = 0; r < nr; ++r) {
    double su = 0.0, sw = 0.0;
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
      su += U[p] * tau[col[p]];
      sw += W[p] * sig[col[p]];
    }
    b[r] = first ? (su - sw) : b[r] + (su - sw);
  }
}

static double weights_d[4][5] = {
    {0}, {1.0, -2.0, 1.0}, {0.5, -1.5, 1.5, -0.5}, {1.0 / 6, -2.0 / 3, 1.0, -2.0 / 3, 1.0 / 6}};

/* The reference's march (marching.py:292-338) as a stateful marcher, so that
 * bench.py can time bounded chunks of the full-problem loop.  All history
 * arrays are (nt-1, ns); u_known / q_known are the Greville samples
 * (marching.py:258-276) and are copied. */
typedef struct {
  omesh m;
  lagstore L;
  int ns, nt, d, window, gstar, n_lags, alpha, status, n_steps, rc;
  double threshold;
  const double* phi_in;
  double *phi, *uk, *qk, *u, *q, *tau, *sig, *rhs;
  double *aval, *adiag, *b, *x, *tt, *st, *tw, *sw;
} omarcher;

static void marcher_free(omarcher* M) {
  if (!M) return;
  free(M->phi); free(M->uk); free(M->qk); free(M->u); free(M->q); free(M->tau); free(M->sig);
  free(M->rhs); free(M->aval); free(M->adiag); free(M->b); free(M->x); free(M->tt); free(M->st);
  free(M->tw); free(M->sw);
  lag_free(&M->L);
  mesh_free(&M->m);
  free(M);
}

static double* dup_arr(const double* src, size_t n) {
  double* p = malloc(sizeof(double) * (n ? n : 1));
  if (p && src) memcpy(p, src, sizeof(double) * n);
  else if (p) memset(p, 0, sizeof(double) * n);
  return p;
}

/* reset the history to the start of the loop (alpha = 1) */
void oracle_marcher_reset(omarcher* M) {
  size_t n = (size_t)(M->nt - 1) * M->ns;
  memset(M->u, 0, sizeof(double) * n);
  memset(M->q, 0, sizeof(double) * n);
  memset(M->tau, 0, sizeof(double) * n);
  memset(M->sig, 0, sizeof(double) * n);
  if (M->rhs) memset(M->rhs, 0, sizeof(double) * n);
  M->alpha = 1;
  M->status = 0;
  M->n_steps = 0;
  M->rc = OR_OK;
}

int oracle_marcher_create(int nv, const double* verts, int ns, const int64_t* tris,
                          const double* phi, int bie, int d, double c, double dt, int nt,
                          int window, double threshold, const double* u_known,
                          const double* q_known, int want_rhs, omarcher** out,
                          double* t_asm_out) {
  *out = 0;
  if (d < 1 || d > 3 || nt < 2) return OR_INVALID;
  omarcher* M = calloc(1, sizeof(omarcher));
  if (!M) return OR_NOMEM;
  int rc = mesh_build(&M->m, ns, verts, tris);
  if (rc) { marcher_free(M); return rc; }
  M->ns = ns; M->nt = nt; M->d = d; M->window = window; M->threshold = threshold;
  M->gstar = oracle_gamma_star(nv, verts, ns, tris, d, c, dt);
  M->n_lags = window ? (M->gstar < nt - 1 ? M->gstar : nt - 1) : nt - 1;
#ifdef _OPENMP
  double t0 = omp_get_wtime();
#endif
  rc = lag_build(&M->L, &M->m, 0, ns, M->n_lags, bie, d, c, dt);
#ifdef _OPENMP
  if (t_asm_out) *t_asm_out = omp_get_wtime() - t0;
#endif
  if (rc) { marcher_free(M); return rc; }
  size_t n = (size_t)(nt - 1) * ns;
  M->phi = dup_arr(phi, ns);
  M->uk = dup_arr(u_known, n);
  M->qk = dup_arr(q_known, n);
  M->u = dup_arr(0, n); M->q = dup_arr(0, n); M->tau = dup_arr(0, n); M->sig = dup_arr(0, n);
  M->rhs = want_rhs ? dup_arr(0, n) : 0;
  M->b = dup_arr(0, ns); M->x = dup_arr(0, ns); M->tt = dup_arr(0, ns); M->st = dup_arr(0, ns);
  M->tw = dup_arr(0, ns); M->sw = dup_arr(0, ns);
  if (!M->phi || !M->uk || !M->qk || !M->u || !M->q || !M->tau || !M->sig || !M->b || !M->x ||
      !M->tt || !M->st || !M->tw || !M->sw || (want_rhs && !M->rhs)) {
    marcher_free(M);
    return OR_NOMEM;
  }
  /* step matrix A = w0 (W1 phi - U1 (1 - phi)) (marching.py:279-289), lag-1 CSR pattern */
  const double w0 = weights_d[d][0];
  const int64_t* arow = M->L.rowptr[0];
  const int32_t* acol = M->L.col[0];
  M->aval = malloc(sizeof(double) * (arow[ns] + 1));
  M->adiag = malloc(sizeof(double) * ns);
  if (!M->aval || !M->adiag) { marcher_free(M); return OR_NOMEM; }
  int singular = 0;
  for (int i = 0; i < ns; ++i) {
    M->adiag[i] = 0.0;
    for (int64_t k = arow[i]; k < arow[i + 1]; ++k) {
      int j = acol[k];
      M->aval[k] = w0 * (M->L.W[0][k] * phi[j] - M->L.U[0][k] * (1.0 - phi[j]));
      if (j == i) M->adiag[i] = M->aval[k];
    }
    if (M->adiag[i] == 0.0) singular = 1;
  }
  if (singular) { marcher_free(M); return OR_SINGULAR; }
  oracle_marcher_reset(M);
  *out = M;
  return OR_OK;
}

/* Advance up to n_adv steps (stops at the end of the loop, a blow-up or an
 * error).  *done = 1 when the loop is over.  *t_loop = wall seconds. */
int oracle_marcher_run(omarcher* M, int n_adv, int* done, double* t_loop) {
  const int ns = M->ns, nt = M->nt, d = M->d, gstar = M->gstar, n_lags = M->n_lags;
  const int window = M->window;
  const double* w = weights_d[d];
  const double w0 = w[0];
  const lagstore* L = &M->L;
  const int64_t* arow = L->rowptr[0];
  const int32_t* acol = L->col[0];
  const double *aval = M->aval, *adiag = M->adiag, *phi = M->phi;
  double *u = M->u, *q = M->q, *tau = M->tau, *sig = M->sig, *b = M->b, *x = M->x;
  double *tt = M->tt, *st = M->st, *tw = M->tw, *sw = M->sw;
#ifdef _OPENMP
  double t0 = omp_get_wtime();
#endif
  int rc = M->rc;
  for (int it_adv = 0; it_adv < n_adv && rc == OR_OK && M->status == 0 && M->alpha < nt;
       ++it_adv) {
    const int alpha = M->alpha;
    int beta0 = alpha - 1;
    int beta_star = alpha - gstar;
    const double* uk = M->uk + (size_t)beta0 * ns;
    const double* qk = M->qk + (size_t)beta0 * ns;
    /* tilde sums (marching.py:227-237) */
    for (int j = 0; j < ns; ++j) {
      tt[j] = w0 * qk[j] * phi[j];
      st[j] = w0 * uk[j] * (1.0 - phi[j]);
    }
    int kt = d + 1 < beta0 ? d + 1 : beta0;
    for (int k = 1; k <= kt; ++k)
      for (int j = 0; j < ns; ++j) {
        tt[j] += w[k] * q[(size_t)(beta0 - k) * ns + j];
        st[j] += w[k] * u[(size_t)(beta0 - k) * ns + j];
      }
    lag_apply(L, 1, tt, st, b, 1);
    int gmax = alpha < n_lags ? alpha : n_lags;
    for (int g = 2; g <= gmax; ++g) {
      int beta = alpha - g;
      const double *tp, *sp;
      if (window && beta - beta_star <= d) {
        /* windowed_sums (marching.py:216-225) */
        int kmax = d + 1;
        if (beta - beta_star < kmax) kmax = beta - beta_star;
        if (beta < kmax) kmax = beta;
        for (int j = 0; j < ns; ++j) { tw[j] = 0.0; sw[j] = 0.0; }
        for (int k = 0; k <= kmax; ++k)
          for (int j = 0; j < ns; ++j) {
            tw[j] += w[k] * q[(size_t)(beta - k) * ns + j];
            sw[j] += w[k] * u[(size_t)(beta - k) * ns + j];
          }
        tp = tw; sp = sw;
      } else {
        tp = tau + (size_t)beta * ns;
        sp = sig + (size_t)beta * ns;
      }
      lag_apply(L, g, tp, sp, b, 0);
    }
    if (M->rhs) memcpy(M->rhs + (size_t)beta0 * ns, b, sizeof(double) * ns);
    /* solve A x = b: Gauss-Seidel to round-off, then the reference residual test */
    double bn = 0.0;
    for (int i = 0; i < ns; ++i) { x[i] = b[i] / adiag[i]; bn += b[i] * b[i]; }
    bn = sqrt(bn);
    for (int it = 0; it < 200; ++it) {
      double dn = 0.0, xn = 0.0;
      for (int i = 0; i < ns; ++i) {
        double acc = b[i];
        for (int64_t k = arow[i]; k < arow[i + 1]; ++k)
          if (acol[k] != i) acc -= aval[k] * x[acol[k]];
        double xi = acc / adiag[i];
        dn += (xi - x[i]) * (xi - x[i]);
        xn += xi * xi;
        x[i] = xi;
      }
      if (dn <= 1e-34 * xn || xn == 0.0) break;
    }
    double rn = 0.0;
    for (int i = 0; i < ns; ++i) {
      double acc = -b[i];
      for (int64_t k = arow[i]; k < arow[i + 1]; ++k) acc += aval[k] * x[acol[k]];
      rn += acc * acc;
    }
    rn = sqrt(rn);
    if (rn > 1e-10 * (bn > 1e-300 ? bn : 1e-300)) { rc = OR_RESIDUAL; break; }
    /* finalize_step (marching.py:239-242) */
    double xmax = 0.0;
    for (int j = 0; j < ns; ++j) {
      size_t o = (size_t)beta0 * ns + j;
      u[o] = phi[j] == 1.0 ? x[j] : uk[j];
      q[o] = phi[j] == 1.0 ? qk[j] : x[j];
      if (fabs(x[j]) > xmax) xmax = fabs(x[j]);
    }
    int ks = d + 1 < beta0 ? d + 1 : beta0;
    for (int j = 0; j < ns; ++j) {
      double ta = 0.0, sa = 0.0;
      for (int k = 0; k <= ks; ++k) {
        ta += w[k] * q[(size_t)(beta0 - k) * ns + j];
        sa += w[k] * u[(size_t)(beta0 - k) * ns + j];
      }
      tau[(size_t)beta0 * ns + j] = ta;
      sig[(size_t)beta0 * ns + j] = sa;
    }
    M->n_steps = alpha;
    M->alpha = alpha + 1;
    if (xmax > M->threshold) M->status = 1;
  }
  M->rc = rc;
#ifdef _OPENMP
  if (t_loop) *t_loop = omp_get_wtime() - t0;
#endif
  if (done) *done = (rc != OR_OK || M->status != 0 || M->alpha >= nt);
  return rc;
}

/* copy the history out (any pointer may be NULL) */
int oracle_marcher_get(const omarcher* M, double* u, double* q, double* tau, double* sig,
                       double* rhs_trace, int* n_steps, int* status) {
  size_t n = sizeof(double) * (size_t)(M->nt - 1) * M->ns;
  if (u) memcpy(u, M->u, n);
  if (q) memcpy(q, M->q, n);
  if (tau) memcpy(tau, M->tau, n);
  if (sig) memcpy(sig, M->sig, n);
  if (rhs_trace && M->rhs) memcpy(rhs_trace, M->rhs, n);
  if (n_steps) *n_steps = M->n_steps;
  if (status) *status = M->status;
  return M->rc;
}

void oracle_marcher_destroy(omarcher* M) { marcher_free(M); }

/* Full march (marching.py:292-338): create + run to the end + copy out. */
int oracle_march(int nv, const double* verts, int ns, const int64_t* tris, const double* phi,
                 int bie, int d, double c, double dt, int nt, int window, double threshold,
                 const double* u_known, const double* q_known, double* u, double* q, double* tau,
                 double* sig, double* rhs_trace, int* n_steps, int* status, double* t_asm_out) {
  omarcher* M = 0;
  int rc = oracle_marcher_create(nv, verts, ns, tris, phi, bie, d, c, dt, nt, window, threshold,
                                 u_known, q_known, rhs_trace != 0, &M, t_asm_out);
  if (rc) return rc;
  int done = 0;
  rc = oracle_marcher_run(M, nt, &done, 0);
  oracle_marcher_get(M, u, q, tau, sig, rhs_trace, n_steps, status);
  oracle_marcher_destroy(M);
  return rc;
}

/* Right-hand sides of the reference's march for a sample of rows, recomputed
 * from a GIVEN history (u, q, tau, sigma: (nt-1, ns), e.g. the GPU's), in the
 * reference's sigma/tau lag-CSR form (marching.py:315-327) restricted to those
 * rows.  For each (row, step) pair k: b[k] = b_row^alpha, and
 * res[k] = (A x^{alpha-1})_row - b[k] with A the lag-1 step matrix
 * (marching.py:279-289) and x the history's unknown density at beta0.
 * rows/alphas: n_rows rows x n_alpha steps (alpha >= 1), outputs row-major. */
int oracle_rhs_rows(int nv, const double* verts, int ns, const int64_t* tris, const double* phi,
                    int bie, int d, double c, double dt, int nt, int window, int n_rows,
                    const int* rows, int n_alpha, const int* alphas, const double* u_known,
                    const double* q_known, const double* u, const double* q, const double* tau,
                    const double* sig, double* b_out, double* res_out) {
  if (d < 1 || d > 3 || nt < 2) return OR_INVALID;
  omesh m;
  int rc = mesh_build(&m, ns, verts, tris);
  if (rc) return rc;
  int gstar = oracle_gamma_star(nv, verts, ns, tris, d, c, dt);
  int n_lags = window ? (gstar < nt - 1 ? gstar : nt - 1) : nt - 1;
  const double* w = weights_d[d];
  const double w0 = w[0];
  lagstore L;
  memset(&L, 0, sizeof(L));
  rc = lag_build_list(&L, &m, 0, n_rows, rows, n_lags, bie, d, c, dt);
  if (rc) { lag_free(&L); mesh_free(&m); return rc; }
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int r = 0; r < n_rows; ++r)
    for (int a = 0; a < n_alpha; ++a) {
      const int alpha = alphas[a];
      const int beta0 = alpha - 1, beta_star = alpha - gstar;
      const int gmax = alpha < n_lags ? alpha : n_lags;
      double bsum = 0.0;
      for (int g = 1; g <= gmax; ++g) {
        const int64_t* rp = L.rowptr[g - 1] + r;
        const int32_t* col = L.col[g - 1];
        const int beta = alpha - g;
        double su = 0.0, sw = 0.0;
        for (int64_t p = rp[0]; p < rp[1]; ++p) {
          const int j = col[p];
          double tj, sj;
          if (g == 1) { /* tilde sums (marching.py:227-237) */
            tj = w0 * q_known[(size_t)beta0 * ns + j] * phi[j];
            sj = w0 * u_known[(size_t)beta0 * ns + j] * (1.0 - phi[j]);
            int kt = d + 1 < beta0 ? d + 1 : beta0;
            for (int k = 1; k <= kt; ++k) {
              tj += w[k] * q[(size_t)(beta0 - k) * ns + j];
              sj += w[k] * u[(size_t)(beta0 - k) * ns + j];
            }
          } else if (window && beta - beta_star <= d) { /* windowed_sums (:216-225) */
            int kmax = d + 1;
            if (beta - beta_star < kmax) kmax = beta - beta_star;
            if (beta < kmax) kmax = beta;
            tj = 0.0; sj = 0.0;
            for (int k = 0; k <= kmax; ++k) {
              tj += w[k] * q[(size_t)(beta - k) * ns + j];
              sj += w[k] * u[(size_t)(beta - k) * ns + j];
            }
          } else {
            tj = tau[(size_t)beta * ns + j];
            sj = sig[(size_t)beta * ns + j];
          }
          su += L.U[g - 1][p] * tj;
          sw += L.W[g - 1][p] * sj;
        }
        bsum += su - sw;
      }
      b_out[(size_t)r * n_alpha + a] = bsum;
      /* residual of the lag-1 row against the history's solution at beta0 */
      double ax = 0.0;
      const int64_t* rp = L.rowptr[0] + r;
      for (int64_t p = rp[0]; p < rp[1]; ++p) {
        const int j = L.col[0][p];
        const double aij = w0 * (L.W[0][p] * phi[j] - L.U[0][p] * (1.0 - phi[j]));
        const double xj = phi[j] == 1.0 ? u[(size_t)beta0 * ns + j] : q[(size_t)beta0 * ns + j];
        ax += aij * xj;
      }
      if (res_out) res_out[(size_t)r * n_alpha + a] = ax - bsum;
    }
  lag_free(&L);
  mesh_free(&m);
  return rc;
}

/* Bounded CPU-baseline sample (bench.py cpu_baseline / --impl reference):
 * assemble the lag CSR for rows [row_lo, row_hi) and run n_steps of the
 * per-step history SpMVs for those rows over synthetic densities.  Returns the
 * assembly and loop wall seconds and the number of stored lag-CSR triples. */
int oracle_sample(int nv, const double* verts, int ns, const int64_t* tris, int bie, int d,
                  double c, double dt, int nt, int row_lo, int row_hi, int n_steps,
                  double* t_asm, double* t_loop, int64_t* n_triples) {
  omesh m;
  int rc = mesh_build(&m, ns, verts, tris);
  if (rc) return rc;
  int gstar = oracle_gamma_star(nv, verts, ns, tris, d, c, dt);
  int n_lags = gstar < nt - 1 ? gstar : nt - 1;
  lagstore L;
  memset(&L, 0, sizeof(L));
  int nr = row_hi - row_lo;
#ifdef _OPENMP
  double t0 = omp_get_wtime();
#endif
  rc = lag_build(&L, &m, row_lo, row_hi, n_lags, bie, d, c, dt);
#ifdef _OPENMP
  *t_asm = omp_get_wtime() - t0;
#endif
  *n_triples = L.nvals;
  double* hist = malloc(sizeof(double) * 2 * (size_t)ns * (n_lags + 1));
  for (size_t k = 0; k < 2 * (size_t)ns * (n_lags + 1); ++k) hist[k] = 1e-3 * (double)(k % 97);
  double* b = malloc(sizeof(double) * (nr > 0 ? nr : 1));
#ifdef _OPENMP
  t0 = omp_get_wtime();
#endif
  for (int st = 0; st < n_steps && rc == OR_OK; ++st) {
    for (int g = 1; g <= n_lags; ++g) {
      const double* tp = hist + (size_t)(2 * g) * ns / 2;
      const double* sp = hist + (size_t)(2 * g + 1) * ns / 2;
      lag_apply(&L, g, tp, sp, b, g == 1);
    }
  }
#ifdef _OPENMP
  *t_loop = omp_get_wtime() - t0;
#endif
  free(hist); free(b);
  lag_free(&L);
  mesh_free(&m);
  return rc;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
