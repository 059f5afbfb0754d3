// assemble.cu -- banded kappa-combined coefficient store + lag-1 step matrix.
//
// Replaces marching.build_retarded_matrices (marching.py:132-181) and
// build_step_matrix (marching.py:279-289).  Instead of the reference's per-lag
// CSR of U^(g) over every arrived pair (no upper cutoff, marching.py:76-81),
// the store holds the kappa-combined coefficients
//     V^(gamma)_ij = sum_{kappa=0}^{d+1} w^kappa U^(gamma-kappa)_ij
// (and the same for W) only on each pair's band [glo, ghi], where
//     glo = max(arrival_ij, floor(r_min/(c dt)) + 1)       (first lag the wavefront touches E_j)
//     ghi = min(cap, floor(r_max/(c dt)) + 1 + d)          (after that V is identically zero:
//                                                          U is a degree-d polynomial in gamma
//                                                          once the wavefront has passed E_j and
//                                                          the w^kappa annihilate it)
// arrival_ij is the reference's conservative lag (marching.py:108-110); U^(g)
// for g < arrival_ij is zero exactly as in the reference's lag CSR.  The history
// sum b = sum_g (U^(g) tau - W^(g) sigma) (marching.py:320-327) is then the
// banded convolution sum_gamma (V_U^(gamma) q - V_W^(gamma) u).
//
// Layout: rows in Morton order, columns cut in
// 32-wide J-tiles.  A segment = (row, J-tile) = 32 pairs = one warp; its pairs
// are sorted by band length (descending) and their coefficients are stored
// k-major ("jagged"): entry (k, lane) at segoff + sum_{k'<k} n_k' + lane where
// n_k = #pairs with len > k.  The convolution warp therefore reads 16 B per
// lane per k fully coalesced with no padding.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cmath>

#include "coeff.cuh"
#include "tdw_impl.cuh"

namespace tdw {

#define FULLMASK 0xffffffffu

struct Elem {
  double v0[3], v1[3], v2[3], n[3], c[3], rad;
};

__device__ __forceinline__ void load_elem(const double* __restrict__ E, int j, Elem& e) {
  const double* p = E + (size_t)j * TDW_ELEM_STRIDE;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e.v0[k] = p[k];
    e.v1[k] = p[3 + k];
    e.v2[k] = p[6 + k];
    e.n[k] = p[9 + k];
    e.c[k] = p[12 + k];
  }
  e.rad = p[15];
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// exact point-triangle distance (closest point by Voronoi region)
__device__ double point_triangle_distance(const double* p, const double* a, const double* b,
                                          const double* c) {
  double ab[3], ac[3], ap[3], q[3];
  for (int k = 0; k < 3; ++k) {
    ab[k] = b[k] - a[k];
    ac[k] = c[k] - a[k];
    ap[k] = p[k] - a[k];
  }
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    for (int k = 0; k < 3; ++k) q[k] = a[k];
  } else {
    double bp[3] = {p[0] - b[0], p[1] - b[1], p[2] - b[2]};
    double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
    double cp[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
    double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    double vc = d1 * d4 - d3 * d2, vb = d5 * d2 - d1 * d6, va = d3 * d6 - d5 * d4;
    if (d3 >= 0.0 && d4 <= d3) {
      for (int k = 0; k < 3; ++k) q[k] = b[k];
    } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
      double v = d1 / (d1 - d3);
      for (int k = 0; k < 3; ++k) q[k] = a[k] + v * ab[k];
    } else if (d6 >= 0.0 && d5 <= d6) {
      for (int k = 0; k < 3; ++k) q[k] = c[k];
    } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
      double w = d2 / (d2 - d6);
      for (int k = 0; k < 3; ++k) q[k] = a[k] + w * ac[k];
    } else if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
      double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
      for (int k = 0; k < 3; ++k) q[k] = b[k] + w * (c[k] - b[k]);
    } else {
      double den = 1.0 / (va + vb + vc);
      double v = vb * den, w = vc * den;
      for (int k = 0; k < 3; ++k) q[k] = a[k] + ab[k] * v + ac[k] * w;
    }
  }
  double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
  return sqrt(dx * dx + dy * dy + dz * dz);
}

// conservative arrival lag of the reference (marching.py:108-110)
__device__ __forceinline__ int arrival_lag(const double* ci, const Elem& ej, double cdt) {
  double dx = ci[0] - ej.c[0], dy = ci[1] - ej.c[1], dz = ci[2] - ej.c[2];
  double dist = sqrt(dx * dx + dy * dy + dz * dz);
  dist = fmax(dist - ej.rad, 0.0);
  int a = (int)ceil(dist / cdt) - 1;
  return a > 1 ? a : 1;
}

struct Band {
  int glo, ghi, arr;
};

__device__ __forceinline__ Band pair_band(const double* ci, const Elem& ej, double cdt, int d,
                                          int cap) {
  Band b;
  b.arr = arrival_lag(ci, ej, cdt);
  double rmin = point_triangle_distance(ci, ej.v0, ej.v1, ej.v2);
  double r0 = sqrt((ci[0] - ej.v0[0]) * (ci[0] - ej.v0[0]) + (ci[1] - ej.v0[1]) * (ci[1] - ej.v0[1]) +
                   (ci[2] - ej.v0[2]) * (ci[2] - ej.v0[2]));
  double r1 = sqrt((ci[0] - ej.v1[0]) * (ci[0] - ej.v1[0]) + (ci[1] - ej.v1[1]) * (ci[1] - ej.v1[1]) +
                   (ci[2] - ej.v1[2]) * (ci[2] - ej.v1[2]));
  double r2 = sqrt((ci[0] - ej.v2[0]) * (ci[0] - ej.v2[0]) + (ci[1] - ej.v2[1]) * (ci[1] - ej.v2[1]) +
                   (ci[2] - ej.v2[2]) * (ci[2] - ej.v2[2]));
  double rmax = fmax(fmax(r0, r1), r2);
  // first lag with c*g*dt > r_min (with a relative guard: an extra noise-level
  // entry is harmless, a missing one is not)
  int g0 = (int)floor(rmin / cdt * (1.0 - 1e-10)) + 1;
  b.glo = max(max(g0, b.arr), 1);
  int gfull = (int)floor(rmax / cdt * (1.0 + 1e-10)) + 1;
  b.ghi = min(cap, gfull + d);
  return b;
}

__device__ __forceinline__ void bspline_weights(int d, double* w) {
  if (d == 1) { w[0] = 1.0; w[1] = -2.0; w[2] = 1.0; }
  if (d == 2) { w[0] = 0.5; w[1] = -1.5; w[2] = 1.5; w[3] = -0.5; }
  if (d == 3) { w[0] = 1.0 / 6.0; w[1] = -(2.0 / 3.0); w[2] = 1.0; w[3] = -(2.0 / 3.0); w[4] = 1.0 / 6.0; }
}

// Pair restrictions of the store:
//  * FMM near field: only pairs whose leaf cells are adjacent (fmm_tree.py:163-177);
//  * build_retarded_matrices(pairs=(ii, jj)) (marching.py:132-181): only the listed
//    pairs -- per row a sorted column list (internal order), binary search.
__device__ __forceinline__ bool pair_allowed(const int* leafc, const int* pptr, const int* pcol, int i, int j) {
  if (pptr) {
    int lo = pptr[i], hi = pptr[i + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int c = pcol[mid];
      if (c == j) return true;
      if (c < j) lo = mid + 1; else hi = mid;
    }
    return false;
  }
  if (!leafc) return true;
  const int a = leafc[i], b = leafc[j];
  const int dx = (a & 1023) - (b & 1023), dy = ((a >> 10) & 1023) - ((b >> 10) & 1023),
            dz = ((a >> 20) & 1023) - ((b >> 20) & 1023);
  return dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1;
}

struct AsmArgs {
  const double* elem;
  const int* leafc;                    // packed leaf-cell coords (FMM near field) or null
  const int* pptr;                     // pairs= restriction: [ns+1] row pointers or null
  const int* pcol;                     // sorted columns per row
  int split_lag2;                      // 1: lag 2..nsl+1 entries keep the known density only
  int nsl;                             // split lags
  int ns, row_lo, rows_loc, ntiles, d, cap;
  double c, dt, K;
  uint32_t* hdr;
  unsigned long long* segcount;  // count pass output / fill pass: segoff
  int2* unit;
  unsigned long long* n_evals;
  unsigned long long* n_pairs;
  const double* phi;                   // internal order
  const unsigned long long* unit_off;  // byte offset of each unit in the store
  unsigned char* units;                // unit-major store (tdw_impl.cuh "unit layout")
  int* flags;
};

__global__ void __launch_bounds__(256) count_kernel(AsmArgs a) {
  const int lane = threadIdx.x & 31;
  const long long seg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nseg = (long long)a.rows_loc * a.ntiles;
  if (seg >= nseg) return;
  const int rloc = (int)(seg / a.ntiles), t = (int)(seg % a.ntiles);
  const int i = a.row_lo + rloc, j = t * TDW_TJ + lane;
  const double cdt = a.c * a.dt;
  int len = 0, glo = 0;
  bool any = false;
  if (i < a.ns && j < a.ns && pair_allowed(a.leafc, a.pptr, a.pcol, i, j)) {
    Elem ej;
    load_elem(a.elem, j, ej);
    const double* ci = a.elem + (size_t)i * TDW_ELEM_STRIDE + 12;
    Band b = pair_band(ci, ej, cdt, a.d, a.cap);
    any = b.ghi >= b.glo;
    if (any) {
      len = b.ghi - b.glo + 1;
      glo = b.glo;
    }
    if (len > 255) { atomicExch(&a.flags[3], 2); len = 255; }
  }
  // lane = column: the convolution's lanes then read one 512-byte row of the
  // [lag][column] history box (no shared-memory bank conflicts)
  a.hdr[seg * TDW_TJ + lane] = hdr_pack(lane, len, glo);
  const int lmax = __reduce_max_sync(FULLMASK, len);
  int tot = len, gmin = len ? glo : INT_MAX, gmax = len ? glo + len - 1 : -1, np = any ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tot += __shfl_xor_sync(FULLMASK, tot, o);
    np += __shfl_xor_sync(FULLMASK, np, o);
    gmin = min(gmin, __shfl_xor_sync(FULLMASK, gmin, o));
    gmax = max(gmax, __shfl_xor_sync(FULLMASK, gmax, o));
  }
  if (lane == 0) {
    a.segcount[seg] = (unsigned long long)tot | ((unsigned long long)lmax << TDW_SEG_LMAX_SHIFT);
    if (np) atomicAdd(a.n_pairs, (unsigned long long)np);
    if (tot) {
      int2* u = &a.unit[(rloc / TDW_TI) * a.ntiles + t];
      atomicMin(&u->x, gmin);
      atomicMax(&u->y, gmax);
    }
  }
}

// blocks per SM the register budget is sized for (spills accepted: latency-bound
// kernel, occupancy wins).  With the compact (not unrolled) closed forms, 4 blocks
// (128 registers) is best for every order: config 2 (d = 1) 37.1 ms (5 blocks:
// 38.2), config 3 (d = 2) 804 ms (3 blocks: 835, 5 blocks: 905)
#ifndef TDW_FILL_MINB
#define TDW_FILL_MINB(D) 4
#endif
template <int D, bool BM>
__global__ void __launch_bounds__(128, TDW_FILL_MINB(D)) fill_kernel(AsmArgs a) {
  const int lane = threadIdx.x & 31;
  const long long seg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nseg = (long long)a.rows_loc * a.ntiles;
  if (seg >= nseg) return;
  const int rloc = (int)(seg / a.ntiles), t = (int)(seg % a.ntiles);
  unsigned char* ub = a.units + a.unit_off[(size_t)(rloc / TDW_TI) * a.ntiles + t];
  const int r = rloc % TDW_TI;
  const unsigned coef_off = *(const uint32_t*)(ub + TDW_UNIT_LAG_OFF + 12);
  const int gmax = ((const int2*)(ub + TDW_UNIT_LAG_OFF))->y;
  int jl, len, rel;
  unit_hdr(ub, coef_off, gmax, r * TDW_TJ + lane, jl, len, rel);
  const int glo = gmax - rel;
  const int lmax = __reduce_max_sync(FULLMASK, len);
  if (lmax == 0) return;
  const int i = a.row_lo + rloc, j = t * TDW_TJ + jl;
  double2* coef = (double2*)(ub + coef_off);
  const unsigned long long base = ((const uint32_t*)ub)[r];
  const double cdt = a.c * a.dt;
  double w[D + 2];
  bspline_weights(D, w);
  double ru[D + 2], rw[D + 2];
#pragma unroll
  for (int k = 0; k < D + 2; ++k) { ru[k] = 0.0; rw[k] = 0.0; }
  PairGeom g;
  long long nev = 0;
  if (len > 0) {
    Elem ej;
    load_elem(a.elem, j, ej);
    const double* pi = a.elem + (size_t)i * TDW_ELEM_STRIDE;
    double ci[3] = {pi[12], pi[13], pi[14]};
    double nx[3] = {-pi[9], -pi[10], -pi[11]};  // BM operator normal (marching.py:168-173)
    pair_geom<BM>(ci, ej.v0, ej.v1, ej.v2, ej.n, nx, g);
    const int arr = arrival_lag(ci, ej, cdt);
    const int gfirst = max(max(arr, 1), glo - (D + 1));
    for (int gg = gfirst; gg < glo; ++gg) {
      double u, v;
      coeff_eval<D, BM>(g, (double)gg * a.c * a.dt, a.K, u, v);
#pragma unroll
      for (int k = D + 1; k > 0; --k) { ru[k] = ru[k - 1]; rw[k] = rw[k - 1]; }
      ru[0] = u;
      rw[0] = v;
      ++nev;
    }
  }
  unsigned long long off = base;
  for (int k = 0; k < lmax; ++k) {
    const unsigned m = __ballot_sync(FULLMASK, len > k);
    if (len > k) {
      const int gg = glo + k;
      double u, v;
      coeff_eval<D, BM>(g, (double)gg * a.c * a.dt, a.K, u, v);
#pragma unroll
      for (int q = D + 1; q > 0; --q) { ru[q] = ru[q - 1]; rw[q] = rw[q - 1]; }
      ru[0] = u;
      rw[0] = v;
      ++nev;
      double vu = 0.0, vw = 0.0;
#pragma unroll
      for (int q = 0; q < D + 2; ++q) {
        vu += w[q] * ru[q];
        vw += w[q] * rw[q];
      }
      if (a.split_lag2 && gg >= 2 && gg <= a.nsl + 1) {
        // lags 2..nsl+1: keep only the coefficient of the KNOWN density of
        // element j (q if phi_j = 1, u if phi_j = 0); the unknown one is applied
        // through the near structure after each solve, so the convolution pass
        // of steps alpha..alpha+kb-1 waits only for the solve of step
        // alpha-1-overlap (nsl = kb + overlap - 1).
        const double pj = a.phi[j];
        vu = pj == 1.0 ? vu : 0.0;
        vw = pj == 1.0 ? 0.0 : vw;
      }
      coef[off + __popc(m & ((1u << lane) - 1u))] = make_double2(vu, vw);
    }
    off += __popc(m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nev += __shfl_xor_sync(FULLMASK, nev, o);
  if (lane == 0) atomicAdd(a.n_evals, (unsigned long long)nev);
}

// bytes of every unit: header block + 16 B per band entry of its 32 segments;
// the header width (16 or 32 bit) follows from the unit's longest band and lag span
__global__ void unit_size_kernel(const unsigned long long* segcount, const uint32_t* hdr_tmp,
                                 const int2* unit, int ntiles, long long nunit, int force32,
                                 unsigned long long* unit_bytes, unsigned* unit_coef,
                                 unsigned long long* n_band) {
  const int lane = threadIdx.x & 31;
  const long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= nunit) return;
  const long long iblk = u / ntiles, t = u % ntiles;
  const long long sidx = (iblk * TDW_TI + lane) * ntiles + t;
  unsigned long long c = segcount[sidx] & TDW_SEG_COUNT_MASK;
  int lmax = (int)(segcount[sidx] >> TDW_SEG_LMAX_SHIFT);  // longest band of the segment
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(FULLMASK, c, o);
    lmax = max(lmax, __shfl_xor_sync(FULLMASK, lmax, o));
  }
  if (lane == 0) {
    const int2 g = unit[u];
    const int span = g.y >= g.x ? g.y - g.x : 0;
    const unsigned coef = (!force32 && lmax <= 31 && span <= 63) ? TDW_UNIT_COEF_OFF16 : TDW_UNIT_COEF_OFF;
    unit_coef[u] = coef;
    unit_bytes[u] = coef + 16ull * c;
    if (c) atomicAdd(n_band, c);
  }
}

// per-unit header block: segment offsets, lag range, the 32x32 pair headers
__global__ void unit_layout_kernel(const unsigned long long* segcount, const uint32_t* hdr_tmp,
                                   const int2* unit, const unsigned* unit_coef, int ntiles,
                                   long long nunit, const unsigned long long* unit_off,
                                   unsigned char* units, unsigned* max_rel) {
  const int lane = threadIdx.x & 31;
  const long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= nunit) return;
  const long long iblk = u / ntiles, t = u % ntiles;
  unsigned char* ub = units + unit_off[u];
  const unsigned c = (unsigned)(segcount[(iblk * TDW_TI + lane) * ntiles + t] & TDW_SEG_COUNT_MASK);
  unsigned x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(FULLMASK, x, o);
    if (lane >= o) x += y;
  }
  ((uint32_t*)ub)[lane] = x - c;  // exclusive prefix
  const int2 g = unit[u];
  const unsigned coef = unit_coef[u];
  if (lane == 0) {
    *(int2*)(ub + TDW_UNIT_LAG_OFF) = g;
    *(uint32_t*)(ub + TDW_UNIT_LAG_OFF + 8) = (uint32_t)(unit_off[u + 1] - unit_off[u]);
    *(uint32_t*)(ub + TDW_UNIT_LAG_OFF + 12) = coef;
  }
  const uint32_t* src = hdr_tmp + (iblk * TDW_TI * ntiles + t) * TDW_TJ + lane;
  if (coef == TDW_UNIT_COEF_OFF16) {
    uint16_t* h = (uint16_t*)(ub + TDW_UNIT_HDR_OFF);
    for (int r = 0; r < TDW_TI; ++r) {
      const uint32_t w = src[(size_t)r * ntiles * TDW_TJ];
      const int len = hdr_len(w);
      h[hdr16_index(r, lane)] = hdr16_pack(hdr_jl(w), len, len ? g.y - hdr_glo(w) : 0);
    }
  } else {
    uint32_t* h = (uint32_t*)(ub + TDW_UNIT_HDR_OFF);
    for (int r = 0; r < TDW_TI; ++r) h[r * TDW_TJ + lane] = src[(size_t)r * ntiles * TDW_TJ];
  }
  if (lane == 31) atomicMax(max_rel, x);
}

struct NearArgs {
  const double* elem;
  const int* leafc;
  const int* pptr;
  const int* pcol;
  int split_lag2, nsl;
  const double* phi;
  int ns, ntiles, d, cap;
  double c, dt, K;
  int* ncol;      // [TDW_NEAR_MAX][ns]
  double* nval;   // [kb][TDW_NEAR_MAX][ns]: coefficient of the unknown density at lag 2 + index
  int* acol;      // [TDW_ELL_MAX][ns]  lag-1 step matrix (pairs with V^(1))
  double* aval;   // [TDW_ELL_MAX][ns]
  double* adiag;  // [ns]
  int* flags;     // [4]: [2] max near width, [3] overflow
  int* ell_w;
  int* ncnt;      // [ns] near entries per row
  unsigned long long* bound_bits;
  unsigned long long* nnz;
  unsigned long long* n_near;
  unsigned long long* n_evals;
};

// Rows of the lag-1 step matrix and of the "unknown" coupling at the split lags
// g = 2..nsl+1, all rows (replicated on every rank).  With
// V^(g) = sum_kappa w^kappa U^(g-kappa) (U^(m) = 0 for m < max(1, arrival); zero
// outside the pair's band, as in the store):
//   A_ij     = V_W^(1) phi_j - V_U^(1) (1 - phi_j)      (build_step_matrix, marching.py:279-289)
//   N^g_ij   = -V_W^(g) if phi_j = 1 else V_U^(g)       (b_i^alpha += N^g_ij x_j^(alpha-g))
template <int D, bool BM>
__global__ void __launch_bounds__(128) near_kernel(NearArgs a) {
  const int lane = threadIdx.x & 31;
  const int i = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= a.ns) return;
  const double cdt = a.c * a.dt;
  double w[D + 2];
  bspline_weights(D, w);
  const double* pi = a.elem + (size_t)i * TDW_ELEM_STRIDE;
  double ci[3] = {pi[12], pi[13], pi[14]};
  double nx[3] = {-pi[9], -pi[10], -pi[11]};
  const int gtop = a.split_lag2 ? a.nsl + 1 : 1;  // highest split lag
  const size_t gstride = (size_t)TDW_NEAR_MAX * a.ns;
  int cnt = 0, acnt = 0;
  double diag = 0.0, offsum = 0.0;
  long long nev = 0;
  for (int t = 0; t < a.ntiles; ++t) {
    const int j = t * TDW_TJ + lane;
    Elem ej;
    Band b{0, -1, 1};
    bool cand = false;
    if (j < a.ns) {
      load_elem(a.elem, j, ej);
      double dx = ci[0] - ej.c[0], dy = ci[1] - ej.c[1], dz = ci[2] - ej.c[2];
      double dcc = sqrt(dx * dx + dy * dy + dz * dz);
      if (dcc - ej.rad <= (gtop + 1) * cdt * (1.0 + 1e-9) && pair_allowed(a.leafc, a.pptr, a.pcol, i, j)) {
        b = pair_band(ci, ej, cdt, a.d, a.cap);
        cand = true;
      }
    }
    const bool has1 = cand && b.glo <= 1 && b.ghi >= 1;
    const bool has2 = a.split_lag2 && cand && b.glo <= gtop && b.ghi >= 2;
    const unsigned m1 = __ballot_sync(FULLMASK, has1);
    const unsigned m2 = __ballot_sync(FULLMASK, has2);
    const int apos = acnt + __popc(m1 & ((1u << lane) - 1u));
    const int pos = cnt + __popc(m2 & ((1u << lane) - 1u));
    if (has1 || has2) {
      PairGeom g;
      pair_geom<BM>(ci, ej.v0, ej.v1, ej.v2, ej.n, nx, g);
      // U^(m), m = 1..gtop (zero before arrival)
      double uu[TDW_NSL_MAX + 2], ww[TDW_NSL_MAX + 2];
#pragma unroll
      for (int m = 0; m < TDW_NSL_MAX + 2; ++m) { uu[m] = 0.0; ww[m] = 0.0; }
      for (int m = 1; m <= gtop; ++m)
        if (b.arr <= m) { coeff_eval<D, BM>(g, (double)m * a.c * a.dt, a.K, uu[m], ww[m]); ++nev; }
      const double pj = a.phi[j];
      if (has1) {
        const double v1u = w[0] * uu[1], v1w = w[0] * ww[1];
        const double val = v1w * pj - v1u * (1.0 - pj);
        if (apos < TDW_ELL_MAX) {
          a.acol[(size_t)apos * a.ns + i] = j;
          a.aval[(size_t)apos * a.ns + i] = val;
        }
        if (j == i) diag = val;
        else offsum += fabs(val);
      }
      if (has2 && pos < TDW_NEAR_MAX) {
        a.ncol[(size_t)pos * a.ns + i] = j;
        for (int gg = 2; gg <= gtop; ++gg) {
          double vu = 0.0, vw = 0.0;
          for (int k = 0; k <= D + 1 && k < gg; ++k) {
            vu += w[k] * uu[gg - k];
            vw += w[k] * ww[gg - k];
          }
          const bool in_band = gg >= b.glo && gg <= b.ghi;
          a.nval[(gg - 2) * gstride + (size_t)pos * a.ns + i] = in_band ? (pj == 1.0 ? -vw : vu) : 0.0;
        }
      }
    }
    cnt += __popc(m2);
    acnt += __popc(m1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    diag += __shfl_xor_sync(FULLMASK, diag, o);
    offsum += __shfl_xor_sync(FULLMASK, offsum, o);
    nev += __shfl_xor_sync(FULLMASK, nev, o);
  }
  for (int p = cnt + lane; p < TDW_NEAR_MAX; p += 32) {
    a.ncol[(size_t)p * a.ns + i] = i;
    for (int gg = 2; gg <= gtop; ++gg) a.nval[(gg - 2) * gstride + (size_t)p * a.ns + i] = 0.0;
  }
  for (int p = acnt + lane; p < TDW_ELL_MAX; p += 32) {
    a.acol[(size_t)p * a.ns + i] = i;
    a.aval[(size_t)p * a.ns + i] = 0.0;
  }
  if (lane == 0) {
    a.adiag[i] = diag;
    a.ncnt[i] = min(cnt, TDW_NEAR_MAX);
    atomicMax(&a.flags[2], cnt);
    atomicMax(a.ell_w, acnt);
    if (cnt > TDW_NEAR_MAX || acnt > TDW_ELL_MAX) atomicExch(&a.flags[3], 1);
    atomicAdd(a.nnz, (unsigned long long)acnt);
    atomicAdd(a.n_near, (unsigned long long)cnt);
    atomicAdd(a.n_evals, (unsigned long long)nev);
    double bound = diag != 0.0 ? offsum / fabs(diag) : 1e300;
    atomicMax(a.bound_bits, (unsigned long long)__double_as_longlong(bound));
  }
}

template <int D, bool BM>
static void launch_fill(const AsmArgs& a, long long nseg, cudaStream_t st) {
  const int threads = 128;
  long long blocks = (nseg * 32 + threads - 1) / threads;
  fill_kernel<D, BM><<<(unsigned)blocks, threads, 0, st>>>(a);
}

template <int D, bool BM>
static void launch_near(const NearArgs& a, cudaStream_t st) {
  const int threads = 128;
  long long blocks = ((long long)a.ns * 32 + threads - 1) / threads;
  near_kernel<D, BM><<<(unsigned)blocks, threads, 0, st>>>(a);
}

__global__ void fill_unit_init(int2* u, long long n) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x)
    u[k] = make_int2(INT_MAX, -1);
}

// ---------------------------------------------------------------- K2, on the fly
// On-the-fly history convolution (coefficient mode TDW_MODE_ON_THE_FLY; SURVEY
// 8(b) `mode`, north_star (1) "recomputed on the fly (FP64-pipe bound)"): no
// banded store.  Every pass re-evaluates, per pair, the closed forms
// U^(g), W^(g) for g in [glo - d - 1, ghi] (elemint.py:89-186 through the same
// coeff_eval as the fill kernel), kappa-combines them into V^(gamma) exactly as
// the fill kernel does -- including the known-density-only split lags -- and
// multiplies them straight into the pass's kb step sums, reading the history
// from global memory.  One warp per (row, group of OTF_TG J-tiles), lane =
// column; the group's row partial goes to bpart[step][row][group], summed by
// reduce_parts in group order.  Same sums as the stored path up to the order
// of the additions; the cost is FP64-bound (~100x the stored pass), so the
// loop uses it only when the store does not fit (or when asked).
struct OtfArgs {
  const double* elem;
  const int* leafc;
  const int* pptr;
  const int* pcol;
  const double* phi;
  const double2* hist;
  double* bpart;
  const int* flags;
  unsigned long long* n_evals;
  const int* ready;  // streamed march: chunks of known data on the device
  int need_ready;    //   chunks this pass needs (0: not streamed)
  int hcols, pad, ns, row_lo, rows_loc, ntiles, tg, S, cap, split_lag2, nsl, alpha, nb;
  double c, dt, K;
};

template <int D, bool BM>
__global__ void __launch_bounds__(128, TDW_FILL_MINB(D)) otf_conv_kernel(OtfArgs a) {
  if (a.need_ready > 0) {  // streamed march: wait for the known rows this pass reads
    if (threadIdx.x == 0) {
      for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.ready) : "memory");
        if (v >= a.need_ready || *(volatile const int*)a.flags != 0) break;
        __nanosleep(500);
      }
    }
    __syncthreads();
  }
  if (*(volatile const int*)a.flags != 0) return;
  const int lane = threadIdx.x & 31;
  const long long task = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (task >= (long long)a.rows_loc * a.S) return;
  const int rloc = (int)(task / a.S), grp = (int)(task % a.S);
  const int i = a.row_lo + rloc;
  double acc[TDW_KB_MAX];
#pragma unroll
  for (int s = 0; s < TDW_KB_MAX; ++s) acc[s] = 0.0;
  long long nev = 0;
  if (i < a.ns) {
    const double cdt = a.c * a.dt;
    double w[D + 2];
    bspline_weights(D, w);
    const double* pi = a.elem + (size_t)i * TDW_ELEM_STRIDE;
    const double ci[3] = {pi[12], pi[13], pi[14]};
    const double nx[3] = {-pi[9], -pi[10], -pi[11]};  // BM operator normal (marching.py:168-173)
    const int t1 = min(a.ntiles, (grp + 1) * a.tg);
    for (int t = grp * a.tg; t < t1; ++t) {
      const int j = t * TDW_TJ + lane;
      if (j >= a.ns || !pair_allowed(a.leafc, a.pptr, a.pcol, i, j)) continue;
      Elem ej;
      load_elem(a.elem, j, ej);
      const Band b = pair_band(ci, ej, cdt, D, a.cap);
      if (b.ghi < b.glo) continue;
      PairGeom g;
      pair_geom<BM>(ci, ej.v0, ej.v1, ej.v2, ej.n, nx, g);
      const double pj = a.phi[j];
      double ru[D + 2], rw[D + 2];
#pragma unroll
      for (int k = 0; k < D + 2; ++k) { ru[k] = 0.0; rw[k] = 0.0; }
      for (int gg = max(b.arr, b.glo - (D + 1)); gg <= b.ghi; ++gg) {
        double u, v;
        coeff_eval<D, BM>(g, (double)gg * a.c * a.dt, a.K, u, v);
        ++nev;
#pragma unroll
        for (int q = D + 1; q > 0; --q) { ru[q] = ru[q - 1]; rw[q] = rw[q - 1]; }
        ru[0] = u;
        rw[0] = v;
        if (gg < b.glo) continue;
        double vu = 0.0, vw = 0.0;
#pragma unroll
        for (int q = 0; q < D + 2; ++q) {
          vu += w[q] * ru[q];
          vw += w[q] * rw[q];
        }
        if (a.split_lag2 && gg >= 2 && gg <= a.nsl + 1) {  // known density only (as the fill kernel)
          vu = pj == 1.0 ? vu : 0.0;
          vw = pj == 1.0 ? 0.0 : vw;
        }
        // step alpha + s at lag gg reads time alpha + s - gg (zero rows before t = 0)
        const double2* h = a.hist + (size_t)(a.pad + a.alpha - gg) * a.hcols + j;
#pragma unroll
        for (int s = 0; s < TDW_KB_MAX; ++s)
          if (s < a.nb) {
            const double2 x = __ldcg(h + (size_t)s * a.hcols);  // L2: rows may have arrived during this launch
            acc[s] = fma(-vw, x.y, fma(vu, x.x, acc[s]));
          }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < TDW_KB_MAX; ++s) {
    double v = acc[s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    if (lane == 0 && s < a.nb) a.bpart[(size_t)s * a.rows_loc * a.S + (size_t)rloc * a.S + grp] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nev += __shfl_xor_sync(FULLMASK, nev, o);
  if (lane == 0 && a.n_evals) atomicAdd(a.n_evals, (unsigned long long)nev);
}

}  // namespace tdw

using namespace tdw;

static int choose_conv_schedule(tdw_problem* pb) {
  tdw_ctx* ctx = pb->ctx;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  // FIFO capacity: all opt-in shared memory but the kernel's static part
  size_t cap = std::min<size_t>((size_t)maxsm - 1024, 224 * 1024) / 128 * 128;
  if (const char* e = getenv("TDW_CONV_CAP"))  // experiments: a smaller FIFO (KB)
    cap = std::min(cap, (size_t)atoi(e) * 1024 / 128 * 128);
  pb->wbox = pb->wmax;
  if (pb->wbox + pb->kb - 1 > 256)
    return tdw_fail(ctx, TDW_ERR_LIMIT, "history slice of a unit exceeds 256 lags (TMA box limit)");
  const size_t hist_bytes = sizeof(double2) * TDW_TJ * (size_t)(pb->wbox + pb->kb - 1);
  const size_t worst = (pb->max_unit_bytes + 127) / 128 * 128 + (hist_bytes + 127) / 128 * 128;
  if (worst > cap)
    return tdw_fail(ctx, TDW_ERR_LIMIT,
                    "a store unit (" + std::to_string(pb->max_unit_bytes) + " B + history " +
                        std::to_string(hist_bytes) + " B) exceeds shared memory");
  pb->conv_stage_bytes = cap;
  pb->conv_nstages = 4;
  // keep the solver's SMs free (overlap) unless the bandwidth they would add to
  // the convolution is worth more than the solve time (~100 us per step)
  const double conv_est = (double)(pb->n_band * 16) / 6.0e12;
  bool reserve = pb->conv_reserve_model >= 0 ? pb->conv_reserve_model == 1
                                             : conv_est * pb->sp_cl / ctx->num_sms < 100e-6;
  if (const char* r = getenv("TDW_CONV_RESERVE")) reserve = atoi(r) != 0;  // experiments
  pb->conv_reserve = reserve;
  const int G = std::max(1, ctx->num_sms - (reserve ? pb->sp_cl : 0));
  // items = (I-block, tile split); pick the split count that balances the waves
  int bestS = 1;
  double best = -1.0;
  for (int S = 1; S <= std::min(pb->ntiles, 128); ++S) {
    const long long items = (long long)pb->n_iblk * S;
    const long long waves = (items + G - 1) / G;
    double eff = (double)items / (double)(waves * G);
    if (items < 2LL * G && S < pb->ntiles) eff *= 0.9;  // keep a few units per CTA in flight
    if (eff > best + 1e-9) { best = eff; bestS = S; }
  }
  pb->conv_S = bestS;
  pb->conv_grid = (int)std::min<long long>(G, (long long)pb->n_iblk * bestS);
  return TDW_OK;
}

// host wall-clock split of tdw_assemble (TDW_TRACE_ASM=1, stderr)
static double asm_now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int tdw_assemble_impl(tdw_problem* pb) {
  static const bool trace_asm = getenv("TDW_TRACE_ASM") != nullptr;
  const double tw0 = asm_now_ms();
  tdw_ctx* ctx = pb->ctx;
  cudaStream_t st = ctx->stream;
  cudaEvent_t e0, e1, f0, f1;
  TDW_CUDA(ctx, cudaEventCreate(&e0));
  TDW_CUDA(ctx, cudaEventCreate(&e1));
  TDW_CUDA(ctx, cudaEventCreate(&f0));
  TDW_CUDA(ctx, cudaEventCreate(&f1));
  TDW_CUDA(ctx, cudaEventRecord(e0, st));

  const long long nseg = (long long)pb->rows_per_rank * pb->ntiles;
  const long long nunit = (long long)pb->n_iblk * pb->ntiles;
  uint32_t* d_hdr_tmp = nullptr;
  unsigned long long* d_segcnt = nullptr;
  unsigned long long* d_cnt = nullptr;  // {n_evals, n_pairs, nnz, bound_bits, max_rel, n_near, near_evals}
  TDW_CUDA(ctx, cudaMalloc(&d_hdr_tmp, sizeof(uint32_t) * nseg * TDW_TJ));
  TDW_CUDA(ctx, cudaMalloc(&d_segcnt, sizeof(unsigned long long) * nseg));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_unit, sizeof(int2) * nunit));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_unit_off, sizeof(unsigned long long) * (nunit + 1)));
  TDW_CUDA(ctx, cudaMalloc(&d_cnt, sizeof(unsigned long long) * 8));
  unsigned* d_ucoef = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&d_ucoef, sizeof(unsigned) * nunit));
  TDW_CUDA(ctx, cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 8, st));
  TDW_CUDA(ctx, cudaMemsetAsync(pb->d_flags, 0, sizeof(int) * 4, st));
  fill_unit_init<<<256, 256, 0, st>>>(pb->d_unit, nunit);

  const bool bm = pb->bie == TDW_BIE_BMBIE;
  // near structure (split lags 2..nsl+1) and lag-1 step matrix, all rows.  Built
  // first: the pass overlap, then the temporal block kb, shrink until the near
  // structure fits.
  TDW_CUDA(ctx, cudaMalloc(&pb->d_acol, sizeof(int) * (size_t)TDW_ELL_MAX * pb->ns));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_aval, sizeof(double) * (size_t)TDW_ELL_MAX * pb->ns));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_adiag, sizeof(double) * pb->ns));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_ncol, sizeof(int) * (size_t)TDW_NEAR_MAX * pb->ns));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_nval, sizeof(double) * (size_t)pb->nsl * TDW_NEAR_MAX * pb->ns));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_ncnt, sizeof(int) * (size_t)pb->ns));
  int* d_ellw = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&d_ellw, sizeof(int)));
  for (;;) {
  TDW_CUDA(ctx, cudaMemsetAsync(d_ellw, 0, sizeof(int), st));
  TDW_CUDA(ctx, cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 8, st));
  TDW_CUDA(ctx, cudaMemsetAsync(pb->d_flags, 0, sizeof(int) * 4, st));
  NearArgs s{};
  s.elem = pb->d_elem;
  s.leafc = pb->d_leafc;
  s.pptr = pb->d_pair_ptr;
  s.pcol = pb->d_pair_col;
  s.split_lag2 = pb->split_lag2;
  s.nsl = pb->nsl;
  s.phi = pb->d_phi;
  s.ns = pb->ns;
  s.ntiles = pb->ntiles;
  s.d = pb->d;
  s.cap = pb->cap;
  s.c = pb->c;
  s.dt = pb->dt;
  s.K = pb->K;
  s.ncol = pb->d_ncol;
  s.nval = pb->d_nval;
  s.acol = pb->d_acol;
  s.aval = pb->d_aval;
  s.adiag = pb->d_adiag;
  s.flags = pb->d_flags;
  s.ell_w = d_ellw;
  s.ncnt = pb->d_ncnt;
  s.bound_bits = d_cnt + 3;
  s.nnz = d_cnt + 2;
  s.n_near = d_cnt + 5;
  s.n_evals = d_cnt + 6;
  if (pb->d == 1) { if (bm) launch_near<1, true>(s, st); else launch_near<1, false>(s, st); }
  if (pb->d == 2) { if (bm) launch_near<2, true>(s, st); else launch_near<2, false>(s, st); }
  if (pb->d == 3) { if (bm) launch_near<3, true>(s, st); else launch_near<3, false>(s, st); }
  TDW_CUDA(ctx, cudaGetLastError());
  int nf[4];
  TDW_CUDA(ctx, cudaMemcpyAsync(nf, pb->d_flags, sizeof(nf), cudaMemcpyDeviceToHost, st));
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  if (nf[3] == 1 && pb->nsl > 1) {
    if (pb->overlap > 1) --pb->overlap;
    else --pb->kb;
    pb->overlap = std::min(pb->overlap, pb->kb);
    pb->nsl = pb->kb + pb->overlap - 1;
    pb->bring = pb->kb + pb->overlap;
    continue;
  }
  break;
  }
  // the near kernel's results (complete: synchronised above); the solver setup
  // below needs them while the fill kernel is still running
  {
    unsigned long long hc[8];
    int hfl[4], hellw = 0;
    TDW_CUDA(ctx, cudaMemcpy(hc, d_cnt, sizeof(hc), cudaMemcpyDeviceToHost));
    TDW_CUDA(ctx, cudaMemcpy(hfl, pb->d_flags, sizeof(hfl), cudaMemcpyDeviceToHost));
    TDW_CUDA(ctx, cudaMemcpy(&hellw, d_ellw, sizeof(int), cudaMemcpyDeviceToHost));
    pb->n_near = (int64_t)hc[5];
    pb->n_near_evals = (int64_t)hc[6];
    pb->near_w = hfl[2];
    pb->step_nnz = (int)hc[2];
    double bound;
    memcpy(&bound, &hc[3], sizeof(bound));
    pb->jac_bound = bound;
    pb->ell_w = hellw;
    if (hfl[3] == 1)
      return tdw_fail(ctx, TDW_ERR_LIMIT, "near structure: more than the supported pairs near a row");
    // a zero diagonal: the reference's splu raises "step matrix is singular"
    // (marching.py:284-288); the loop's solver divides by the diagonal
    std::vector<double> dg(pb->ns);
    TDW_CUDA(ctx, cudaMemcpy(dg.data(), pb->d_adiag, sizeof(double) * pb->ns, cudaMemcpyDeviceToHost));
    for (int i = 0; i < pb->ns; ++i)
      if (!(dg[i] != 0.0) || !std::isfinite(dg[i]))
        return tdw_fail(ctx, TDW_ERR_SINGULAR, "step matrix is singular (zero diagonal)");
    // sweeps for a contraction of 1e-17 under the infinity-norm bound (cap; the
    // solver stops earlier once the update is at round-off); bound >= 0.9 selects
    // the BiCGSTAB solver (tdw_setup_cluster_solver)
    const int it = (bound > 0.0 && bound < 0.9) ? (int)ceil(log(1e-17) / log(bound)) : 400;
    pb->jac_iters = std::max(2, std::min(it, 400));
  }

  AsmArgs a{};
  a.elem = pb->d_elem;
  a.leafc = pb->d_leafc;
  a.pptr = pb->d_pair_ptr;
  a.pcol = pb->d_pair_col;
  a.split_lag2 = pb->split_lag2;
  a.nsl = pb->nsl;
  a.ns = pb->ns;
  a.row_lo = pb->row_lo;
  a.rows_loc = pb->rows_per_rank;
  a.ntiles = pb->ntiles;
  a.d = pb->d;
  a.cap = pb->cap;
  a.c = pb->c;
  a.dt = pb->dt;
  a.K = pb->K;
  a.hdr = d_hdr_tmp;
  a.segcount = d_segcnt;
  a.unit = pb->d_unit;
  a.n_evals = d_cnt;
  a.n_pairs = d_cnt + 1;
  a.flags = pb->d_flags;
  {
    const int threads = 256;
    long long blocks = (nseg * 32 + threads - 1) / threads;
    count_kernel<<<(unsigned)blocks, threads, 0, st>>>(a);
    TDW_CUDA(ctx, cudaGetLastError());
    blocks = (nunit * 32 + threads - 1) / threads;
    const char* f32 = getenv("TDW_HDR32");
    unit_size_kernel<<<(unsigned)blocks, threads, 0, st>>>(d_segcnt, d_hdr_tmp, pb->d_unit, pb->ntiles, nunit,
                                                          f32 && f32[0] == '1', pb->d_unit_off, d_ucoef,
                                                          d_cnt + 7);
    TDW_CUDA(ctx, cudaGetLastError());
  }
  // unit byte offsets: exclusive scan of the unit sizes (in place; last slot = total)
  {
    TDW_CUDA(ctx, cudaMemsetAsync(pb->d_unit_off + nunit, 0, sizeof(unsigned long long), st));
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, pb->d_unit_off, pb->d_unit_off, nunit + 1, st);
    void* tmp = nullptr;
    TDW_CUDA(ctx, cudaMalloc(&tmp, tmp_bytes));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, pb->d_unit_off, pb->d_unit_off, nunit + 1, st);
    TDW_CUDA(ctx, cudaGetLastError());
    TDW_CUDA(ctx, cudaStreamSynchronize(st));
    cudaFree(tmp);
  }
  int hflags[4];
  TDW_CUDA(ctx, cudaMemcpy(hflags, pb->d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  if (hflags[3] == 2)
    return tdw_fail(ctx, TDW_ERR_LIMIT, "a pair band exceeds 255 lags (c*dt far below the element size)");
  std::vector<unsigned long long> uoff(nunit + 1);
  TDW_CUDA(ctx, cudaMemcpy(uoff.data(), pb->d_unit_off, sizeof(unsigned long long) * (nunit + 1),
                           cudaMemcpyDeviceToHost));
  const unsigned long long total_bytes = uoff[nunit];
  {
    unsigned long long nb = 0;
    TDW_CUDA(ctx, cudaMemcpy(&nb, d_cnt + 7, sizeof(nb), cudaMemcpyDeviceToHost));
    pb->n_band = (int64_t)nb;
  }
  pb->max_unit_bytes = 0;
  for (long long u = 0; u < nunit; ++u)
    pb->max_unit_bytes = std::max<size_t>(pb->max_unit_bytes, uoff[u + 1] - uoff[u]);
  std::vector<int2> hu(nunit);
  std::vector<unsigned> ucoef;  // coefficient offset of every unit (= its header block size)
  {
    TDW_CUDA(ctx, cudaMemcpy(hu.data(), pb->d_unit, sizeof(int2) * nunit, cudaMemcpyDeviceToHost));
    ucoef.resize(nunit);
    TDW_CUDA(ctx, cudaMemcpy(ucoef.data(), d_ucoef, sizeof(unsigned) * nunit, cudaMemcpyDeviceToHost));
    int wm = 1;
    pb->n_units = pb->units_hdr32 = 0;
    for (long long u = 0; u < nunit; ++u)
      if (hu[u].y >= hu[u].x) {
        wm = std::max(wm, hu[u].y - hu[u].x + 1);
        ++pb->n_units;
        pb->units_hdr32 += ucoef[u] == TDW_UNIT_COEF_OFF;
      }
    pb->wmax = wm;
    // TMA box heights for the units' history slices (rows = lag span + kb - 1): the
    // 50 / 80 / 95 % quantiles of the spans and the largest
    std::vector<int> spans;
    spans.reserve(nunit);
    for (long long u = 0; u < nunit; ++u)
      if (hu[u].y >= hu[u].x) spans.push_back(hu[u].y - hu[u].x + 1);
    std::sort(spans.begin(), spans.end());
    pb->hbox_n = 0;
    const double qs[4] = {0.5, 0.8, 0.95, 1.0};
    for (int k = 0; k < 4; ++k) {
      const int w = spans.empty() ? wm : spans[std::min(spans.size() - 1, (size_t)(qs[k] * (spans.size() - 1) + 0.5))];
      const int rows = (k == 3 ? wm : w) + pb->kb - 1;
      if (pb->hbox_n == 0 || rows > pb->hbox_rows[pb->hbox_n - 1]) pb->hbox_rows[pb->hbox_n++] = rows;
    }
  }
  // coefficient mode (SURVEY 8(b) `mode`): the banded store when it fits in device
  // memory (TDW_MODE_AUTO) or when asked; otherwise the coefficients are
  // recomputed by every convolution pass (otf_conv_kernel)
  {
    size_t fr = 0, tot = 0;
    TDW_CUDA(ctx, cudaMemGetInfo(&fr, &tot));
    pb->otf = pb->mode == TDW_MODE_ON_THE_FLY ||
              (pb->mode == TDW_MODE_AUTO && total_bytes + (2ull << 30) > (unsigned long long)fr);
  }
  if (!pb->otf) {
  TDW_CUDA(ctx, cudaMalloc(&pb->d_units, total_bytes));
  {
    const int threads = 256;
    long long blocks = (nunit * 32 + threads - 1) / threads;
    unit_layout_kernel<<<(unsigned)blocks, threads, 0, st>>>(d_segcnt, d_hdr_tmp, pb->d_unit, d_ucoef,
                                                            pb->ntiles, nunit, pb->d_unit_off,
                                                            pb->d_units, (unsigned*)(d_cnt + 4));
    TDW_CUDA(ctx, cudaGetLastError());
  }
  a.unit_off = pb->d_unit_off;
  a.units = pb->d_units;
  a.phi = pb->d_phi;
  TDW_CUDA(ctx, cudaEventRecord(f0, st));
  if (pb->d == 1) { if (bm) launch_fill<1, true>(a, nseg, st); else launch_fill<1, false>(a, nseg, st); }
  if (pb->d == 2) { if (bm) launch_fill<2, true>(a, nseg, st); else launch_fill<2, false>(a, nseg, st); }
  if (pb->d == 3) { if (bm) launch_fill<3, true>(a, nseg, st); else launch_fill<3, false>(a, nseg, st); }
  TDW_CUDA(ctx, cudaGetLastError());
  TDW_CUDA(ctx, cudaEventRecord(f1, st));
  } else {
    TDW_CUDA(ctx, cudaEventRecord(f0, st));
    TDW_CUDA(ctx, cudaEventRecord(f1, st));
  }

  TDW_CUDA(ctx, cudaEventRecord(e1, st));
  // Cluster solver first: its CTAs' SMs are kept free of convolution CTAs so the
  // far convolution of the next step overlaps the solve.  Its setup is host work
  // (partition, halo sets) on the near kernel's results: it runs here, while the
  // fill kernel -- most of the assembly's device time -- is still running.
  {
    const double tw1 = asm_now_ms();
    int src = tdw_setup_cluster_solver(pb);
    if (trace_asm)
      fprintf(stderr, "assemble: launches + host readback %.2f ms, solver setup (beside the fill kernel) %.2f ms\n",
              tw1 - tw0, asm_now_ms() - tw1);
    if (src) {
      cudaStreamSynchronize(st);
      return src;
    }
  }
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  cudaFree(d_hdr_tmp);
  cudaFree(d_segcnt);
  cudaFree(d_ucoef);

  unsigned long long hc[8];
  TDW_CUDA(ctx, cudaMemcpy(hc, d_cnt, sizeof(hc), cudaMemcpyDeviceToHost));
  TDW_CUDA(ctx, cudaMemcpy(hflags, pb->d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  cudaFree(d_cnt);
  cudaFree(d_ellw);
  pb->n_evals = (int64_t)hc[0];
  pb->n_pairs = (int64_t)hc[1];
  float ms = 0.f, fms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventElapsedTime(&fms, f0, f1);
  pb->t_assemble_ms = ms;
  pb->t_fill_ms = fms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(f0);
  cudaEventDestroy(f1);
  if (trace_asm) fprintf(stderr, "assemble: fill kernel done at %.2f ms\n", asm_now_ms() - tw0);
  if (pb->otf) {
    // on the fly: one warp per (row, group of 8 J-tiles), partials per group
    pb->otf_tg = 8;
    const int S = (pb->ntiles + pb->otf_tg - 1) / pb->otf_tg;
    pb->nsplit = pb->conv_S = S;
    pb->conv_grid = 0;
    cudaFree(pb->d_bpart);
    TDW_CUDA(ctx, cudaMalloc(&pb->d_bpart, pb->kb * sizeof(double) * (size_t)S * pb->rows_per_rank));
    TDW_CUDA(ctx, cudaMemset(pb->d_bpart, 0, pb->kb * sizeof(double) * (size_t)S * pb->rows_per_rank));
    TDW_CUDA(ctx, cudaMalloc(&pb->d_bnear, sizeof(double) * (size_t)pb->nsl * (pb->nsl + 1) * pb->ns));
    if (!pb->d_otf_evals) TDW_CUDA(ctx, cudaMalloc(&pb->d_otf_evals, sizeof(unsigned long long)));
    TDW_CUDA(ctx, cudaMemset(pb->d_otf_evals, 0, sizeof(unsigned long long)));
    pb->store_bytes = 0;
    pb->assembled = true;
    return TDW_OK;
  }
  // convolution schedule (persistent CTAs, unit list per CTA)
  {
    int rc = choose_conv_schedule(pb);
    if (rc) return rc;
  }
  {
    int G = pb->conv_grid, S = pb->conv_S;
    std::vector<unsigned> sched, sitem, soff(G + 1, 0);
    sched.reserve(nunit);
    sitem.reserve(nunit);
    auto streamed = [&](long long u) { return hu[u].y >= hu[u].x || !pb->skip_empty_units; };
    const char* sm = getenv("TDW_SCHED");
    if (!(sm && strcmp(sm, "rr") == 0)) {
      // Fixed summation groups: the J-tiles of an I-block are cut into groups of
      // gt consecutive tiles.  A group is always summed by
      // ONE CTA (units in tile order, then the warp's lane reduction) into its own
      // partial, and the partials of a row are added in group order
      // (reduce_parts / sum_parts).  The grouping depends on the problem only, not
      // on the grid size or on how rows are sharded over ranks, so b -- and every
      // density -- is bit-identical for any rank count and any SM reservation.
      // The persistent CTAs get byte-balanced contiguous runs of whole groups.
      // weight: coefficient bytes + a fixed per-unit cost (header, history box);
      // independent of the header width, so both widths give the same schedule
      const double per_unit = 4096.0;
      auto weight = [&](long long u) { return (double)(uoff[u + 1] - uoff[u] - ucoef[u]) + per_unit; };
      // groups per I-block: 4, more when the whole problem has few I-blocks (at
      // least 2 groups per SM); from the WHOLE problem's I-block count, so every
      // rank count cuts the same groups.  A bandwidth-bound pass tolerates the
      // coarse balance (config 2: 2% slower than cuts at unit granularity)
      const int nblk_total = (pb->ns + TDW_TI - 1) / TDW_TI;
      const int gpi = std::min(pb->ntiles, std::max(4, (2 * ctx->num_sms + nblk_total - 1) / nblk_total));
      int gt = (pb->ntiles + gpi - 1) / gpi;
      if (const char* e = getenv("TDW_GROUP_TILES")) gt = std::max(1, atoi(e));
      const int SG = (pb->ntiles + gt - 1) / gt;
      const long long ngroup = (long long)pb->n_iblk * SG;
      std::vector<double> gw(ngroup, 0.0);
      std::vector<char> gstream(ngroup, 0);
      double total = 0.0;
      for (long long u = 0; u < nunit; ++u)
        if (streamed(u)) {
          const long long ib = u / pb->ntiles, t = u % pb->ntiles, gidx = ib * SG + t / gt;
          gw[gidx] += weight(u);
          gstream[gidx] = 1;
          total += weight(u);
        }
      long long nlive = 0;
      for (long long gidx = 0; gidx < ngroup; ++gidx) nlive += gstream[gidx];
      G = (int)std::max(1LL, std::min<long long>(ctx->num_sms - (pb->conv_reserve ? pb->sp_cl : 0), nlive));
      if (const char* gm = getenv("TDW_CONV_GRID_MAX")) G = std::max(1, std::min(G, atoi(gm)));  // experiments
      soff.assign(G + 1, 0);
      std::vector<int> chunk_of_group(ngroup, -1);
      double acc = 0.0;
      for (long long gidx = 0; gidx < ngroup; ++gidx) {
        if (!gstream[gidx]) continue;
        chunk_of_group[gidx] = std::min(G - 1, (int)((acc + 0.5 * gw[gidx]) / total * G));
        acc += gw[gidx];
      }
      int k = 0;
      for (long long u = 0; u < nunit; ++u) {
        if (!streamed(u)) continue;
        const long long ib = u / pb->ntiles, t = u % pb->ntiles, gidx = ib * SG + t / gt;
        const int c = chunk_of_group[gidx];
        while (k <= c) soff[k++] = (unsigned)sched.size();
        sched.push_back((unsigned)u);
        sitem.push_back((unsigned)gidx);
      }
      while (k < G) soff[k++] = (unsigned)sched.size();
      pb->conv_grid = G;
      pb->conv_S = S = SG;
    } else {
    const long long items = (long long)pb->n_iblk * S;
    for (int b = 0; b < G; ++b) {
      soff[b] = (unsigned)sched.size();
      for (long long it2 = b; it2 < items; it2 += G) {
        const long long iblk = it2 / S, sp = it2 % S;
        const int tb = (int)(sp * pb->ntiles / S), te = (int)((sp + 1) * pb->ntiles / S);
        const size_t before = sched.size();
        for (int t = tb; t < te; ++t) {
          const long long u = iblk * pb->ntiles + t;
          // units without band entries (FMM near field: non-adjacent patches) are not streamed
          if (streamed(u)) {
            sched.push_back((unsigned)u);
            sitem.push_back((unsigned)it2);
          }
        }
        if (sched.size() == before) {  // nothing to stream: an entry that only flushes zeros
          sched.push_back(TDW_EMPTY_UNIT);
          sitem.push_back((unsigned)it2);
        }
      }
    }
    }
    soff[G] = (unsigned)sched.size();
    TDW_CUDA(ctx, cudaMalloc(&pb->d_sched, sizeof(unsigned) * std::max<size_t>(1, sched.size())));
    TDW_CUDA(ctx, cudaMalloc(&pb->d_sched_off, sizeof(unsigned) * (G + 1)));
    TDW_CUDA(ctx, cudaMemcpy(pb->d_sched, sched.data(), sizeof(unsigned) * sched.size(), cudaMemcpyHostToDevice));
    TDW_CUDA(ctx, cudaMalloc(&pb->d_sched_item, sizeof(unsigned) * std::max<size_t>(1, sitem.size())));
    TDW_CUDA(ctx, cudaMemcpy(pb->d_sched_item, sitem.data(), sizeof(unsigned) * sitem.size(), cudaMemcpyHostToDevice));
    TDW_CUDA(ctx, cudaMemcpy(pb->d_sched_off, soff.data(), sizeof(unsigned) * (G + 1), cudaMemcpyHostToDevice));
    pb->nsplit = S;
    cudaFree(pb->d_bpart);
    // [kb][rows][S]: one pass's partials (reduced on the pass's stream before the next pass)
    TDW_CUDA(ctx, cudaMalloc(&pb->d_bpart, pb->kb * sizeof(double) * (size_t)S * pb->rows_per_rank));
    TDW_CUDA(ctx, cudaMemset(pb->d_bpart, 0, pb->kb * sizeof(double) * (size_t)S * pb->rows_per_rank));
    TDW_CUDA(ctx, cudaMalloc(&pb->d_bnear, sizeof(double) * (size_t)pb->nsl * (pb->nsl + 1) * pb->ns));
  }
  pb->store_bytes = (int64_t)(total_bytes + sizeof(unsigned long long) * (nunit + 1) + sizeof(int2) * nunit);
  pb->assembled = true;
  if (trace_asm) fprintf(stderr, "assemble: total %.2f ms\n", asm_now_ms() - tw0);
  return TDW_OK;
}

// one on-the-fly convolution pass of steps alpha .. alpha + nb - 1 into bpart
int launch_otf_conv(tdw_problem* pb, int alpha, int nb, cudaStream_t st) {
  OtfArgs o{};
  o.elem = pb->d_elem;
  o.leafc = pb->d_leafc;
  o.pptr = pb->d_pair_ptr;
  o.pcol = pb->d_pair_col;
  o.phi = pb->d_phi;
  o.hist = pb->d_hist;
  o.bpart = pb->d_bpart;
  o.flags = pb->d_flags;
  o.n_evals = pb->d_otf_evals;
  o.ready = pb->d_ready;
  o.need_ready = pb->need_ready;
  o.hcols = pb->hcols;
  o.pad = pb->pad;
  o.ns = pb->ns;
  o.row_lo = pb->row_lo;
  o.rows_loc = pb->rows_per_rank;
  o.ntiles = pb->ntiles;
  o.tg = pb->otf_tg;
  o.S = pb->nsplit;
  o.cap = pb->cap;
  o.split_lag2 = pb->split_lag2;
  o.nsl = pb->nsl;
  o.alpha = alpha;
  o.nb = nb;
  o.c = pb->c;
  o.dt = pb->dt;
  o.K = pb->K;
  const bool bm = pb->bie == TDW_BIE_BMBIE;
  const long long threads = (long long)pb->rows_per_rank * pb->nsplit * 32;
  const unsigned blocks = (unsigned)((threads + 127) / 128);
  if (pb->d == 1) { if (bm) otf_conv_kernel<1, true><<<blocks, 128, 0, st>>>(o); else otf_conv_kernel<1, false><<<blocks, 128, 0, st>>>(o); }
  if (pb->d == 2) { if (bm) otf_conv_kernel<2, true><<<blocks, 128, 0, st>>>(o); else otf_conv_kernel<2, false><<<blocks, 128, 0, st>>>(o); }
  if (pb->d == 3) { if (bm) otf_conv_kernel<3, true><<<blocks, 128, 0, st>>>(o); else otf_conv_kernel<3, false><<<blocks, 128, 0, st>>>(o); }
  TDW_CUDA(pb->ctx, cudaGetLastError());
  return TDW_OK;
}
