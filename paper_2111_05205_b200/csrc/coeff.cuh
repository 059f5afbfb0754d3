// coeff.cuh -- device evaluation of the retarded element coefficients.
//
// B200 restatement of elemint.retarded_coeff_table
// (reference: pkg/src/tdwavebem/elemint.py:89-186).  The per-(point, triangle)
// geometry that does not depend on the retarded radius s -- edge frames
// (elemint.py:36-57), the free-term side sgn (:123-124), the |y| tolerance test
// (:129-130), the solid-angle increments datan (:139) and the Burton-Miller
// normal projections (:166-168) -- is hoisted into PairGeom once per pair; the
// s-dependent part (wavefront clipping :60-76, masked bundles :79-86, the
// U/W and Ubar/Wbar combinations :145-186) runs per lag.  Predicates are
// reproduced exactly (strict/non-strict comparisons, masked substitution).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "closed_forms.cuh"

namespace tdw {

constexpr double kYTol = 1e-12;  // elemint.py:33

struct PairGeom {
  double za, sgn, n3;
  double x1[3], x2[3], y[3], datan[3];
  double n1[3], n2[3];
  bool yok[3];
};

__device__ __forceinline__ double clipd(double a, double lo, double hi) {
  double t = a > lo ? a : lo;
  return t < hi ? t : hi;
}

template <int E>
__device__ __forceinline__ double ipow(double v) {
  double r = 1.0;
#pragma unroll
  for (int k = 0; k < E; ++k) r *= v;
  return r;
}

// P: collocation point; A,B,C: triangle; ez: unit normal; nx: BM operator
// normal (nullptr for the uw kind).
template <bool BM>
__device__ __forceinline__ void pair_geom(const double* P, const double* A, const double* B,
                                          const double* C, const double* ez, const double* nx,
                                          PairGeom& g) {
  const double* V1[3] = {A, B, C};
  const double* V2[3] = {B, C, A};
  double zs = (P[0] - A[0]) * ez[0] + (P[1] - A[1]) * ez[1] + (P[2] - A[2]) * ez[2];
  double O0 = P[0] - zs * ez[0], O1 = P[1] - zs * ez[1], O2 = P[2] - zs * ez[2];
  double elen[3];
  g.za = fabs(zs);
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    double e0 = V2[e][0] - V1[e][0], e1 = V2[e][1] - V1[e][1], e2 = V2[e][2] - V1[e][2];
    elen[e] = sqrt(e0 * e0 + e1 * e1 + e2 * e2);
    double h0 = e0 / elen[e], h1 = e1 / elen[e], h2 = e2 / elen[e];
    double k0 = ez[1] * h2 - ez[2] * h1;
    double k1 = ez[2] * h0 - ez[0] * h2;
    double k2 = ez[0] * h1 - ez[1] * h0;
    double r0 = V1[e][0] - O0, r1 = V1[e][1] - O1, r2 = V1[e][2] - O2;
    g.x1[e] = r0 * h0 + r1 * h1 + r2 * h2;
    g.x2[e] = g.x1[e] + elen[e];
    g.y[e] = r0 * k0 + r1 * k1 + r2 * k2;
    g.yok[e] = fabs(g.y[e]) > kYTol * (elen[e] + g.za);
    g.datan[e] = g.yok[e] ? (atan(g.x2[e] / g.y[e]) - atan(g.x1[e] / g.y[e])) : 0.0;
    if (BM) {
      g.n1[e] = nx[0] * h0 + nx[1] * h1 + nx[2] * h2;
      g.n2[e] = nx[0] * k0 + nx[1] * k1 + nx[2] * k2;
    }
  }
  double emax = fmax(fmax(elen[0], elen[1]), elen[2]);
  g.sgn = zs > 1e-12 * (emax + fabs(zs)) ? 1.0 : -1.0;
  if (BM) g.n3 = nx[0] * ez[0] + nx[1] * ez[1] + nx[2] * ez[2];
}

template <int D>
__device__ __forceinline__ void uw_bundle(double x, double y, double z, double s, double* o) {
  if (D == 1) tdw_uw_d1(x, y, z, s, o);
  if (D == 2) tdw_uw_d2(x, y, z, s, o);
  if (D == 3) tdw_uw_d3(x, y, z, s, o);
}
template <int D>
__device__ __forceinline__ void bm_bundle(double x, double y, double z, double s, double* o) {
  if (D == 1) tdw_bm_d1(x, y, z, s, o);
  if (D == 2) tdw_bm_d2(x, y, z, s, o);
  if (D == 3) tdw_bm_d3(x, y, z, s, o);
}

// (U, W) for BM == false; (Ubar, Wbar) for BM == true.  K = 1/(4 pi (c dt)^D).
template <int D, bool BM>
__device__ __forceinline__ void coeff_eval(const PairGeom& g, double s, double K, double& o0,
                                           double& o1) {
  double acc0 = 0.0, acc1 = 0.0;
  // Not unrolled: the closed-form bundles are large (bm d1: ~200 operations), and
  // 3 edges x 2 limits of inlined copies overflow the instruction cache (the fill
  // kernel stalled on instruction fetch more than on anything else); one copy of
  // the bundle evaluated for both limits in a 2-trip loop keeps the code small.
#pragma unroll 1
  for (int e = 0; e < 3; ++e) {
    const bool alive = g.yok[e] && (s > g.za);
    if (!alive) continue;  // every term of a dead sub-triangle is exactly zero
    const double y = g.y[e], x1 = g.x1[e], x2 = g.x2[e], datan = g.datan[e];
    const double xc2 = s * s - y * y - g.za * g.za;
    const bool has = xc2 > 0.0;
    const double xc = sqrt(has ? xc2 : 0.0);
    const double xlo = clipd(x1, -xc, xc), xhi = clipd(x2, -xc, xc);
    const bool fmask = has && (xhi > xlo);
    const double pw = s - g.za;
    if (!BM) {
      double lo[2] = {0.0, 0.0}, hi[2] = {0.0, 0.0};
      if (fmask) {
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          double r[2];
          uw_bundle<D>(side ? xhi : xlo, y, g.za, s, r);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (side) hi[k] = r[k];
            else lo[k] = r[k];
          }
        }
      }
      const double a0 = -ipow<D + 1>(pw) / (D + 1) * datan;
      const double az = g.sgn * ipow<D>(pw) * datan;
      acc0 += a0 + hi[0] - lo[0];
      acc1 += az + g.sgn * (hi[1] - lo[1]);
    } else {
      double lo[8], hi[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) { lo[k] = 0.0; hi[k] = 0.0; }
      if (fmask) {
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          double r[8];
          bm_bundle<D>(side ? xhi : xlo, y, g.za, s, r);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (side) hi[k] = r[k];
            else lo[k] = r[k];
          }
        }
      }
      const bool m1 = fmask && (x1 > -xc) && (x1 < xc);
      const bool m2 = fmask && (x2 > -xc) && (x2 < xc);
      if (!m1) { lo[0] = 0.0; lo[1] = 0.0; }
      if (!m2) { hi[0] = 0.0; hi[1] = 0.0; }
      const double pwd = ipow<D>(pw);
      const double az = g.sgn * pwd * datan;
      const double as = -pwd * datan;
      const double azz = D > 1 ? -D * ipow<(D > 1 ? D - 1 : 0)>(pw) * datan
                               : -(pw > 0.0 ? 1.0 : 0.0) * datan;
      const double azs = -g.sgn * azz;
      const double dPx = lo[0] - hi[0];
      const double dPy = -(hi[2] - lo[2]);
      const double dz = az + g.sgn * (hi[3] - lo[3]);
      const double ds = as + hi[4] - lo[4];
      const double dzPx = g.sgn * (lo[1] - hi[1]);
      const double dzPy = -g.sgn * (hi[5] - lo[5]);
      const double dzz = azz + hi[6] - lo[6];
      const double dzs = azs + g.sgn * (hi[7] - lo[7]);
      acc0 += g.n1[e] * dPx + g.n2[e] * dPy + g.n3 * dz - ds;
      acc1 += g.n1[e] * dzPx + g.n2[e] * dzPy + g.n3 * dzz - dzs;
    }
  }
  o0 = K * acc0;
  o1 = -K * acc1;
}

__host__ __device__ inline double kfactor(int d, double c, double dt) {
  double cd = c * dt, p = 1.0;
  for (int k = 0; k < d; ++k) p *= cd;
  return 1.0 / (4.0 * 3.14159265358979323846 * p);
}

}  // namespace tdw
