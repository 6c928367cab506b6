// geom.cuh -- geometry shared by the device cull kernels and the host-side
// partition traversal (rc_exchange_partners): restriction of the tree's
// Bernstein-Bezier points to a subcube, bilinear patch points, and the
// pixel-centre rectangle of a camera-space AABB.  One definition
// on both sides, so the host's virtual-node boxes nest the device's leaf boxes.
#pragma once
#include <math.h>

#include "rc_internal.cuh"

namespace rc {

// Restriction of a degree-R Bernstein polynomial (along one axis) to [u,v]:
// new control points are blossom values P(u..u, v..v) (de Casteljau).
template <int R>
__host__ __device__ __forceinline__ void bz_restrict_row(double u, double v, double M[R + 1][R + 1]);

template <>
__host__ __device__ __forceinline__ void bz_restrict_row<1>(double u, double v, double M[2][2]) {
  M[0][0] = 1 - u; M[0][1] = u;
  M[1][0] = 1 - v; M[1][1] = v;
}
template <>
__host__ __device__ __forceinline__ void bz_restrict_row<2>(double u, double v, double M[3][3]) {
  // blossom P(x,y) = (1-x)(1-y) p0 + ((1-x)y + x(1-y)) p1 + x y p2
  double x[3] = {u, u, v}, y[3] = {u, v, v};
  for (int r = 0; r < 3; ++r) {
    M[r][0] = (1 - x[r]) * (1 - y[r]);
    M[r][1] = (1 - x[r]) * y[r] + x[r] * (1 - y[r]);
    M[r][2] = x[r] * y[r];
  }
}

// Camera-space AABB of an element's Bernstein points: the
// tree's points Btree (index [m3][m2][m1][xyz]) restricted to the subcube
// t0 + [0,h]^3 by the blossom rows of each axis, one coordinate at a time and
// sum-factorised (axis 3, then 2, then 1), min / max taken on the fly -- few
// doubles live at once (one thread per leaf in k_cull_curved).
template <int R>
__host__ __device__ inline void element_aabb(const double* __restrict__ Btree, const double t0[3], double h,
                                             double lo[3], double hi[3]) {
  constexpr int n1 = R + 1;
  double M[3][n1][n1];
#pragma unroll
  for (int k = 0; k < 3; ++k) bz_restrict_row<R>(t0[k], t0[k] + h, M[k]);
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    double l = 1e300, u = -1e300;
#pragma unroll
    for (int r3 = 0; r3 < n1; ++r3) {
      double T2[n1 * n1];
#pragma unroll
      for (int q21 = 0; q21 < n1 * n1; ++q21) {
        double s = 0.0;
#pragma unroll
        for (int q3 = 0; q3 < n1; ++q3) s = fma(M[2][r3][q3], Btree[(q3 * n1 * n1 + q21) * 3 + c], s);
        T2[q21] = s;
      }
#pragma unroll
      for (int r2 = 0; r2 < n1; ++r2) {
        double T1[n1];
#pragma unroll
        for (int q1 = 0; q1 < n1; ++q1) {
          double s = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < n1; ++q2) s = fma(M[1][r2][q2], T2[q2 * n1 + q1], s);
          T1[q1] = s;
        }
#pragma unroll
        for (int r1 = 0; r1 < n1; ++r1) {
          double v = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < n1; ++q1) v = fma(M[0][r1][q1], T1[q1], v);
          l = fmin(l, v);
          u = fmax(u, v);
        }
      }
    }
    lo[c] = l;
    hi[c] = u;
  }
}

// X(s) of the tree patch with corners Z [m2][m1][xyz] (TreeConst Bw / Bc)
__host__ __device__ __forceinline__ void patch_point(const double* __restrict__ Z, double s1, double s2, double X[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
    X[c] = (1.0 - s2) * ((1.0 - s1) * Z[c] + s1 * Z[3 + c]) + s2 * ((1.0 - s1) * Z[6 + c] + s1 * Z[9 + c]);
}

// pixel-centre rectangle of a camera-space AABB; false: culled
__host__ __device__ __forceinline__ bool project_rect(const CamConst& cc, const double lo[3], const double hi[3], Rect16& rc) {
  double pmin[2], pmax[2];
  int dims[2] = {cc.W, cc.H};
  if (cc.proj == RC_PERSPECTIVE) {
    if (hi[2] < cc.n || lo[2] > cc.far_dist) return false;
    double z0 = fmax(lo[2], cc.n), z1 = fmax(hi[2], cc.n);
    double s = cc.n / cc.ell;
    for (int d = 0; d < 2; ++d) {
      double a = lo[d] / z0, b = lo[d] / z1, c = hi[d] / z0, e = hi[d] / z1;
      pmin[d] = s * fmin(fmin(a, b), fmin(c, e)) + 0.5 * (dims[d] - 1);
      pmax[d] = s * fmax(fmax(a, b), fmax(c, e)) + 0.5 * (dims[d] - 1);
    }
  } else {
    if (hi[2] < 0.0 || lo[2] > cc.far_dist) return false;
    for (int d = 0; d < 2; ++d) {
      pmin[d] = lo[d] / cc.ell + 0.5 * (dims[d] - 1);
      pmax[d] = hi[d] / cc.ell + 0.5 * (dims[d] - 1);
    }
  }
  int r[4];
  for (int d = 0; d < 2; ++d) {
    double a = ceil(pmin[d]), b = floor(pmax[d]);
    a = fmax(a, 0.0);
    b = fmin(b, (double)(dims[d] - 1));
    if (!(a <= b)) return false;
    r[2 * d] = (int)a;
    r[2 * d + 1] = (int)b;
  }
  rc.i0 = (int16_t)r[0];
  rc.i1 = (int16_t)r[1];
  rc.j0 = (int16_t)r[2];
  rc.j1 = (int16_t)r[3];
  return true;
}

}  // namespace rc
