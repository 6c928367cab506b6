// cast_curved.cu -- the segment kernel for curved (R = 2) trees: rows a4
// (intersection), a5 (GL segment integration) and a6 (on-chip fold) of
// SURVEY.md §8(a), for C3-C5, fused into one persistent kernel
// (k_cast_curved<P,N>, described at its definition below and in DESIGN.md
// §6.1).  Building blocks, in file order:
//  - Bernstein evaluation of the element map X_E (relative to the element
//    origin) and of a face patch; the padded shared-memory slot layout;
//  - the projected-patch root finding of App. A.1:
//    Bezier hull rejection, injectivity bound ||A J(s) - I|| < 1, chord /
//    Newton iteration, Bezier subdivision (rare: grazing rays);
//  - element preparation (fp64 restriction of the tree's Bernstein points to
//    the element's subcube; the affine model and its
//    nonlinearity bounds);
//  - phase 1 (per 32 packed candidate pairs), phase 2 (per 32 items),
//    phase 3 (bucket fold per unit) and the kernel.
#include <cuda_runtime.h>
#include <math.h>

#include "device_math.cuh"
#include "kernels.cuh"

namespace rc {

namespace {

constexpr int WARPS = 4;
constexpr float FACE_TOL = 2e-6f;   // accepted face-parameter overshoot (~20x fp32 rounding of s)

struct RootRec {
  float beta;
  float xi[3];
};

__device__ __forceinline__ void bern(float t, float& b0, float& b1, float& b2) {
  float u = 1.0f - t;
  b0 = u * u;
  b1 = 2.0f * t * u;
  b2 = t * t;
}
__device__ __forceinline__ void dbern(float t, float& d0, float& d1, float& d2) {
  d0 = 2.0f * t - 2.0f;
  d1 = 2.0f - 4.0f * t;
  d2 = 2.0f * t;
}

// Element slot layout in shared memory (floats, 16-byte aligned rows): the
// 27 Bernstein points relative to the element origin as 9 rows (m3, m2) of
// 3 points (m1) x 3 coordinates padded to 12 floats; the nodal field (P = 2:
// 3 rows of 9 values padded to 12; P = 1: 8 values); the affine model.
__host__ __device__ constexpr int GI(int m) { return (m / 3) * 12 + (m % 3) * 3; }   // point m = (m3*3+m2)*3+m1
__host__ __device__ constexpr int FI(int q, int NF) { return NF == 27 ? (q / 9) * 12 + q % 9 : q; }
constexpr int SLOT_FIELD = 108;
constexpr int SLOT_AFF = 144;      // Xc[3], J0inv[9], dp[3], eta
constexpr int SLOT_STRIDE = 164;   // 160 used; 164 mod 32 = 4 spreads slot banks, 656 B keeps 16-B alignment
constexpr int SLOT_USED = 160;     // floats of a slot in the global slot buffer (640 B, one bulk copy)

// one row (m3, m2) of 3 points by three 16-byte loads
__device__ __forceinline__ void load_row(const float* __restrict__ sB, int row, float p0[3], float p1[3], float p2[3]) {
  const float4* r = reinterpret_cast<const float4*>(sB + row * 12);
  const float4 v0 = r[0], v1 = r[1], v2 = r[2];
  p0[0] = v0.x; p0[1] = v0.y; p0[2] = v0.z;
  p1[0] = v0.w; p1[1] = v1.x; p1[2] = v1.y;
  p2[0] = v1.z; p2[1] = v1.w; p2[2] = v2.x;
}

// X_E(xi) - C_E (tensor Bernstein form of the degree-2 element map).
__device__ __forceinline__ void eval_X(const float* __restrict__ sB, const float xi[3], float X[3]) {
  float a0, a1, a2, b0, b1, b2, c0, c1, c2;
  bern(xi[0], a0, a1, a2);
  bern(xi[1], b0, b1, b2);
  bern(xi[2], c0, c1, c2);
  const float bb[3] = {b0, b1, b2}, cc[3] = {c0, c1, c2};
  X[0] = X[1] = X[2] = 0.0f;
#pragma unroll
  for (int m3 = 0; m3 < 3; ++m3) {
    float y[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int m2 = 0; m2 < 3; ++m2) {
      float p0[3], p1[3], p2[3];
      load_row(sB, m3 * 3 + m2, p0, p1, p2);
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = fmaf(bb[m2], fmaf(a2, p2[c], fmaf(a1, p1[c], a0 * p0[c])), y[c]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) X[c] = fmaf(cc[m3], y[c], X[c]);
  }
}

// Two points at once (independent FMA chains, each control point loaded once).
__device__ __forceinline__ void eval_X2(const float* __restrict__ sB, const float xa[3], const float xb[3], float XA[3],
                                        float XB[3]) {
  float a[3], b[3], c[3], e[3], g[3], h[3];
  bern(xa[0], a[0], a[1], a[2]);
  bern(xa[1], b[0], b[1], b[2]);
  bern(xa[2], c[0], c[1], c[2]);
  bern(xb[0], e[0], e[1], e[2]);
  bern(xb[1], g[0], g[1], g[2]);
  bern(xb[2], h[0], h[1], h[2]);
#pragma unroll
  for (int q = 0; q < 3; ++q) XA[q] = XB[q] = 0.0f;
#pragma unroll
  for (int m3 = 0; m3 < 3; ++m3) {
    float ya[3] = {0.f, 0.f, 0.f}, yb[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int m2 = 0; m2 < 3; ++m2) {
      float p0[3], p1[3], p2[3];
      load_row(sB, m3 * 3 + m2, p0, p1, p2);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        ya[q] = fmaf(b[m2], fmaf(a[2], p2[q], fmaf(a[1], p1[q], a[0] * p0[q])), ya[q]);
        yb[q] = fmaf(g[m2], fmaf(e[2], p2[q], fmaf(e[1], p1[q], e[0] * p0[q])), yb[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      XA[q] = fmaf(c[m3], ya[q], XA[q]);
      XB[q] = fmaf(h[m3], yb[q], XB[q]);
    }
  }
}

// Field at xi from the padded nodal values (node order [k3][k2][k1]).
template <int P>
__device__ __forceinline__ float field_pad(const float* __restrict__ f, float x1, float x2, float x3);
template <>
__device__ __forceinline__ float field_pad<1>(const float* __restrict__ f, float x1, float x2, float x3) {
  const float4 lo = reinterpret_cast<const float4*>(f)[0], hi = reinterpret_cast<const float4*>(f)[1];
  const float a00 = fmaf(x1, lo.y - lo.x, lo.x), a10 = fmaf(x1, lo.w - lo.z, lo.z);
  const float a01 = fmaf(x1, hi.y - hi.x, hi.x), a11 = fmaf(x1, hi.w - hi.z, hi.z);
  const float b0 = fmaf(x2, a10 - a00, a00), b1 = fmaf(x2, a11 - a01, a01);
  return fmaf(x3, b1 - b0, b0);
}
template <>
__device__ __forceinline__ float field_pad<2>(const float* __restrict__ f, float x1, float x2, float x3) {
  float p0, p1, p2, q0, q1, q2, r0, r1, r2;
  lag2(x1, p0, p1, p2);
  lag2(x2, q0, q1, q2);
  lag2(x3, r0, r1, r2);
  const float rr[3] = {r0, r1, r2};
  float out = 0.0f;
#pragma unroll
  for (int k3 = 0; k3 < 3; ++k3) {
    float g[9];
    load_row(f, k3, g, g + 3, g + 6);
    const float s0 = fmaf(p2, g[2], fmaf(p1, g[1], p0 * g[0]));
    const float s1 = fmaf(p2, g[5], fmaf(p1, g[4], p0 * g[3]));
    const float s2 = fmaf(p2, g[8], fmaf(p1, g[7], p0 * g[6]));
    out = fmaf(rr[k3], fmaf(q2, s2, fmaf(q1, s1, q0 * s0)), out);
  }
  return out;
}

// X_E on face (axis k fixed): 9 Bernstein points at padded float offsets
// base + ia*sa + jb*sb (offset of point (m1,m2,m3) = 3 m1 + 12 m2 + 36 m3).
__device__ __forceinline__ void eval_face(const float* __restrict__ sB, int base, int sa, int sb, float s1, float s2,
                                          float X[3]) {
  float a0, a1, a2, b0, b1, b2;
  bern(s1, a0, a1, a2);
  bern(s2, b0, b1, b2);
  const float bb[3] = {b0, b1, b2};
  X[0] = X[1] = X[2] = 0.0f;
#pragma unroll
  for (int jb = 0; jb < 3; ++jb) {
    const float* p0 = sB + base + jb * sb;
    const float* p1 = p0 + sa;
    const float* p2 = p1 + sa;
#pragma unroll
    for (int c = 0; c < 3; ++c) X[c] = fmaf(bb[jb], fmaf(a2, p2[c], fmaf(a1, p1[c], a0 * p0[c])), X[c]);
  }
}


__device__ __forceinline__ bool inv3(const float J[3][3], float I[3][3]) {
  float c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  float c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  float c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  float det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  if (!(fabsf(det) > 0.0f)) return false;
  float id = 1.0f / det;
  I[0][0] = c00 * id;
  I[1][0] = c01 * id;
  I[2][0] = c02 * id;
  I[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
  I[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
  I[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
  I[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
  I[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
  I[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  return true;
}

// ---- 2D biquadratic patch G(s) = sum g[j][i] B_i(s1) B_j(s2) (g: [9][2]) ----
struct Patch {
  float gx[9], gy[9];
};

__device__ __forceinline__ void patch_eval(const Patch& p, float s1, float s2, float& Gx, float& Gy, float& J11,
                                           float& J12, float& J21, float& J22) {
  float a0, a1, a2, b0, b1, b2, da0, da1, da2, db0, db1, db2;
  bern(s1, a0, a1, a2);
  bern(s2, b0, b1, b2);
  dbern(s1, da0, da1, da2);
  dbern(s2, db0, db1, db2);
  const float bb[3] = {b0, b1, b2}, dbb[3] = {db0, db1, db2};
  Gx = Gy = J11 = J12 = J21 = J22 = 0.0f;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float vx = fmaf(a2, p.gx[3 * j + 2], fmaf(a1, p.gx[3 * j + 1], a0 * p.gx[3 * j]));
    float vy = fmaf(a2, p.gy[3 * j + 2], fmaf(a1, p.gy[3 * j + 1], a0 * p.gy[3 * j]));
    float dx = fmaf(da2, p.gx[3 * j + 2], fmaf(da1, p.gx[3 * j + 1], da0 * p.gx[3 * j]));
    float dy = fmaf(da2, p.gy[3 * j + 2], fmaf(da1, p.gy[3 * j + 1], da0 * p.gy[3 * j]));
    Gx = fmaf(bb[j], vx, Gx);
    Gy = fmaf(bb[j], vy, Gy);
    J11 = fmaf(bb[j], dx, J11);
    J21 = fmaf(bb[j], dy, J21);
    J12 = fmaf(dbb[j], vx, J12);
    J22 = fmaf(dbb[j], vy, J22);
  }
}

__device__ __forceinline__ bool hull_excludes_origin(const Patch& p) {
  float xmn = p.gx[0], xmx = p.gx[0], ymn = p.gy[0], ymx = p.gy[0];
#pragma unroll
  for (int q = 1; q < 9; ++q) {
    xmn = fminf(xmn, p.gx[q]);
    xmx = fmaxf(xmx, p.gx[q]);
    ymn = fminf(ymn, p.gy[q]);
    ymx = fmaxf(ymx, p.gy[q]);
  }
  return xmn > 0.0f || xmx < 0.0f || ymn > 0.0f || ymx < 0.0f;
}

// Provable injectivity on the patch: with A = J(1/2,1/2)^-1 and the Bernstein
// coefficients of dG/ds1 (2(g[j][i+1]-g[j][i])) and dG/ds2 (2(g[j+1][i]-g[j][i])),
// every J(s) = [conv(d1), conv(d2)] so ||A J(s) - I||_1 <= q; q < 1 means
// G(s) - G(s') = (I + E)(s - s') != 0: at most one root.  Returns q.
__device__ __forceinline__ float injectivity_bound(const Patch& p, float& A11, float& A12, float& A21, float& A22,
                                                   float& Gcx, float& Gcy) {
  float J11, J12, J21, J22;
  patch_eval(p, 0.5f, 0.5f, Gcx, Gcy, J11, J12, J21, J22);
  float det = J11 * J22 - J12 * J21;
  if (!(fabsf(det) > 0.0f)) return 1e30f;
  float id = 1.0f / det;
  A11 = J22 * id;
  A12 = -J12 * id;
  A21 = -J21 * id;
  A22 = J11 * id;
  float q1 = 0.0f, q2 = 0.0f;
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      float dx = 2.0f * (p.gx[3 * j + i + 1] - p.gx[3 * j + i]);
      float dy = 2.0f * (p.gy[3 * j + i + 1] - p.gy[3 * j + i]);
      float e1 = fmaf(A11, dx, A12 * dy) - 1.0f, e2 = fmaf(A21, dx, A22 * dy);
      q1 = fmaxf(q1, fabsf(e1) + fabsf(e2));
    }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      float dx = 2.0f * (p.gx[3 * (j + 1) + i] - p.gx[3 * j + i]);
      float dy = 2.0f * (p.gy[3 * (j + 1) + i] - p.gy[3 * j + i]);
      float e1 = fmaf(A11, dx, A12 * dy), e2 = fmaf(A21, dx, A22 * dy) - 1.0f;
      q2 = fmaxf(q2, fabsf(e1) + fabsf(e2));
    }
  return fmaxf(q1, q2);
}

// Newton on the patch (local coordinates), started at `s`.  Returns true when
// converged; s receives the root.
__device__ __forceinline__ bool patch_newton(const Patch& p, float& s1, float& s2, float tol, int max_it) {
  for (int it = 0; it < max_it; ++it) {
    float Gx, Gy, J11, J12, J21, J22;
    patch_eval(p, s1, s2, Gx, Gy, J11, J12, J21, J22);
    float det = J11 * J22 - J12 * J21;
    if (!(fabsf(det) > 0.0f)) return false;
    float id = 1.0f / det;
    float d1 = (J22 * Gx - J12 * Gy) * id, d2 = (J11 * Gy - J21 * Gx) * id;
    s1 -= d1;
    s2 -= d2;
    if (!(fabsf(s1) < 8.0f && fabsf(s2) < 8.0f)) return false;
    if (fabsf(d1) < tol && fabsf(d2) < tol) return true;
  }
  return false;
}

// de Casteljau split of a patch at 1/2 along s1 (dir 0) or s2 (dir 1)
__device__ void patch_split(const Patch& p, int dir, Patch& lo, Patch& hi) {
#pragma unroll
  for (int o = 0; o < 3; ++o) {
    int i0 = dir == 0 ? 3 * o : o, st = dir == 0 ? 1 : 3;
    float x0 = p.gx[i0], x1 = p.gx[i0 + st], x2 = p.gx[i0 + 2 * st];
    float y0 = p.gy[i0], y1 = p.gy[i0 + st], y2 = p.gy[i0 + 2 * st];
    float x01 = 0.5f * (x0 + x1), x12 = 0.5f * (x1 + x2), xm = 0.5f * (x01 + x12);
    float y01 = 0.5f * (y0 + y1), y12 = 0.5f * (y1 + y2), ym = 0.5f * (y01 + y12);
    lo.gx[i0] = x0; lo.gx[i0 + st] = x01; lo.gx[i0 + 2 * st] = xm;
    lo.gy[i0] = y0; lo.gy[i0 + st] = y01; lo.gy[i0 + 2 * st] = ym;
    hi.gx[i0] = xm; hi.gx[i0 + st] = x12; hi.gx[i0 + 2 * st] = x2;
    hi.gy[i0] = ym; hi.gy[i0 + st] = y12; hi.gy[i0 + 2 * st] = y2;
  }
}

// Root of an injective patch (q < 1, A = J(centre)^-1).  The chord map
// T(s) = s - A G(s) contracts towards the unique root s* in D = [0,1]^2 with
// factor q (1-norm) on D, so ||T(c) - s*||_1 <= q: if T(c) is farther than q
// from D, s* does not exist.  Otherwise Newton from T(c).
// Returns 1 (root in s1,s2), -1 (no root in D), 0 (not converged).
__device__ __forceinline__ int chord_root(const Patch& pt, float A11, float A12, float A21, float A22, float gcx,
                                          float gcy, float q, float tol, int max_it, float& s1, float& s2) {
  // first chord step from the centre: ||s1 - s*||_1 <= q ||c - s*||_1 <= q
  s1 = 0.5f - (A11 * gcx + A12 * gcy);
  s2 = 0.5f - (A21 * gcx + A22 * gcy);
  float dout = fmaxf(0.0f, -s1) + fmaxf(0.0f, s1 - 1.0f) + fmaxf(0.0f, -s2) + fmaxf(0.0f, s2 - 1.0f);
  if (dout > q + FACE_TOL) return -1;   // proof: the unique root is not in D
  // Newton from there (quadratic convergence also when q is close to 1)
  for (int it = 0; it < max_it; ++it) {
    float Gx, Gy, J11, J12, J21, J22;
    patch_eval(pt, s1, s2, Gx, Gy, J11, J12, J21, J22);
    float det = J11 * J22 - J12 * J21;
    if (!(fabsf(det) > 0.0f)) return 0;
    float id = 1.0f / det;
    float d1 = (J22 * Gx - J12 * Gy) * id, d2 = (J11 * Gy - J21 * Gx) * id;
    s1 -= d1;
    s2 -= d2;
    if (!(fabsf(s1 - 0.5f) < 4.0f && fabsf(s2 - 0.5f) < 4.0f)) return -1;   // left far from D
    if (fabsf(d1) < tol && fabsf(d2) < tol) return 1;
  }
  return 0;
}

// Face f's 9 Bernstein points (relative to the element origin) projected on
// the plane spanned by d1, d2 perpendicular to the ray, origin at the ray
// (Eq. intersectiontwod).
__device__ __forceinline__ void project_face(const float* __restrict__ sB, int f, const float d1[3],
                                             const float d2[3], float o1, float o2, Patch& pt) {
  const int k = f >> 1, side = f & 1;
  const int ka = (k + 1) % 3, kb = (k + 2) % 3;
  const int str[3] = {1, 3, 9};
  const int base = 2 * side * str[k], sa = str[ka], sbb = str[kb];
#pragma unroll
  for (int jb = 0; jb < 3; ++jb)
#pragma unroll
    for (int ia = 0; ia < 3; ++ia) {
      const int m = base + ia * sa + jb * sbb;
      const float bx = sB[GI(m)], by = sB[GI(m) + 1], bz = sB[GI(m) + 2];
      pt.gx[3 * jb + ia] = fmaf(d1[0], bx, fmaf(d1[1], by, fmaf(d1[2], bz, -o1)));
      pt.gy[3 * jb + ia] = fmaf(d2[0], bx, fmaf(d2[1], by, fmaf(d2[2], bz, -o2)));
    }
}

// All roots of a projected face patch by Bezier subdivision (App. A.1,
// PAPER.md:1481-1514).  Roots are written to u[2*t], u[2*t+1].
__device__ __noinline__ int face_roots_subdiv(const Patch& root, float tol, int max_it, float* u, int stride,
                                              int cap, int* fails) {
  struct Item {
    Patch p;
    float s1a, s2a, w;
  };
  Item stack[32];
  int top = 0, nr = 0;
  stack[top++] = Item{root, 0.0f, 0.0f, 1.0f};
  int visited = 0;
  while (top > 0) {
    Item it = stack[--top];
    if (hull_excludes_origin(it.p)) continue;
    ++visited;
    float A11, A12, A21, A22, gcx, gcy;
    float q = injectivity_bound(it.p, A11, A12, A21, A22, gcx, gcy);
    if (q < 1.0f) {
      float s1, s2;
      int st = chord_root(it.p, A11, A12, A21, A22, gcx, gcy, q, tol / it.w, max_it, s1, s2);
      if (st == 1) {
        float lt = FACE_TOL / it.w;
        if (s1 >= -lt && s1 <= 1.0f + lt && s2 >= -lt && s2 <= 1.0f + lt && nr < cap) {
          u[(2 * nr) * stride] = it.s1a + it.w * s1;
          u[(2 * nr + 1) * stride] = it.s2a + it.w * s2;
          ++nr;
        }
        continue;
      } else if (st == -1) {
        continue;
      } else if (it.w < 1.0f / 1024.0f || top > 28 || visited > 1024) {
        ++*fails;
        continue;
      }
      // not converged: split further (sub-patches have smaller q)
    } else if (it.w < 1.0f / 1024.0f || top > 28 || visited > 1024) {
      // depth limit without an injectivity proof (tangency): Newton from the centre
      float s1 = 0.5f, s2 = 0.5f;
      if (patch_newton(it.p, s1, s2, tol / it.w, max_it) && s1 >= -1e-3f && s1 <= 1.001f && s2 >= -1e-3f &&
          s2 <= 1.001f && nr < cap) {
        u[(2 * nr) * stride] = it.s1a + it.w * s1;
        u[(2 * nr + 1) * stride] = it.s2a + it.w * s2;
        ++nr;
      }
      continue;
    }
    Patch a, b, aa, ab, ba, bb;
    patch_split(it.p, 0, a, b);
    patch_split(a, 1, aa, ab);
    patch_split(b, 1, ba, bb);
    float h = 0.5f * it.w;
    stack[top++] = Item{aa, it.s1a, it.s2a, h};
    stack[top++] = Item{ab, it.s1a, it.s2a + h, h};
    stack[top++] = Item{ba, it.s1a + h, it.s2a, h};
    stack[top++] = Item{bb, it.s1a + h, it.s2a + h, h};
  }
  return nr;
}





// ---------------------------------------------------------------------------
// The fused segment kernel (rows a4 + a5 + a6 of SURVEY §8(a)).  Persistent
// CTAs of CWARPS warps take fold units from a global counter; a unit is a
// range of <= RC_UNIT_CHUNKS chunks of <= RC_UNIT_LEAVES visible leaves
// inside one node of the fold level (k_unit_* in kernels.cu).  Per unit:
//  phase 0: the unit's elements are prepared once into shared memory
//    (Bernstein points relative to the element origin, nodal field, affine
//    model and its nonlinearity bounds; warps take elements);
//  phase 1 (intersection): warps take the unit's chunks from a shared counter;
//    per chunk (32 candidate pixels of one element):
//    1a per lane: ray re-based near the element (fp64), affine prefilter and
//       the proof of "no root" per face -> candidate (pixel, face) tasks;
//    1b the chunk's face tasks in full warps (one task per lane): certified
//       affine-model iteration, else the projected-patch method of App. A.1;
//       roots go to the pixel's list in shared memory;
//    1c per lane: roots sorted by beta, deduplicated, paired entry/exit; each
//       inside interval becomes a 64-byte item in the CTA's scratch (L2):
//         float xin[3], xout[3]  entry / exit point relative to the element origin
//         float xiin[3], xiout[3] reference coordinates of entry / exit
//         float alpha_near, alpha_far; uint32 pixel; int32 visible index
//  phase 2 (integration): warps take 32 items at a time (full warps, no idle
//    lanes on misses) and integrate them with the N-point GL rule;
//  phase 3 (fold, fold level >= 1): the unit's segments are bucketed by
//    pixel in shared memory, ordered per pixel under a total order, and every
//    maximal run of touching segments of one pixel (|gap| <= 1e-6 max(1,
//    alpha)) is combined nearest-first with Eq. aggregate
//     into one record keyed by the node: the first levels of
//    the paper's coarsening done on chip.
//    Without folding every segment is a record keyed by its leaf.
// ---------------------------------------------------------------------------
#ifndef RC_CWARPS
#define RC_CWARPS 6   // A/B at C4 (s11): 4 x 3 CTAs 559.3 ms, 6 x 2 CTAs 552.6 ms, 12 x 1 CTA 605.3 ms
#endif
#ifndef RC_CAST_CTAS
#define RC_CAST_CTAS 2
#endif
constexpr int CWARPS = RC_CWARPS;   // warps per CTA
constexpr float FAST_Q = 0.7f;       // contraction bound below which a face root takes the certified fast path
constexpr int CAST_CTAS_PER_SM = RC_CAST_CTAS;  // resident CTAs per SM (launch bounds: 168 registers)
constexpr int MAXR = 8;                                   // face roots per (element, pixel) pair
constexpr int ITEM_CAP = (MAXR / 2) * RC_CHUNK * RC_UNIT_CHUNKS;   // <= MAXR/2 segments per pair
constexpr int MAXT = 6 * RC_CHUNK;                        // face tasks of one chunk
constexpr float FOLD_TAU = 1e-6f;
constexpr int PS_N = 14;                                  // per-pixel ray state (floats)

struct WarpIsect {
  float ps[PS_N][32];       // P0[3], rf[3], xl0[3], dl[3], alpha0, rr
  float roots[MAXR][4][32]; // [k][beta, xi0, xi1, xi2][lane]
  uint8_t rord[MAXR][32];   // per-lane sorted root order (1c)
  int nroots[32];
  int pw[32];               // element (unit slot) of each lane's pixel
  int queue[64];            // packed pairs kept by the fp32 prefilter
  int stats[2];             // face tasks, 2D-path tasks (flushed per unit)
  uint8_t task[MAXT];       // lane << 3 | face
};
constexpr int PIXCAP = 4096;   // pixels of a unit's bounding rectangle for the bucket fold
constexpr int FCAP = 4096;     // segments of a unit for the bucket fold
union PhaseSmem {              // per-phase scratch of phases 0-2
  WarpIsect isect[CWARPS];
  float scr[RC_MAX_N * CWARPS * 32];   // phase 2: per-thread node values
};
struct UnitMeta {
  double org[RC_UNIT_LEAVES][4];        // element origins (fp64; 32-B rows, bulk-copied)
  Rect16 rect[RC_UNIT_LEAVES];          // pixel rectangles of the unit's elements
  int32_t pa[RC_UNIT_LEAVES];           // first pair of each element in this unit (rect raster index)
  int32_t pstart[RC_UNIT_LEAVES + 1];   // prefix of the elements' pair counts in the unit
  uint8_t vmap[RC_UNIT_CHUNKS + 16];    // element of the first pair of each 32-pair chunk
  float Dc[RC_UNIT_LEAVES][3];          // (float)(origin - O0): prefilter ray re-basing
  float pm[RC_UNIT_LEAVES];             // prefilter margin in xi~ units
  float rwinv[RC_UNIT_LEAVES];          // 1 / rectangle width
};
struct Phase012 {
  float slot[RC_UNIT_LEAVES][SLOT_STRIDE];
  PhaseSmem ph;
};
struct FoldSmem {              // phase 3 (the slots are dead by then)
  float2 alpha[FCAP];          // (alpha_near, alpha_far) of every segment
  int off[PIXCAP + 1];         // per-pixel counts, then offsets
  uint16_t rank[FCAP];         // segment -> slot within its pixel
  uint16_t order[FCAP];        // pixel-bucketed segment indices
};
static_assert(sizeof(FoldSmem) <= sizeof(Phase012), "the fold's shared memory lives in the slots' space");
struct CastSmem {
  UnitMeta meta;
  union __align__(16) {   // the slots are read with 16-byte loads
    Phase012 p;
    FoldSmem fold;
  } u;
};
struct CastCtl {
  unsigned long long mbar;     // mbarrier of the unit's slot bulk copies
  int64_t unit;
  int64_t ubeg, uend;          // this launch's unit range (the batch's units)
  int next_chunk;
  int nitems;
  unsigned long long base;
  int warp_sum[CWARPS];
  int bb[4];                   // unit pixel bounding rectangle: -i0, i1, -j0, j1 (atomicMax)
};

// ---- bulk copies global -> shared, tracked by an mbarrier (sm_90+ async proxy) ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// generic-proxy accesses of shared memory before async-proxy writes into it
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- element preparation kernel -------------------------------------------
// Slots of the visible leaves [v0, v1) (v1 clipped to the visible count) into
// the global slot buffer (record v - v0: SLOT_USED floats + the fp64 origin as
// 4 doubles); the segment kernel stages a unit's records with bulk copies.
// PREP_E elements per CTA, three threads per element (warp c = coordinate c):
//  1. fp64: coordinate c of the 27 Bernstein points of X_E by restriction of
//     the tree's Bernstein points to the element's subcube (blossoms
//     (u,u), (u,u+h), (u+h,u+h) per axis, sum-factorised: axis 3, 2, 1),
//     stored fp32 relative to the origin B_(1,1,1);
//  2. fp32: row c of the affine model A(xi) = Xc + J0 (xi - 1/2) (Bernstein
//     coefficients at the centre);
//  3. fp32: J0^-1 (each thread), the bound dp_c of the nonlinear remainder in
//     J0^-1 coordinates and the part of eta (sup |dE/dxi|) along axis c;
//  then the slots are written out coalesced.
// Stages 2-3 of k_prep_slots for coordinate C (one warp per coordinate).
// One instance for the three coordinate warps (runtime, warp-uniform C): a
// third of the code of per-coordinate template instances (the prep kernel's
// top stall is instruction fetch; A/B at C4, s10: 38.6 -> 36.4 ms per frame).
__device__ __forceinline__ void prep_affine_rt(const float* __restrict__ slw, float* sJw, bool act, int C) {
  constexpr float wq[3] = {0.25f, 0.5f, 0.25f}, dq[3] = {-1.0f, 0.0f, 1.0f};
  if (act) {
    float xc = 0.f, j0 = 0.f, j1 = 0.f, j2 = 0.f;
#pragma unroll
    for (int m = 0; m < 27; ++m) {
      const int a1 = m % 3, a2 = (m / 3) % 3, a3 = m / 9;
      const float b = slw[GI(m) + C];
      xc = fmaf(wq[a1] * wq[a2] * wq[a3], b, xc);
      j0 = fmaf(dq[a1] * wq[a2] * wq[a3], b, j0);
      j1 = fmaf(wq[a1] * dq[a2] * wq[a3], b, j1);
      j2 = fmaf(wq[a1] * wq[a2] * dq[a3], b, j2);
    }
    sJw[C] = xc;
    sJw[3 + 3 * C] = j0;
    sJw[4 + 3 * C] = j1;
    sJw[5 + 3 * C] = j2;
  }
}
__device__ __forceinline__ void prep_bounds_rt(const float* __restrict__ slw, const float* sJw, float (*sbw)[3],
                                               float (&Ji)[3][3], bool act, int C) {
  if (!act) return;
  float J[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) J[i][a] = sJw[3 + 3 * i + a];
  const float Xc[3] = {sJw[0], sJw[1], sJw[2]};
  if (!inv3(J, Ji)) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int a = 0; a < 3; ++a) Ji[i][a] = 0.0f;
  }
  float JC[3];   // row C of J0^-1
#pragma unroll
  for (int a = 0; a < 3; ++a) JC[a] = C == 0 ? Ji[0][a] : (C == 1 ? Ji[1][a] : Ji[2][a]);
  const float e0C = C == 0 ? 1.0f : 0.0f, e1C = C == 1 ? 1.0f : 0.0f, e2C = C == 2 ? 1.0f : 0.0f;
  float dpc = 0.0f, eta = 0.0f;
#pragma unroll
  for (int m = 0; m < 27; ++m) {
    const int mmv[3] = {m % 3, (m / 3) % 3, m / 9};
    const float* b = slw + GI(m);
    const float x0 = 0.5f * mmv[0] - 0.5f, x1 = 0.5f * mmv[1] - 0.5f, x2 = 0.5f * mmv[2] - 0.5f;
    const float r0 = b[0] - (Xc[0] + J[0][0] * x0 + J[0][1] * x1 + J[0][2] * x2);
    const float r1 = b[1] - (Xc[1] + J[1][0] * x0 + J[1][1] * x1 + J[1][2] * x2);
    const float r2 = b[2] - (Xc[2] + J[2][0] * x0 + J[2][1] * x1 + J[2][2] * x2);
    dpc = fmaxf(dpc, fabsf(JC[0] * r0 + JC[1] * r1 + JC[2] * r2));
    // eta: Bernstein coefficients of dE/dxi_C = 2 J0^-1 (B_{m+e_C} - B_m) - e_C (inf-norm)
    const int mC = C == 0 ? mmv[0] : (C == 1 ? mmv[1] : mmv[2]);
    if (mC < 2) {
      const int nxt = C == 0 ? (mmv[0] < 2 ? GI(m + 1) : 0) : (C == 1 ? (mmv[1] < 2 ? GI(m + 3) : 0)
                                                                      : (mmv[2] < 2 ? GI(m + 9) : 0));
      const float* b2 = slw + nxt;
      const float e0 = 2.0f * (b2[0] - b[0]), e1 = 2.0f * (b2[1] - b[1]), e2 = 2.0f * (b2[2] - b[2]);
      const float t0 = Ji[0][0] * e0 + Ji[0][1] * e1 + Ji[0][2] * e2 - e0C;
      const float t1 = Ji[1][0] * e0 + Ji[1][1] * e1 + Ji[1][2] * e2 - e1C;
      const float t2 = Ji[2][0] * e0 + Ji[2][1] * e1 + Ji[2][2] * e2 - e2C;
      eta = fmaxf(eta, fmaxf(fabsf(t0), fmaxf(fabsf(t1), fabsf(t2))));
    }
  }
  sbw[0][C] = dpc;
  sbw[1][C] = eta;
}

constexpr int PREP_E = 32;
#ifndef RC_PREP_CTAS
#define RC_PREP_CTAS 4   // A/B at C4 (s8): 4 = 38.6, 5 = 40.1, 6 = 41.2 ms of prep per frame
#endif
constexpr int PREP_CTAS_PER_SM = RC_PREP_CTAS;   // <= 128 registers x 96 threads; ~31 KB shared memory
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Persistent CTAs over groups of PREP_E visible leaves, software-pipelined:
// while group g is computed, the keys and nodal field of group g + G and the
// visible-list entries of group g + 2G (G = gridDim.x) are in flight as
// cp.async copies into the other buffer (the loads are dependent gathers,
// vis -> leaf -> field, that 15 resident warps per SM cannot hide otherwise).
template <int P>
__global__ void __launch_bounds__(3 * PREP_E, PREP_CTAS_PER_SM) k_prep_slots(
    const TreeConst* __restrict__ trees, DevLeafView L, const int32_t* __restrict__ vis,
    const int64_t* __restrict__ nvis_p, int64_t v0, int64_t v1, float4* __restrict__ gslot,
    double* __restrict__ gorg) {
  constexpr int NF = (P + 1) * (P + 1) * (P + 1);
  // rows of SLOT_STRIDE floats keep the 16-byte write-out (an odd stride, free of the 4-way
  // bank conflicts of the per-lane row reads, needs scalar stores: 39.7 -> 44.8 ms per C4 frame)
  __shared__ __align__(16) float sl[PREP_E][SLOT_STRIDE];
  __shared__ float sfb[2][PREP_E][NF];   // nodal fields in flight (copied into the slots per group)
  __shared__ double so[PREP_E][4];
  __shared__ float sJ[PREP_E][12];     // Xc[3], J[3][3]
  __shared__ float sb[PREP_E][2][3];   // per coordinate thread: dp_c, eta part
  __shared__ int32_t seb[2][PREP_E];   // visible-list entries (leaf indices) of the next two groups
  __shared__ int32_t skb[2][PREP_E][6];  // tree, level word, anchor[3], level byte offset
  const int64_t vend = min(v1, *nvis_p);
  const int64_t ngroups = (vend - v0 + PREP_E - 1) / PREP_E;
  const int64_t G = gridDim.x;
  const int c = threadIdx.x >> 5, w = threadIdx.x & 31;
  auto group_n = [&](int64_t g) -> int { return (int)min((int64_t)PREP_E, vend - (v0 + g * PREP_E)); };
  // stage the visible-list entries of group g into seb[b]
  auto issue_vis = [&](int64_t g, int b) {
    if (g < ngroups && threadIdx.x < group_n(g)) cp_async4(&seb[b][threadIdx.x], &vis[v0 + g * PREP_E + threadIdx.x]);
  };
  // stage keys and field of group g (leaf indices in seb[b]) into buffer b
  auto issue_data = [&](int64_t g, int b) {
    if (g >= ngroups) return;
    const int nl = group_n(g);
    for (int k = threadIdx.x; k < nl * 5; k += 3 * PREP_E) {
      const int ew = k / 5, q = k - ew * 5;
      const int64_t e = seb[b][ew];
      const void* src = q == 0 ? (const void*)&L.tree[e]
                        : (q == 1 ? (const void*)(L.level + (e & ~(int64_t)3)) : (const void*)&L.anchor[3 * e + q - 2]);
      cp_async4(&skb[b][ew][q], src);
    }
    for (int k = threadIdx.x; k < nl * NF; k += 3 * PREP_E) {
      const int ew = k / NF, q = k - ew * NF;
      cp_async4(&sfb[b][ew][q], &L.field[(int64_t)seb[b][ew] * NF + q]);
    }
  };
  int64_t g = blockIdx.x;
  if (g >= ngroups) return;
  // prologue: entries of g and g + G, data of g
  issue_vis(g, 0);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  issue_data(g, 0);
  issue_vis(g + G, 1);
  cp_async_commit();
  for (int cb = 0; g < ngroups; g += G, cb ^= 1) {
    const int nb = cb ^ 1;
    cp_async_wait_all();
    __syncthreads();   // group g's data and group g + G's entries have landed
    const int nloc = group_n(g);
    const int64_t vb = v0 + g * PREP_E;
    if (threadIdx.x < PREP_E) skb[cb][threadIdx.x][5] = (int32_t)(seb[cb][threadIdx.x] & 3);
    for (int k = threadIdx.x; k < nloc * NF; k += 3 * PREP_E) {
      const int ew = k / NF, q = k - ew * NF;
      sl[ew][SLOT_FIELD + FI(q, NF)] = sfb[cb][ew][q];
    }
    issue_data(g + G, nb);      // the next group's gathers fly while this one computes
    __syncthreads();
    issue_vis(g + 2 * G, cb);   // seb[cb] is free once the level offsets are taken
    cp_async_commit();
    const bool act = w < nloc;
    float* slw = sl[w];
    // 1. restriction (fp64), coordinate c
    if (act) {
      const double h = ldexp(1.0, -(int)(int8_t)(skb[cb][w][1] >> (8 * skb[cb][w][5])));
      const double* __restrict__ Bw = trees[skb[cb][w][0]].Bw;   // [q3][q2][q1][xyz]
      double uu[3];
  #pragma unroll
      for (int k = 0; k < 3; ++k) uu[k] = ldexp((double)skb[cb][w][2 + k], -RC_MAXLEVEL);
      auto Mrow = [&](int k, int r, double m[3]) {   // blossom row r of axis k
        const double u = uu[k], v = u + h;
        const double x = r == 2 ? v : u, y = r == 0 ? u : v;
        m[0] = (1 - x) * (1 - y);
        m[1] = (1 - x) * y + x * (1 - y);
        m[2] = x * y;
      };
      double m0[3], m1[3], m2[3];
      Mrow(0, 1, m0);
      Mrow(1, 1, m1);
      Mrow(2, 1, m2);
      double o = 0.0;   // origin = point (1,1,1)
  #pragma unroll
      for (int q3 = 0; q3 < 3; ++q3)
  #pragma unroll
        for (int q2 = 0; q2 < 3; ++q2) {
          const double w23 = m2[q3] * m1[q2];
  #pragma unroll
          for (int q1 = 0; q1 < 3; ++q1) o = fma(w23 * m0[q1], Bw[((q3 * 3 + q2) * 3 + q1) * 3 + c], o);
        }
      so[w][c] = o;
      if (c == 0) so[w][3] = 0.0;
      double M0[3][3];
  #pragma unroll
      for (int r = 0; r < 3; ++r) Mrow(0, r, M0[r]);
  #pragma unroll
      for (int r3 = 0; r3 < 3; ++r3) {
        double m3[3];
        Mrow(2, r3, m3);
        double T2[9];
  #pragma unroll
        for (int q21 = 0; q21 < 9; ++q21) {
          double acc = 0.0;
  #pragma unroll
          for (int q3 = 0; q3 < 3; ++q3) acc = fma(m3[q3], Bw[(q3 * 9 + q21) * 3 + c], acc);
          T2[q21] = acc;
        }
  #pragma unroll
        for (int r2 = 0; r2 < 3; ++r2) {
          double mm2[3];
          Mrow(1, r2, mm2);
          double T1[3];
  #pragma unroll
          for (int q1 = 0; q1 < 3; ++q1) {
            double acc = 0.0;
  #pragma unroll
            for (int q2 = 0; q2 < 3; ++q2) acc = fma(mm2[q2], T2[q2 * 3 + q1], acc);
            T1[q1] = acc;
          }
  #pragma unroll
          for (int r1 = 0; r1 < 3; ++r1) {
            double acc = 0.0;
  #pragma unroll
            for (int q1 = 0; q1 < 3; ++q1) acc = fma(M0[r1][q1], T1[q1], acc);
            slw[GI((r3 * 3 + r2) * 3 + r1) + c] = (float)(acc - o);
          }
        }
      }
    }
    __syncthreads();
    // 2. affine model at the centre, row c (fp32); 3. J0^-1, dp_c and the eta
    // part along axis c.  Per coordinate a fully unrolled instance (constant
    // indices: no integer division or selects in the loops over the 27 points).
    prep_affine_rt(slw, sJ[w], act, c);
    __syncthreads();
    float Ji[3][3];
    prep_bounds_rt(slw, sJ[w], sb[w], Ji, act, c);
    __syncthreads();
    if (act && c == 0) {
      float* af = slw + SLOT_AFF;
      af[0] = sJ[w][0];
      af[1] = sJ[w][1];
      af[2] = sJ[w][2];
  #pragma unroll
      for (int i = 0; i < 3; ++i)
  #pragma unroll
        for (int a = 0; a < 3; ++a) af[3 + 3 * i + a] = Ji[i][a];
      // inflate by a rounding margin relative to the element (fp32)
      af[12] = sb[w][0][0] * 1.001f + 1e-5f;
      af[13] = sb[w][0][1] * 1.001f + 1e-5f;
      af[14] = sb[w][0][2] * 1.001f + 1e-5f;
      af[15] = fmaxf(sb[w][1][0], fmaxf(sb[w][1][1], sb[w][1][2])) * 1.001f + 1e-5f;
    }
    __syncthreads();
    constexpr int Q = SLOT_USED / 4;   // float4 per slot
    float4* dst = gslot + (vb - v0) * Q;
    for (int k = threadIdx.x; k < nloc * Q; k += 3 * PREP_E) dst[k] = reinterpret_cast<const float4*>(sl[k / Q])[k % Q];
    double* od = gorg + (vb - v0) * 4;
    for (int k = threadIdx.x; k < nloc * 4; k += 3 * PREP_E) od[k] = so[k / 4][k % 4];
  }
  cp_async_wait_all();
}

// per-CTA global scratch (bytes)
constexpr size_t SCR_ITEMS = (size_t)ITEM_CAP * 64;
constexpr size_t SCR_SEGS = (size_t)ITEM_CAP * sizeof(rc_seg);
constexpr size_t SCR_PER_CTA = SCR_ITEMS + SCR_SEGS;

// Scratch lines of a finished unit are dead: drop them from L2 without a
// write-back (they would otherwise reach HBM as ~100 B per segment).
__device__ __forceinline__ void discard_l2(const void* base, size_t bytes) {
  const char* p = reinterpret_cast<const char*>(base);
  for (size_t off = (size_t)threadIdx.x * 128; off < bytes; off += (size_t)blockDim.x * 128)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + off) : "memory");
}

// output records: streaming stores (evict-first; they are not re-read by this kernel)
__device__ __forceinline__ void store_seg_cs(rc_seg* dst, uint32_t pixel, float an, float af, float a,
                                             const float b[3], uint32_t key) {
  float4* d = reinterpret_cast<float4*>(dst);
  __stcs(d, make_float4(__uint_as_float(pixel), an, af, a));
  __stcs(d + 1, make_float4(b[0], b[1], b[2], __uint_as_float(key)));
}

// warp-aggregated append on a shared-memory counter
__device__ __forceinline__ int warp_append_smem(int* counter, int want) {
  const unsigned lane = threadIdx.x & 31;
  int incl = want;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if ((int)lane >= off) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 31 && total > 0) base = atomicAdd(counter, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - want;
}

__device__ __forceinline__ void push_root(WarpIsect& W, int pl, float beta, const float xi[3], int& face_fail) {
  const int k = atomicAdd(&W.nroots[pl], 1);
  if (k >= MAXR) {
    ++face_fail;
    return;
  }
  W.roots[k][0][pl] = beta;
  W.roots[k][1][pl] = xi[0];
  W.roots[k][2][pl] = xi[1];
  W.roots[k][3][pl] = xi[2];
}

// Rigorous 2D path of one (pixel, face) task (App. A.1):
// project the face on d1, d2 perpendicular to r, reject by the Bezier hull,
// prove injectivity and iterate, else subdivide.  Out of line: ~1% of tasks.
__device__ __noinline__ void face_2d(WarpIsect& W, const float* __restrict__ sB, int pl, int f, const float tP0[3],
                                     const float trf[3], float trr, float tol, int max_it, int& face_fail) {
  const int fk = f >> 1, fside = f & 1;
  const int fa = (fk + 1) % 3, fb = (fk + 2) % 3;
  // rigorous 2D path (App. A.1): project the face on d1, d2 perpendicular to r
  float ax[3] = {0.f, 0.f, 0.f};
  {
    const float a0 = fabsf(trf[0]), a1 = fabsf(trf[1]), a2 = fabsf(trf[2]);
    ax[(a0 <= a1 && a0 <= a2) ? 0 : (a1 <= a2 ? 1 : 2)] = 1.0f;
  }
  float d1[3] = {trf[1] * ax[2] - trf[2] * ax[1], trf[2] * ax[0] - trf[0] * ax[2],
                 trf[0] * ax[1] - trf[1] * ax[0]};
  const float n1 = rsqrtf(d1[0] * d1[0] + d1[1] * d1[1] + d1[2] * d1[2]);
  d1[0] *= n1; d1[1] *= n1; d1[2] *= n1;
  float d2[3] = {trf[1] * d1[2] - trf[2] * d1[1], trf[2] * d1[0] - trf[0] * d1[2],
                 trf[0] * d1[1] - trf[1] * d1[0]};
  const float n2 = rsqrtf(d2[0] * d2[0] + d2[1] * d2[1] + d2[2] * d2[2]);
  d2[0] *= n2; d2[1] *= n2; d2[2] *= n2;
  const float o1 = d1[0] * tP0[0] + d1[1] * tP0[1] + d1[2] * tP0[2];
  const float o2 = d2[0] * tP0[0] + d2[1] * tP0[1] + d2[2] * tP0[2];
  Patch pt;
  project_face(sB, f, d1, d2, o1, o2, pt);
  if (!hull_excludes_origin(pt)) {
    float su[8];
    int nf = 0;
    float A11, A12, A21, A22, gcx, gcy;
    const float q = injectivity_bound(pt, A11, A12, A21, A22, gcx, gcy);
    int st = 0;
    float s1 = 0.f, s2 = 0.f;
    if (q < 1.0f) st = chord_root(pt, A11, A12, A21, A22, gcx, gcy, q, tol, max_it, s1, s2);
    if (st == 1) {
      if (s1 >= -FACE_TOL && s1 <= 1.0f + FACE_TOL && s2 >= -FACE_TOL && s2 <= 1.0f + FACE_TOL) {
        su[0] = s1;
        su[1] = s2;
        nf = 1;
      }
    } else if (st == 0) {
      nf = face_roots_subdiv(pt, tol, max_it, su, 1, 4, &face_fail);
    }
    for (int z = 0; z < nf; ++z) {
      float xi[3];
      xi[fk] = (float)fside;
      xi[fa] = fminf(fmaxf(su[2 * z], 0.0f), 1.0f);
      xi[fb] = fminf(fmaxf(su[2 * z + 1], 0.0f), 1.0f);
      float X[3];
      eval_X(sB, xi, X);
      const float beta =
          ((X[0] - tP0[0]) * trf[0] + (X[1] - tP0[1]) * trf[1] + (X[2] - tP0[2]) * trf[2]) / trr;
      push_root(W, pl, beta, xi, face_fail);
    }
  }
}

// ---- phase 1: one chunk (32 candidate pixels of one element) --------------
// The unit's candidate pairs are packed across its elements: pair g of the
// unit belongs to the element w with pstart[w] <= g < pstart[w+1], pixel
// pa[w] + g - pstart[w] of its rectangle (row-major).  A warp takes 32
// consecutive pairs, so small elements (a few pixels each at C4/C5) do not
// leave most lanes idle.
// p = q rw + r for 0 <= p < 2^24 with a float reciprocal (exact after one correction)
__device__ __forceinline__ void divmod_rw(int p, int rw, float rinv, int& q, int& r) {
  q = (int)(((float)p + 0.5f) * rinv);
  r = p - q * rw;
  if (r < 0) { --q; r += rw; }
  else if (r >= rw) { ++q; r -= rw; }
}

__device__ __forceinline__ int pair_element(const CastSmem& S, int g) {
  int w = S.meta.vmap[g / RC_CHUNK];   // the chunk's first element, then forward (1-2 steps at C4)
  while (S.meta.pstart[w + 1] <= g) ++w;
  return w;
}

// Conservative fp32 version of 1a's prefilter: the line of
// pair g in xi~ coordinates must meet the element's box inflated by dp and by
// a margin pm that covers the fp32 re-basing error; keeps every pair the
// exact prefilter keeps.
__device__ __forceinline__ bool prefilter_f32(const CastSmem& S, const CamConst& cc, int g) {
  const int w = pair_element(S, g);
  const float* af = S.u.p.slot[w] + SLOT_AFF;
  const Rect16 r = S.meta.rect[w];
  const int rw = r.i1 - r.i0 + 1;
  const int p = S.meta.pa[w] + g - S.meta.pstart[w];
  int pq, pr;
  divmod_rw(p, rw, S.meta.rwinv[w], pq, pr);
  const float di = (float)(r.i0 + pr) - 0.5f * (cc.W - 1), dj = (float)(r.j0 + pq) - 0.5f * (cc.H - 1);
  float rf[3], D[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    rf[k] = fmaf(dj, cc.f_Ru[k], fmaf(di, cc.f_Rt[k], cc.f_R0[k]));
    D[k] = S.meta.Dc[w][k] - fmaf(dj, cc.f_Ou[k], di * cc.f_Ot[k]);
  }
  const float rr = rf[0] * rf[0] + rf[1] * rf[1] + rf[2] * rf[2];
  const float a0 = (D[0] * rf[0] + D[1] * rf[1] + D[2] * rf[2]) / rr;
  const float q0 = fmaf(a0, rf[0], -D[0]) - af[0], q1 = fmaf(a0, rf[1], -D[1]) - af[1],
              q2 = fmaf(a0, rf[2], -D[2]) - af[2];
  const float m = S.meta.pm[w];
  float ben = -3.4e38f, bex = 3.4e38f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float x0 = 0.5f + af[3 + 3 * k] * q0 + af[4 + 3 * k] * q1 + af[5 + 3 * k] * q2;
    const float dl = af[3 + 3 * k] * rf[0] + af[4 + 3 * k] * rf[1] + af[5 + 3 * k] * rf[2];
    const float lo = -af[12 + k] - m - x0, hi = 1.0f + af[12 + k] + m - x0;
    if (dl == 0.0f) {
      if (lo > 0.0f || hi < 0.0f) return false;
      continue;
    }
    const float inv = 1.0f / dl, ta = lo * inv, tb = hi * inv;
    ben = fmaxf(ben, fminf(ta, tb));
    bex = fminf(bex, fmaxf(ta, tb));
  }
  return bex >= ben;
}

__device__ __forceinline__ void isect_chunk(WarpIsect& W, CastSmem& S, const CamConst& cc, int nvis, int vfirst,
                                            int g, float4* __restrict__ items, int* s_nitems,
                                            int32_t* __restrict__ hits_pp, int& local_hits, int& face_fail) {
  const unsigned lane = threadIdx.x & 31;
  const float tol = cc.newton_tol;
  const int max_it = cc.newton_max;
  const bool active = g >= 0 && g < S.meta.pstart[nvis];
  const int w = active ? pair_element(S, g) : 0;
  const float* sB = S.u.p.slot[w];
  const double* org = S.meta.org[w];
  const Rect16 r = S.meta.rect[w];
  const int v = vfirst + w;
  const float* af = sB + SLOT_AFF;
  const float dpv[3] = {af[12], af[13], af[14]};
  const float dpm = fmaxf(dpv[0], fmaxf(dpv[1], dpv[2]));
  const int rw = r.i1 - r.i0 + 1;
  const int p = S.meta.pa[w] + (active ? g : 0) - S.meta.pstart[w];
  int pq, pr;
  divmod_rw(p, rw, S.meta.rwinv[w], pq, pr);
  const int i = r.i0 + pr, j = r.j0 + pq;

  // ---- 1a: ray of pixel (i,j), re-based near the element (fp64) -----------
  const double di = (double)i - 0.5 * (cc.W - 1), dj = (double)j - 0.5 * (cc.H - 1);
  double Rw[3], D[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    Rw[k] = fma(dj, cc.Ru[k], fma(di, cc.Rt[k], cc.R0[k]));
    const double O = fma(dj, cc.Ou[k], fma(di, cc.Ot[k], cc.O0[k]));
    D[k] = org[k] - O;
  }
  const float rf[3] = {(float)Rw[0], (float)Rw[1], (float)Rw[2]};
  const float rr = rf[0] * rf[0] + rf[1] * rf[1] + rf[2] * rf[2];
  const float alpha0 = ((float)D[0] * rf[0] + (float)D[1] * rf[1] + (float)D[2] * rf[2]) / rr;
  float P0[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) P0[k] = (float)fma((double)alpha0, Rw[k], -D[k]);
  // affine prefilter in xi~ = J0^-1 coordinates: line xl(beta) = xl0 + beta dl
  const float q0 = P0[0] - af[0], q1 = P0[1] - af[1], q2 = P0[2] - af[2];
  const float xl0[3] = {0.5f + af[3] * q0 + af[4] * q1 + af[5] * q2, 0.5f + af[6] * q0 + af[7] * q1 + af[8] * q2,
                        0.5f + af[9] * q0 + af[10] * q1 + af[11] * q2};
  const float dl[3] = {af[3] * rf[0] + af[4] * rf[1] + af[5] * rf[2], af[6] * rf[0] + af[7] * rf[1] + af[8] * rf[2],
                       af[9] * rf[0] + af[10] * rf[1] + af[11] * rf[2]};
  unsigned face_mask = 0;
  if (active) {
    float tin[3], tout[3], inv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      inv[k] = 1.0f / dl[k];
      const float ta = (-dpv[k] - xl0[k]) * inv[k], tb = (1.0f + dpv[k] - xl0[k]) * inv[k];
      tin[k] = fminf(ta, tb);
      tout[k] = fmaxf(ta, tb);
    }
    const float ben = fmaxf(tin[0], fmaxf(tin[1], tin[2])), bex = fminf(tout[0], fminf(tout[1], tout[2]));
    if (bex >= ben) {
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        const int k = f >> 1, fa = (k + 1) % 3, fb = (k + 2) % 3;
        const float side = (float)(f & 1);
        // face slab |xl_k - side| <= dp_k within the inflated box
        const float ta = (side - dpv[k] - xl0[k]) * inv[k], tb = (side + dpv[k] - xl0[k]) * inv[k];
        const float lo = fmaxf(ben, fminf(ta, tb)), hi = fminf(bex, fmaxf(ta, tb));
        if (!(hi >= lo)) continue;
        // proof of "no root" (see 1b): any root x* = (s_a, s_b, beta) solves
        // x* = x0 - M0^-1 E(s*), so |x* - x0|_inf <= ||M0^-1|| max|E| -- no
        // contraction needed; inconclusive (NaN / inf) bounds keep the face
        const float rk = inv[k];
        const float mnorm = fmaxf(fabsf(rk), 1.0f + fabsf(dl[fa] * rk) + fabsf(dl[fb] * rk));
        const float b0 = (side - xl0[k]) * rk;
        const float sa0 = xl0[fa] + b0 * dl[fa], sb0 = xl0[fb] + b0 * dl[fb];
        const float rho = mnorm * dpm + FACE_TOL;
        if (sa0 < -rho || sa0 > 1.0f + rho || sb0 < -rho || sb0 > 1.0f + rho) continue;
        face_mask |= 1u << f;
      }
    }
  }
  W.ps[0][lane] = P0[0]; W.ps[1][lane] = P0[1]; W.ps[2][lane] = P0[2];
  W.ps[3][lane] = rf[0]; W.ps[4][lane] = rf[1]; W.ps[5][lane] = rf[2];
  W.ps[6][lane] = xl0[0]; W.ps[7][lane] = xl0[1]; W.ps[8][lane] = xl0[2];
  W.ps[9][lane] = dl[0]; W.ps[10][lane] = dl[1]; W.ps[11][lane] = dl[2];
  W.ps[13][lane] = rr;
  W.nroots[lane] = 0;
  W.pw[lane] = w;
  int ntask;
  {
    const int want = __popc(face_mask);
    int incl = want;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += y;
    }
    ntask = __shfl_sync(0xffffffffu, incl, 31);
    int t = incl - want;
    for (unsigned m = face_mask; m; m &= m - 1) W.task[t++] = (uint8_t)((lane << 3) | (__ffs(m) - 1));
  }
  __syncwarp();

  // ---- 1b: face tasks, one per lane -----------------------------------------
  int nfallback = 0;
  for (int t0 = 0; t0 < ntask; t0 += 32) {
    const int t = t0 + (int)lane;
    if (t < ntask) {
      const int code = W.task[t];
      const int pl = code >> 3, f = code & 7;
      const float* sB = S.u.p.slot[W.pw[pl]];   // the task's element
      const float* af = sB + SLOT_AFF;
      const float eta2 = 2.0f * af[15];
      const int fk = f >> 1, fside = f & 1;
      const int fa = fk == 2 ? 0 : fk + 1, fb = fk == 0 ? 2 : fk - 1;
      bool done = false;
      {
        // Certified fast path.  In xi~ coordinates the face is
        // (s_a, s_b, side) + E(s) and the ray xl0 + beta dl, so the root
        // x = (s_a, s_b, beta) solves x = x0 - M0^-1 E(s) with M0 = [e_a, e_b, -dl];
        // the map contracts with q = ||M0^-1|| 2 eta < FAST_Q < 1 (uniqueness +
        // convergence; the exclusion was proven in 1a).
        // The axes (k, a, b) are per lane: their components are read from
        // shared memory at computed addresses (rows of J0^-1, the pixel's ray
        // state), never by indexing register arrays (local memory).
        const float dk = W.ps[9 + fk][pl], dla = W.ps[9 + fa][pl], dlb = W.ps[9 + fb][pl];
        const float xlk = W.ps[6 + fk][pl], xla = W.ps[6 + fa][pl], xlb = W.ps[6 + fb][pl];
        const float rk = 1.0f / dk;
        const float mnorm = fmaxf(fabsf(rk), 1.0f + fabsf(dla * rk) + fabsf(dlb * rk));
        const float qf = mnorm * eta2;
        if (qf < FAST_Q) {
          const float side = (float)fside;
          const float b0 = (side - xlk) * rk;
          const float sa0 = xla + b0 * dla, sb0 = xlb + b0 * dlb;
          const float qfac = qf / (1.0f - qf) * 1.01f;
          float sa = sa0, sb = sb0, bt = b0;
          // padded float strides of m1, m2, m3: 3, 12, 36
          const int pk = fk == 0 ? 3 : (fk == 1 ? 12 : 36);
          const int fsa = fk == 0 ? 12 : (fk == 1 ? 36 : 3), fsb = fk == 0 ? 36 : (fk == 1 ? 3 : 12);
          const int fbase = 2 * fside * pk;
          const float* jk = af + 3 + 3 * fk;   // rows k, a, b of J0^-1
          const float* ja = af + 3 + 3 * fa;
          const float* jb = af + 3 + 3 * fb;
#pragma unroll 1
          for (int it = 0; it < max_it; ++it) {
            float X[3];
            eval_face(sB, fbase, fsa, fsb, sa, sb, X);
            // E(s) = J0^-1 (X - Xc) + 1/2 - xi, components k, a, b (xi = side, s_a, s_b)
            const float y0 = X[0] - af[0], y1 = X[1] - af[1], y2 = X[2] - af[2];
            const float Ek = jk[0] * y0 + jk[1] * y1 + jk[2] * y2 + 0.5f - side;
            const float Ea = ja[0] * y0 + ja[1] * y1 + ja[2] * y2 + 0.5f - sa;
            const float Eb = jb[0] * y0 + jb[1] * y1 + jb[2] * y2 + 0.5f - sb;
            // M0^-1 y: beta = -y_k/dl_k, s_a = y_a + beta dl_a, s_b = y_b + beta dl_b
            const float db = -Ek * rk;
            const float nbt = b0 - db;
            const float nsa = sa0 - (Ea + db * dla);
            const float nsb = sb0 - (Eb + db * dlb);
            const float step = fmaxf(fabsf(nsa - sa), fmaxf(fabsf(nsb - sb), fabsf((nbt - bt) * dk)));
            sa = nsa;
            sb = nsb;
            bt = nbt;
            // |x_{k+1} - x*| <= q/(1-q) |x_{k+1} - x_k|
            if (step * qfac < tol) {
              done = true;
              break;
            }
          }
          if (done && sa >= -FACE_TOL && sa <= 1.0f + FACE_TOL && sb >= -FACE_TOL && sb <= 1.0f + FACE_TOL) {
            const int k = atomicAdd(&W.nroots[pl], 1);   // push_root with the components placed by axis
            if (k >= MAXR) {
              ++face_fail;
            } else {
              W.roots[k][0][pl] = bt;
              W.roots[k][1 + fk][pl] = side;
              W.roots[k][1 + fa][pl] = fminf(fmaxf(sa, 0.0f), 1.0f);
              W.roots[k][1 + fb][pl] = fminf(fmaxf(sb, 0.0f), 1.0f);
            }
          }
        }
      }
      if (!done) {
        ++nfallback;
        const float tP0[3] = {W.ps[0][pl], W.ps[1][pl], W.ps[2][pl]};
        const float trf[3] = {W.ps[3][pl], W.ps[4][pl], W.ps[5][pl]};
        const float trr = W.ps[13][pl];
        face_2d(W, sB, pl, f, tP0, trf, trr, tol, max_it, face_fail);
      }
    }
  }
  __syncwarp();
  {
    // diagnostics: face tasks and those that needed the 2D path
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nfallback += __shfl_xor_sync(0xffffffffu, nfallback, off);
    if (lane == 0) {
      atomicAdd(&W.stats[0], ntask);
      atomicAdd(&W.stats[1], nfallback);
    }
  }

  // ---- 1c: per pixel: sort roots, pair entry/exit, emit items ---------------
  int nr = min(W.nroots[lane], MAXR);
  uint8_t* ord = &W.rord[0][lane];   // this lane's sorted root list (stride 32)
  if (nr == 2) {                      // common case: entry and exit
    const bool sw = W.roots[1][0][lane] < W.roots[0][0][lane];
    ord[0] = sw ? 1 : 0;
    ord[32] = sw ? 0 : 1;
  } else
  for (int t = 0; t < nr; ++t) {      // insertion sort by beta
    const float bt = W.roots[t][0][lane];
    int z = t;
    while (z > 0 && W.roots[ord[(z - 1) * 32]][0][lane] > bt) {
      ord[z * 32] = ord[(z - 1) * 32];
      --z;
    }
    ord[z * 32] = (uint8_t)t;
  }
  {
    // dedupe roots found on two faces at a shared edge / vertex
    const float rn = sqrtf(rr);
    const float hw = fabsf(sB[GI(26)] - sB[0]) + fabsf(sB[GI(26) + 1] - sB[1]) + fabsf(sB[GI(26) + 2] - sB[2]);
    const float dtol = 4e-6f * hw / rn;
    int m = 0;
    for (int t = 0; t < nr; ++t) {
      const int o = ord[t * 32];
      if (m > 0 && W.roots[o][0][lane] - W.roots[ord[(m - 1) * 32]][0][lane] < dtol) continue;
      ord[m * 32] = (uint8_t)o;
      ++m;
    }
    nr = m & ~1;   // entry/exit pairs
  }
  const float bmin = (float)(cc.amin - (double)alpha0), bmax = (float)(cc.amax - (double)alpha0);
  int nseg = 0;
  for (int z = 0; z < nr; z += 2)
    nseg += fminf(W.roots[ord[(z + 1) * 32]][0][lane], bmax) > fmaxf(W.roots[ord[z * 32]][0][lane], bmin) ? 1 : 0;
  const uint32_t pix = (uint32_t)(j * cc.W + i);
  if (nseg > 0) {
    ++local_hits;
    atomicAdd(&hits_pp[pix], 1);
  }
  int slot = warp_append_smem(s_nitems, nseg);
#pragma unroll 1
  for (int z = 0; z < nr; z += 2) {
    const int ia = ord[z * 32], ib = ord[(z + 1) * 32];
    const float ba = W.roots[ia][0][lane], bz = W.roots[ib][0][lane];
    if (!(fminf(bz, bmax) > fmaxf(ba, bmin))) continue;
    const float b0 = fmaxf(ba, bmin), b1 = fminf(bz, bmax);
    if (slot < ITEM_CAP) {
      float4* it = items + 4 * slot;
      it[0] = make_float4(fmaf(b0, rf[0], P0[0]), fmaf(b0, rf[1], P0[1]), fmaf(b0, rf[2], P0[2]),
                          fmaf(b1, rf[0], P0[0]));
      it[1] = make_float4(fmaf(b1, rf[1], P0[1]), fmaf(b1, rf[2], P0[2]), W.roots[ia][1][lane],
                          W.roots[ia][2][lane]);
      it[2] = make_float4(W.roots[ia][3][lane], W.roots[ib][1][lane], W.roots[ib][2][lane], W.roots[ib][3][lane]);
      it[3] = make_float4(alpha0 + b0, alpha0 + b1, __uint_as_float((uint32_t)i | ((uint32_t)j << 16)),
                          __int_as_float(v));
    }
    ++slot;
  }
  __syncwarp();   // W is reused by the warp's next chunk
}

// ---- phase 2 with the paper's integrators (rc_camera.scheme, Alg. 1) ---------
// The medium at near-end parameter u: xi(u) by the chord iteration of phase 2
// from the quadratic prediction through (entry, midpoint, exit) xi, then the
// nodal field.  Out of line: an opt-in path that must not grow the default
// phase's code.
template <int P>
struct CurvedMedium {
  const float* gs;
  const CamConst* cc;
  float xin[3], dX[3], xia[3], xm[3], xib[3], Ji[3][3], qfac;
  int* fails;
  __device__ MediumSample operator()(float u) const {
    const float l0 = (1.0f - u) * (1.0f - 2.0f * u), l1 = 4.0f * u * (1.0f - u), l2 = u * (2.0f * u - 1.0f);
    float x[3], t[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      x[d] = l0 * xia[d] + l1 * xm[d] + l2 * xib[d];
      t[d] = fmaf(u, dX[d], xin[d]);
    }
    bool conv = false;
    for (int it = 0; it < 2 * cc->newton_max; ++it) {
      float X[3];
      eval_X(gs, x, X);
      float step = 0.0f;
      const float r0 = t[0] - X[0], r1 = t[1] - X[1], r2 = t[2] - X[2];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const float sd = Ji[d][0] * r0 + Ji[d][1] * r1 + Ji[d][2] * r2;
        x[d] += sd;
        step = fmaxf(step, fabsf(sd));
      }
      if (step * qfac < cc->newton_tol) {
        conv = true;
        break;
      }
    }
    if (!conv) ++*fails;
#pragma unroll
    for (int d = 0; d < 3; ++d) x[d] = fminf(fmaxf(x[d], 0.0f), 1.0f);   // nodes lie inside the element
    return medium_from_f(*cc, field_pad<P>(gs + SLOT_FIELD, x[0], x[1], x[2]) * cc->inv_F);
  }
};

template <int P>
__device__ __noinline__ void integ_scheme(const float* __restrict__ gs, const CamConst& cc, const float xin[3],
                                          const float dX[3], const float xia[3], const float xm[3],
                                          const float xib[3], float Lseg, float qfac, int& fails, int& capped,
                                          float& a_out, float b_out[3]) {
  CurvedMedium<P> med;
  med.gs = gs;
  med.cc = &cc;
  med.qfac = qfac;
  med.fails = &fails;
  const float* afm = gs + SLOT_AFF;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    med.xin[d] = xin[d];
    med.dX[d] = dX[d];
    med.xia[d] = xia[d];
    med.xm[d] = xm[d];
    med.xib[d] = xib[d];
#pragma unroll
    for (int e = 0; e < 3; ++e) med.Ji[d][e] = afm[3 + 3 * d + e];
  }
  segment_scheme(cc, Lseg, med, a_out, b_out, capped);
}

// ---- phase 2: integrate one item per lane ----------------------------------
// The field at each GL node needs xi(x): chord iteration with
// the element's J0^-1, started from a quadratic prediction through (entry,
// midpoint, exit) xi (the midpoint solved first).  Chord map
// T(xi) = xi + J0^-1 (t - X(xi)): |DT|_inf = |I - J0^-1 J|_inf <= 3 eta on the
// element, so after a step s the error is <= q/(1-q) s (q = 3 eta); the
// iteration stops when that bound is below tol (plain s < tol when q >= 1/2).
// scr: this thread's scratch (stride CWARPS*32 floats) for the node values
template <int P, int N, bool ADAPT>
__device__ __forceinline__ void integ_item(const float* __restrict__ gs, const CamConst& cc, float4 i0, float4 i1,
                                           float4 i2, float* __restrict__ scr, int& fails, int& capped, float& a_out,
                                           float b_out[3]) {
  constexpr int ST = CWARPS * 32;
  const float tol = cc.newton_tol;
  const int max_it = cc.newton_max;
  const float* fs = gs + SLOT_FIELD;
  const float* afm = gs + SLOT_AFF;
  float Ji[3][3];
#pragma unroll
  for (int aa = 0; aa < 3; ++aa)
#pragma unroll
    for (int b = 0; b < 3; ++b) Ji[aa][b] = afm[3 + 3 * aa + b];
  const float q3 = 3.0f * afm[15] * 1.1f;
  const float qfac = q3 < 0.5f ? q3 / (1.0f - q3) : 1.0f;
  const float xin[3] = {i0.x, i0.y, i0.z}, xout[3] = {i0.w, i1.x, i1.y};
  const float xia[3] = {i1.z, i1.w, i2.x}, xib[3] = {i2.y, i2.z, i2.w};
  const float dX[3] = {xout[0] - xin[0], xout[1] - xin[1], xout[2] - xin[2]};
  const float Lseg = sqrtf(dX[0] * dX[0] + dX[1] * dX[1] + dX[2] * dX[2]);   // physical length (R2)
  float xm[3] = {0.5f * (xia[0] + xib[0]), 0.5f * (xia[1] + xib[1]), 0.5f * (xia[2] + xib[2])};
  const float tm[3] = {xin[0] + 0.5f * dX[0], xin[1] + 0.5f * dX[1], xin[2] + 0.5f * dX[2]};
  bool ok = false;
#pragma unroll 1
  for (int it = 0; it < 2 * max_it; ++it) {
    float X[3];
    eval_X(gs, xm, X);
    const float r0 = tm[0] - X[0], r1 = tm[1] - X[1], r2 = tm[2] - X[2];
    const float s0 = Ji[0][0] * r0 + Ji[0][1] * r1 + Ji[0][2] * r2;
    const float s1 = Ji[1][0] * r0 + Ji[1][1] * r1 + Ji[1][2] * r2;
    const float s2 = Ji[2][0] * r0 + Ji[2][1] * r1 + Ji[2][2] * r2;
    xm[0] += s0;
    xm[1] += s1;
    xm[2] += s2;
    if (fmaxf(fabsf(s0), fmaxf(fabsf(s1), fabsf(s2))) * qfac < tol) {
      ok = true;
      break;
    }
  }
  if (!ok) ++fails;
  if constexpr (ADAPT) {   // the paper's integrators with Alg. 1 (rc_camera.scheme)
    integ_scheme<P>(gs, cc, xin, dX, xia, xm, xib, Lseg, qfac, fails, capped, a_out, b_out);
    return;
  }
  float sumk = 0.0f;
  // the GL nodes two at a time: independent chord iterations in lockstep
#pragma unroll 1
  for (int q = 0; q < N; q += 2) {
    const int qb = q + 1 < N ? q + 1 : q;
    float xa[3], xb[3], ta[3], tb[3];
    {
      const float u = cc.u[q], w = cc.u[qb];
      const float l0 = (1.0f - u) * (1.0f - 2.0f * u), l1 = 4.0f * u * (1.0f - u), l2 = u * (2.0f * u - 1.0f);
      const float k0 = (1.0f - w) * (1.0f - 2.0f * w), k1 = 4.0f * w * (1.0f - w), k2 = w * (2.0f * w - 1.0f);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        xa[d] = l0 * xia[d] + l1 * xm[d] + l2 * xib[d];
        xb[d] = k0 * xia[d] + k1 * xm[d] + k2 * xib[d];
        ta[d] = fmaf(u, dX[d], xin[d]);
        tb[d] = fmaf(w, dX[d], xin[d]);
      }
    }
    bool conv = false;
#pragma unroll 1
    for (int it = 0; it < 2 * max_it; ++it) {
      float XA[3], XB[3];
      eval_X2(gs, xa, xb, XA, XB);
      float step = 0.0f;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float sa = Ji[r][0] * (ta[0] - XA[0]) + Ji[r][1] * (ta[1] - XA[1]) + Ji[r][2] * (ta[2] - XA[2]);
        const float sb = Ji[r][0] * (tb[0] - XB[0]) + Ji[r][1] * (tb[1] - XB[1]) + Ji[r][2] * (tb[2] - XB[2]);
        xa[r] += sa;
        xb[r] += sb;
        step = fmaxf(step, fmaxf(fabsf(sa), fabsf(sb)));
      }
      if (step * qfac < tol) {
        conv = true;
        break;
      }
    }
    if (!conv) ++fails;
#pragma unroll
    for (int d = 0; d < 3; ++d) {   // nodes lie inside the element
      xa[d] = fminf(fmaxf(xa[d], 0.0f), 1.0f);
      xb[d] = fminf(fmaxf(xb[d], 0.0f), 1.0f);
    }
    const float fa = field_pad<P>(fs, xa[0], xa[1], xa[2]) * cc.inv_F;
    sumk = fmaf(cc.w[q], cc.kappa0 * fa * fa, sumk);
    scr[q * ST] = fa;
    if (qb != q) {
      const float fb = field_pad<P>(fs, xb[0], xb[1], xb[2]) * cc.inv_F;
      sumk = fmaf(cc.w[qb], cc.kappa0 * fb * fb, sumk);
      scr[qb * ST] = fb;
    }
  }
  // node optical depths tau_j = L sum_k S_jk kappa_k
  float tau[N], ftv[N];
#pragma unroll
  for (int q = 0; q < N; ++q) ftv[q] = scr[q * ST];
#pragma unroll
  for (int jj = 0; jj < N; ++jj) {
    tau[jj] = 0.0f;
#pragma unroll
    for (int q = 0; q < N; ++q) tau[jj] = fmaf(cc.S[jj * RC_MAX_N + q], cc.kappa0 * ftv[q] * ftv[q], tau[jj]);
  }
  // a = exp(-L sum w kappa); b_c = L sum w_j q_cj exp(-tau_j)
  a_out = __expf(-Lseg * sumk);
  float E0 = 0.0f, E1 = 0.0f;
#pragma unroll
  for (int jj = 0; jj < N; ++jj) {
    const float ee = cc.w[jj] * __expf(-Lseg * tau[jj]);
    E0 += ee;
    E1 = fmaf(ee, ftv[jj], E1);
  }
  const float sc = 0.5f * Lseg * cc.q0;
  b_out[0] = sc * (E0 + E1);
  b_out[1] = sc * (E0 - E1);
  b_out[2] = sc * E0;
}

// ---- phase 3, common case: bucket fold -------------------------------------
// The unit's segments are bucketed by pixel over the unit's bounding rectangle
// (shared-memory counting sort), each pixel's few segments (one per element
// the ray crosses in the unit) are ordered by alpha_near in place, and
// every maximal run of touching segments is combined nearest-first with
// Eq. aggregate in fp64 and written as one record.

__device__ __forceinline__ int block_excl_scan(CastCtl& ctl, int v, int& total) {
  const unsigned lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if ((int)lane >= off) incl += y;
  }
  __syncthreads();
  if (lane == 31) ctl.warp_sum[warp] = incl;
  __syncthreads();
  int base = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < CWARPS; ++w) {
    base += w < warp ? ctl.warp_sum[w] : 0;
    total += ctl.warp_sum[w];
  }
  return base + incl - v;
}

__device__ __forceinline__ bool touching(float an, float af_prev) {
  return fabsf(an - af_prev) <= FOLD_TAU * fmaxf(1.0f, fabsf(an));
}

// One window of rows [bj0, bj0 + rows) of the unit's pixel rectangle (the
// caller covers the rectangle with windows of <= PIXCAP pixels); segments of
// other rows are left to their window.
// Scratch segments carry the pixel packed relative to the unit's rectangle
// ((row << 16) | col); the window covers rectangle rows [r0, r0 + rows).
__device__ void fold_bucket(CastSmem& S, CastCtl& ctl, const rc_seg* __restrict__ segs, int nitems, int bi0, int bj0,
                            int r0, int bw, int rows, int W, uint32_t ukey, rc_seg* __restrict__ out,
                            int64_t out_cap, int64_t* __restrict__ counters) {
  const int tid = threadIdx.x;
  constexpr int NT = CWARPS * 32;
  FoldSmem& F = S.u.fold;
  const int area = bw * rows;
  __syncthreads();   // the previous window's readers are done
  for (int k = tid; k <= area; k += NT) F.off[k] = 0;
  __syncthreads();
  // one coalesced pass over the unit's segments: (alpha_near, alpha_far) to
  // shared memory, bucket counts per pixel of the window
  for (int k = tid; k < nitems; k += NT) {
    const float4 h = reinterpret_cast<const float4*>(segs + k)[0];   // pixel, alpha_near, alpha_far, a
    const uint32_t lp = __float_as_uint(h.x);
    const int row = (int)(lp >> 16) - r0;
    F.alpha[k] = make_float2(h.y, h.z);
    if (row < 0 || row >= rows) continue;
    const int pl = row * bw + (int)(lp & 0xffffu);
    F.rank[k] = (uint16_t)atomicAdd(&F.off[pl], 1);
  }
  __syncthreads();
  // exclusive scan of the counts over the rectangle (each thread a contiguous range)
  const int per = (area + NT - 1) / NT;
  const int p0 = min(area, tid * per), p1 = min(area, p0 + per);
  int sum = 0;
  for (int k = p0; k < p1; ++k) sum += F.off[k];
  int total;
  int run = block_excl_scan(ctl, sum, total);
  for (int k = p0; k < p1; ++k) {
    const int c = F.off[k];
    F.off[k] = run;
    run += c;
  }
  if (tid == 0) F.off[area] = total;
  __syncthreads();
  for (int k = tid; k < nitems; k += NT) {   // pixel-bucketed order
    const uint32_t lp = segs[k].pixel;
    const int row = (int)(lp >> 16) - r0;
    if (row < 0 || row >= rows) continue;
    const int pl = row * bw + (int)(lp & 0xffffu);
    F.order[F.off[pl] + F.rank[k]] = (uint16_t)k;
  }
  __syncthreads();
  // per pixel: order by (alpha_near, index), count runs, then emit (two passes)
  int nrun = 0;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t pos = 0;
    if (pass == 1) {
      int tot;
      const int ex = block_excl_scan(ctl, nrun, tot);
      if (tid == 0) ctl.base = atomicAdd((unsigned long long*)&counters[CNT_SEGS], (unsigned long long)tot);
      __syncthreads();
      pos = (int64_t)ctl.base + ex;
    }
    for (int pl = tid; pl < area; pl += NT) {
      const int o = F.off[pl], n = F.off[pl + 1] - o;
      if (n == 0) continue;
      uint16_t* ord = F.order + o;
      if (pass == 0) {
        // insertion sort of the pixel's slice, in place, under the total order
        // (alpha_near, alpha_far, visible leaf, slot): the runs, and so the
        // records, do not depend on the order the items were produced in
        for (int t = 1; t < n; ++t) {
          const int k = ord[t];
          const float2 ak = F.alpha[k];
          int z = t;
          while (z > 0) {
            const int kp = ord[z - 1];
            const float2 ap = F.alpha[kp];
            bool after = ap.x > ak.x;
            if (ap.x == ak.x) {
              if (ap.y != ak.y) after = ap.y > ak.y;
              else {
                const uint32_t vp = segs[kp].key, vk = segs[k].key;   // visible leaf index (tie: rare)
                after = vp != vk ? vp > vk : kp > k;
              }
            }
            if (!after) break;
            ord[z] = (uint16_t)kp;
            --z;
          }
          ord[z] = (uint16_t)k;
        }
      }
      int t = 0;
      while (t < n) {
        float afr = F.alpha[ord[t]].y;
        int q = t + 1;
        while (q < n && touching(F.alpha[ord[q]].x, afr)) {
          afr = F.alpha[ord[q]].y;
          ++q;
        }
        if (pass == 0) {
          ++nrun;
        } else {
          // fold the run [t, q) nearest first (Eq. aggregate) in fp64
          double A = 1.0, B0 = 0.0, B1 = 0.0, B2 = 0.0;
          for (int z = t; z < q; ++z) {
            const rc_seg* sq = segs + ord[z];
            const float a = sq->a;
            const float4 hb = reinterpret_cast<const float4*>(sq)[1];   // b0, b1, b2, key
            B0 = fma(A, (double)hb.x, B0);
            B1 = fma(A, (double)hb.y, B1);
            B2 = fma(A, (double)hb.z, B2);
            A *= (double)a;
          }
          const uint32_t pix = (uint32_t)((bj0 + r0 + pl / bw) * W + bi0 + pl % bw);
          if (pos < out_cap) {
            const float bf[3] = {(float)B0, (float)B1, (float)B2};
            store_seg_cs(out + pos, pix, F.alpha[ord[t]].x, afr, (float)A, bf, ukey);
          } else {
            atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
          }
          ++pos;
        }
        t = q;
      }
    }
  }
}

// ---- the kernel --------------------------------------------------------------
template <int P, int N, bool ADAPT>
__global__ void __launch_bounds__(CWARPS * 32, CAST_CTAS_PER_SM) k_cast_curved(CamConst cc, const TreeConst* __restrict__ trees,
                                                                DevLeafView L, const int32_t* __restrict__ vis,
                                                                const Rect16* __restrict__ vrect,
                                                                const int64_t* __restrict__ chunk_off,
                                                                const int32_t* __restrict__ chunk_elem,
                                                                const Unit* __restrict__ units, int64_t nunits,
                                                                int fold, uint32_t key_base,
                                                                unsigned char* __restrict__ scratch,
                                                                rc_seg* __restrict__ out, int64_t out_cap,
                                                                int32_t* __restrict__ hits_pp,
                                                                int64_t* __restrict__ counters,
                                                                const float4* __restrict__ gslot,
                                                                const double* __restrict__ gorg, int64_t v0,
                                                                int64_t v1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CastSmem& S = *reinterpret_cast<CastSmem*>(smem_raw);
  __shared__ CastCtl ctl;
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  unsigned char* my = scratch + (size_t)blockIdx.x * SCR_PER_CTA;
  float4* items = reinterpret_cast<float4*>(my);
  rc_seg* segs = reinterpret_cast<rc_seg*>(my + SCR_ITEMS);
  int local_hits = 0, face_fail = 0, fails = 0, capped = 0;
  long long raw_local = 0, n_tasks = 0, n_fallback = 0;
  int prev_items = 0;
  uint32_t mbar_parity = 0;
  if (tid == 0) {
    mbar_init(&ctl.mbar, 1);
    // this launch's units: those whose visible window starts in [v0, v1) (units are in vfirst order)
    int64_t lo = 0, hi = nunits;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (units[mid].vfirst < v0) lo = mid + 1;
      else hi = mid;
    }
    ctl.ubeg = lo;
    hi = nunits;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (units[mid].vfirst < v1) lo = mid + 1;
      else hi = mid;
    }
    ctl.uend = lo;
  }
  for (;;) {
    __syncthreads();   // the previous unit's shared state (ctl, S) and scratch are no longer read
    if (prev_items > 0) {
      discard_l2(items, ((size_t)prev_items * 64 + 127) & ~(size_t)127);
      if (fold > 0) discard_l2(segs, ((size_t)prev_items * sizeof(rc_seg) + 127) & ~(size_t)127);
    }
    if (tid == 0) {
      ctl.unit = ctl.ubeg + (int64_t)atomicAdd((unsigned long long*)&counters[CNT_UNITS], 1ull);
      ctl.next_chunk = 0;
      ctl.nitems = 0;
    }
    __syncthreads();
    const int64_t u = ctl.unit;
    if (u >= ctl.uend) break;
    const Unit U = units[u];
    // ---- phase 0: the unit's prepared element slots arrive by bulk copies ----
    // (k_prep_slots made them; one 640-byte record per element plus the fp64
    // origins), tracked by the CTA's mbarrier while the threads set up the
    // unit's pair bookkeeping
    if (warp == 0) {   // warp 0's lanes issue the unit's copies (two or three each)
      fence_proxy_async_smem();   // the previous unit's generic reads of the slots are done (barrier above)
      const int64_t g0 = U.vfirst - v0;
      if (lane == 0) mbar_arrive_expect_tx(&ctl.mbar, (uint32_t)U.nvis * (SLOT_USED * 4 + 32));
      __syncwarp();
      for (int w = (int)lane; w < U.nvis; w += 32)
        bulk_g2s(S.u.p.slot[w], gslot + (g0 + w) * (SLOT_USED / 4), SLOT_USED * 4, &ctl.mbar);
      if (lane == 31) bulk_g2s(S.meta.org, gorg + g0 * 4, (uint32_t)U.nvis * 32, &ctl.mbar);
    }
    if (tid < 4) ctl.bb[tid] = -0x7fffffff;
    __syncthreads();
    for (int w = tid; w < U.nvis; w += CWARPS * 32) {
      const Rect16 r = vrect[U.vfirst + w];
      S.meta.rect[w] = r;
      // the element's candidate pairs inside this unit's chunk range
      const int64_t ca = chunk_off[U.vfirst + w], cz = chunk_off[U.vfirst + w + 1];
      const int64_t k0 = max((int64_t)0, U.chunk_begin - ca);
      const int64_t k1 = min(cz - ca, U.chunk_begin + U.nchunks - ca);
      const int area = (r.i1 - r.i0 + 1) * (r.j1 - r.j0 + 1);
      const int pa = (int)(k0 * RC_CHUNK), pb = (int)min((int64_t)area, k1 * RC_CHUNK);
      S.meta.pa[w] = pa;
      S.meta.pstart[w + 1] = max(0, pb - pa);   // counts; prefix-summed below
      atomicMax(&ctl.bb[0], -(int)r.i0);
      atomicMax(&ctl.bb[1], (int)r.i1);
      atomicMax(&ctl.bb[2], -(int)r.j0);
      atomicMax(&ctl.bb[3], (int)r.j1);
    }
    __syncthreads();
    if (warp == 0) {   // prefix of the pair counts (<= 64 elements: two per lane)
      const int a0 = 2 * (int)lane + 1, a1 = a0 + 1;
      const int c0 = a0 <= U.nvis ? S.meta.pstart[a0] : 0, c1 = a1 <= U.nvis ? S.meta.pstart[a1] : 0;
      int incl = c0 + c1;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if ((int)lane >= off) incl += y;
      }
      if (a0 <= U.nvis) S.meta.pstart[a0] = incl - c1;
      if (a1 <= U.nvis) S.meta.pstart[a1] = incl;
      if (lane == 0) S.meta.pstart[0] = 0;
    }
    mbar_wait(&ctl.mbar, mbar_parity);
    mbar_parity ^= 1u;
    __syncthreads();
    for (int w = tid; w < U.nvis; w += CWARPS * 32) {   // chunk -> first element map
      const int a = S.meta.pstart[w], b = S.meta.pstart[w + 1];
      if (b > a)
        for (int c = (a + RC_CHUNK - 1) / RC_CHUNK; c * RC_CHUNK < b; ++c) S.meta.vmap[c] = (uint8_t)w;
      // prefilter constants: re-basing vector and a margin covering its fp32 error
      float dn = 0.0f, jn = 0.0f;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double d = S.meta.org[w][k] - cc.O0[k];
        S.meta.Dc[w][k] = (float)d;
        dn = fmaxf(dn, fabsf((float)d));
        const float* ji = S.u.p.slot[w] + SLOT_AFF + 3 + 3 * k;
        jn = fmaxf(jn, fabsf(ji[0]) + fabsf(ji[1]) + fabsf(ji[2]));
      }
      const float ext = fmaxf(dn, (float)(cc.ell * (cc.W + cc.H)) + dn);   // |D| incl. ortho pixel offsets
      S.meta.pm[w] = 4e-6f * (ext + 1.0f) * jn + 1e-4f;
      S.meta.rwinv[w] = 1.0f / (float)(S.meta.rect[w].i1 - S.meta.rect[w].i0 + 1);
    }
    __syncthreads();
    // ---- phase 1: intersection -----------------------------------------------
    {
      WarpIsect& W = S.u.p.ph.isect[warp];
      if (lane == 0) W.stats[0] = W.stats[1] = 0;
      __syncwarp();
      const int nvchunks = (S.meta.pstart[U.nvis] + RC_CHUNK - 1) / RC_CHUNK;
      // candidates that pass the conservative fp32 prefilter are queued and
      // intersected 32 at a time (misses no longer occupy the exact path)
      const int npairs = S.meta.pstart[U.nvis];
      int qn = 0;
      // one call site of the (large, inlined) isect_chunk: full batches and
      // the tail share it (halves the phase's code, instruction-cache bound)
      bool drained = false;
      for (;;) {
        if (!drained) {
          int k = 0;
          if (lane == 0) k = atomicAdd(&ctl.next_chunk, 1);
          k = __shfl_sync(0xffffffffu, k, 0);
          if (k >= nvchunks) {
            drained = true;
          } else {
            const int g = k * RC_CHUNK + (int)lane;
            const bool keep = g < npairs && prefilter_f32(S, cc, g);
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) W.queue[qn + __popc(bal & ((1u << lane) - 1u))] = g;
            qn += __popc(bal);
            __syncwarp();
          }
        }
        if (qn >= 32 || (drained && qn > 0)) {
          const int gq = (int)lane < qn ? W.queue[lane] : -1;
          const int rest = qn > 32 + (int)lane ? W.queue[32 + lane] : 0;
          __syncwarp();
          if (32 + (int)lane < qn) W.queue[lane] = rest;
          qn = qn > 32 ? qn - 32 : 0;
          __syncwarp();
          isect_chunk(W, S, cc, U.nvis, U.vfirst, gq, items, &ctl.nitems, hits_pp, local_hits, face_fail);
        } else if (drained) {
          break;
        }
      }
      if (lane == 0) {
        n_tasks += W.stats[0];
        n_fallback += W.stats[1];
      }
    }
    __syncthreads();
    const int nitems = min(ctl.nitems, ITEM_CAP);
    raw_local += (tid == 0) ? nitems : 0;
    prev_items = nitems;
    // ---- phase 2: integration ---------------------------------------------------
    const int ubi0 = -ctl.bb[0], ubj0 = -ctl.bb[2];
    {
      const int ngroups = (nitems + 31) / 32;
      for (int g = warp; g < ngroups; g += CWARPS) {
        const int idx = g * 32 + (int)lane;
        const bool act = idx < nitems;
        float a = 1.0f, bb[3] = {0.f, 0.f, 0.f};
        uint32_t pix = 0;
        float an = 0.f, afar = 0.f;
        int v = 0;
        if (act) {
          const float4* it = items + 4 * idx;
          const float4 i0 = it[0], i1 = it[1], i2 = it[2], i3 = it[3];
          v = __float_as_int(i3.w);
          const uint32_t ij = __float_as_uint(i3.z);
          // fold: pixel packed relative to the unit's rectangle; else global j W + i
          pix = fold > 0 ? ((((ij >> 16) - (uint32_t)ubj0) << 16) | ((ij & 0xffffu) - (uint32_t)ubi0))
                         : (ij >> 16) * (uint32_t)cc.W + (ij & 0xffffu);
          an = i3.x;
          afar = i3.y;
          integ_item<P, N, ADAPT>(S.u.p.slot[v - U.vfirst], cc, i0, i1, i2, S.u.p.ph.scr + tid, fails, capped, a, bb);
        }
        if (fold > 0) {
          if (act) {
            store_seg(segs + idx, pix, an, afar, a, bb, (uint32_t)v);   // key field: visible leaf (fold tie-break)
          }
        } else {
          const int64_t slot = warp_append(&counters[CNT_SEGS], act ? 1 : 0);
          if (act) {
            if (slot < out_cap) store_seg_cs(out + slot, pix, an, afar, a, bb, key_base + (uint32_t)vis[v]);
            else atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
          }
        }
      }
    }
    if (fold == 0) continue;   // next unit (the loop head synchronises first)
    __syncthreads();
    // ---- phase 3: fold -----------------------------------------------------------
    {
      const int bi0 = -ctl.bb[0], bi1 = ctl.bb[1], bj0 = -ctl.bb[2], bj1 = ctl.bb[3];
      const int bw = bi1 - bi0 + 1, bh = bj1 - bj0 + 1;
      if (bw <= PIXCAP && nitems <= FCAP) {
        const int rows = PIXCAP / bw;
        for (int r0 = 0; r0 < bh; r0 += rows)
          fold_bucket(S, ctl, segs, nitems, bi0, bj0, r0, bw, min(rows, bh - r0), cc.W, U.key, out, out_cap,
                      counters);
        continue;
      }
    }
    // large units (more segments or a wider rectangle than the bucket fold
    // holds; none at C3-C5): every segment is its own record, keyed by the
    // node (folding is optional: rc_aggregate / the composite combine them)
    {
      int tot;
      const int per = (nitems + CWARPS * 32 - 1) / (CWARPS * 32);
      const int k0 = min(nitems, tid * per), k1 = min(nitems, k0 + per);
      const int ex = block_excl_scan(ctl, k1 - k0, tot);
      if (tid == 0) ctl.base = atomicAdd((unsigned long long*)&counters[CNT_SEGS], (unsigned long long)tot);
      __syncthreads();
      int64_t pos = (int64_t)ctl.base + ex;
      for (int k = k0; k < k1; ++k, ++pos) {
        const rc_seg& sq = segs[k];
        if (pos < out_cap) {
          const uint32_t gpix = (uint32_t)((ubj0 + (int)(sq.pixel >> 16)) * cc.W + ubi0 + (int)(sq.pixel & 0xffffu));
          store_seg_cs(out + pos, gpix, sq.alpha_near, sq.alpha_far, sq.a, sq.b, U.key);
        } else {
          atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
        }
      }
    }
    if (tid == 0) atomicAdd((unsigned long long*)&counters[CNT_UNFOLDED], 1ull);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    local_hits += __shfl_down_sync(0xffffffffu, local_hits, off);
    face_fail += __shfl_down_sync(0xffffffffu, face_fail, off);
    fails += __shfl_down_sync(0xffffffffu, fails, off);
  }
  if (lane == 0) {
    if (local_hits) atomicAdd((unsigned long long*)&counters[CNT_HITPAIRS], (unsigned long long)local_hits);
    if (face_fail) atomicAdd((unsigned long long*)&counters[CNT_FACE_FAIL], (unsigned long long)face_fail);
    if (face_fail + fails)
      atomicAdd((unsigned long long*)&counters[CNT_NEWTON_FAIL], (unsigned long long)(face_fail + fails));
  }
  if (tid == 0 && raw_local) atomicAdd((unsigned long long*)&counters[CNT_RAW], (unsigned long long)raw_local);
  if (capped) atomicAdd((unsigned long long*)&counters[CNT_DEPTH_CAP], (unsigned long long)capped);
  if (lane == 0 && n_tasks) {
    atomicAdd((unsigned long long*)&counters[CNT_TASKS], (unsigned long long)n_tasks);
    atomicAdd((unsigned long long*)&counters[CNT_FALLBACK], (unsigned long long)n_fallback);
  }
}

}  // namespace

size_t cast_curved_scratch_per_cta() { return SCR_PER_CTA; }
int cast_curved_ctas_per_sm() { return CAST_CTAS_PER_SM; }

template <int P, int N, bool ADAPT>
static cudaError_t cast_PNA(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                            const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                            const Unit* units, int64_t nunits, int fold, uint32_t key_base, void* scratch, rc_seg* out,
                            int64_t out_cap, int32_t* hits_pp, int64_t* counters, int grid, const float4* gslot,
                            const double* gorg, int64_t v0, int64_t v1, cudaStream_t s) {
  const size_t smem = sizeof(CastSmem);
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(k_cast_curved<P, N, ADAPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_cast_curved<P, N, ADAPT><<<grid, CWARPS * 32, smem, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, units,
                                                             nunits, fold, key_base, (unsigned char*)scratch, out,
                                                             out_cap, hits_pp, counters, gslot, gorg, v0, v1);
  return cudaGetLastError();
}

// the default GL rule (R13) and the opt-in integrators (Alg. 1) are separate instantiations,
// so the default path carries no code or registers of the other
template <int P, int N>
static cudaError_t cast_PN(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                           const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem, const Unit* units,
                           int64_t nunits, int fold, uint32_t key_base, void* scratch, rc_seg* out, int64_t out_cap,
                           int32_t* hits_pp, int64_t* counters, int grid, const float4* gslot, const double* gorg,
                           int64_t v0, int64_t v1, cudaStream_t s) {
  if (cc.scheme != RC_SCHEME_GL || cc.c_rk > 0.0f)
    return cast_PNA<P, N, true>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, units, nunits, fold, key_base, scratch,
                                out, out_cap, hits_pp, counters, grid, gslot, gorg, v0, v1, s);
  return cast_PNA<P, N, false>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, units, nunits, fold, key_base, scratch,
                               out, out_cap, hits_pp, counters, grid, gslot, gorg, v0, v1, s);
}

size_t slot_record_bytes() { return SLOT_USED * sizeof(float) + 4 * sizeof(double); }

cudaError_t launch_prep_slots(const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                              const int64_t* nvis_p, int64_t v0, int64_t v1, void* gslot, void* gorg,
                              cudaStream_t s) {
  if (v1 <= v0) return cudaSuccess;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned grid = (unsigned)std::min<int64_t>((v1 - v0 + PREP_E - 1) / PREP_E, (int64_t)sms * PREP_CTAS_PER_SM);
  if (P == 1)
    k_prep_slots<1><<<grid, 3 * PREP_E, 0, s>>>(trees, L, vis, nvis_p, v0, v1, (float4*)gslot, (double*)gorg);
  else
    k_prep_slots<2><<<grid, 3 * PREP_E, 0, s>>>(trees, L, vis, nvis_p, v0, v1, (float4*)gslot, (double*)gorg);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_cast_curved(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               const Unit* units, int64_t nunits, int fold, uint32_t key_base, void* scratch,
                               rc_seg* out, int64_t out_cap, int32_t* hits_pp, int64_t* counters, int grid,
                               const void* gslot, const void* gorg, int64_t v0, int64_t v1, cudaStream_t s) {
  ++g_launches;
#define CASE(PP, NN)                                                                                             \
  if (P == PP && cc.N == NN)                                                                                     \
    return cast_PN<PP, NN>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, units, nunits, fold, key_base, scratch, \
                           out, out_cap, hits_pp, counters, grid, (const float4*)gslot, (const double*)gorg, v0, v1, \
                           s);
  CASE(1, 1) CASE(1, 2) CASE(1, 3) CASE(1, 4) CASE(1, 5) CASE(1, 6) CASE(1, 7) CASE(1, 8)
  CASE(2, 1) CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(2, 5) CASE(2, 6) CASE(2, 7) CASE(2, 8)
#undef CASE
  return cudaErrorInvalidValue;
}

}  // namespace rc
