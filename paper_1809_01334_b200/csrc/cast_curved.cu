// cast_curved.cu -- segment kernel for curved (R=2) trees: rows a4 + a5 of
// SURVEY.md §8(a) for C3-C5.
//
// Per warp work item = 32 candidate pixels of one element (pair generation,
// kernels.cu).  Steps:
//  1. element prep (27 lanes, fp64): Bernstein control points of X_E from the
//     tree's by three sum-factorised blossom passes through shared memory
//     (restriction of the tensor-product map to the element's subcube,
//     PAPER.md:104-107); stored fp32 relative to the local origin
//     C_E = B_(1,1,1) (exactly representable reference point).
//  2. per lane: ray of pixel (i,j) re-based in fp64 near C_E.
//  3. per face (App. A.1): project the face's Bernstein
//     points on d1,d2 perpendicular to r (Eq. intersectiontwod); reject when
//     the projected hull excludes the ray; else prove at most one root with
//     ||A J(s) - I|| < 1 (A = J(centre)^-1, J's Bernstein derivative
//     coefficients bound J(s) on the patch) and run Newton; patches that
//     fail the test are subdivided (rare: grazing rays).
//  4. sort roots by alpha, pair entry/exit, and per segment
//     integrate with the N-point GL rule; the field at each node needs
//     xi(x): simplified Newton on X_E(xi) = x warm-started on the straight
//     line between entry and exit xi (tol = camera newton_tol).
#include <cuda_runtime.h>
#include <math.h>

#include "device_math.cuh"
#include "kernels.cuh"

namespace rc {

namespace {

constexpr int WARPS = 4;
constexpr int MAX_ROOTS = 4;   // two segments per (element, ray); more is counted as a failure
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

// X_E(xi) - C_E from the relative Bernstein points sB[m*3+c], m = (m3*3+m2)*3+m1.
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
      const float* p = sB + ((m3 * 3 + m2) * 3) * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = fmaf(bb[m2], fmaf(a2, p[6 + c], fmaf(a1, p[3 + c], a0 * p[c])), y[c]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) X[c] = fmaf(cc[m3], y[c], X[c]);
  }
}

// X and J = dX/dxi (J[c][d]).
__device__ __forceinline__ void eval_XJ(const float* __restrict__ sB, const float xi[3], float X[3], float J[3][3]) {
  float a[3], b[3], c[3], da[3], db[3], dc[3];
  bern(xi[0], a[0], a[1], a[2]);
  bern(xi[1], b[0], b[1], b[2]);
  bern(xi[2], c[0], c[1], c[2]);
  dbern(xi[0], da[0], da[1], da[2]);
  dbern(xi[1], db[0], db[1], db[2]);
  dbern(xi[2], dc[0], dc[1], dc[2]);
#pragma unroll
  for (int q = 0; q < 3; ++q) X[q] = J[q][0] = J[q][1] = J[q][2] = 0.0f;
#pragma unroll
  for (int m3 = 0; m3 < 3; ++m3) {
    float y[3] = {0, 0, 0}, y1[3] = {0, 0, 0}, y2[3] = {0, 0, 0};
#pragma unroll
    for (int m2 = 0; m2 < 3; ++m2) {
      const float* p = sB + ((m3 * 3 + m2) * 3) * 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float v = fmaf(a[2], p[6 + q], fmaf(a[1], p[3 + q], a[0] * p[q]));
        float dv = fmaf(da[2], p[6 + q], fmaf(da[1], p[3 + q], da[0] * p[q]));
        y[q] = fmaf(b[m2], v, y[q]);
        y1[q] = fmaf(b[m2], dv, y1[q]);
        y2[q] = fmaf(db[m2], v, y2[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      X[q] = fmaf(c[m3], y[q], X[q]);
      J[q][0] = fmaf(c[m3], y1[q], J[q][0]);
      J[q][1] = fmaf(c[m3], y2[q], J[q][1]);
      J[q][2] = fmaf(dc[m3], y[q], J[q][2]);
    }
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

// Roots of one face patch in face coordinates [0,1]^2.  Common case: hull
// test + injectivity + Newton.  Rare case: subdivision with a small stack.
// Returns the number of roots written to (u1[], u2[]).
__device__ __noinline__ int face_roots_subdiv(const Patch& root, float tol, int max_it, float* u1, float* u2,
                                              int cap, int* fails) {
  struct Item {
    Patch p;
    float s1a, s2a, w;
  };
  Item stack[32];
  int sp = 0, nr = 0;
  stack[sp++] = Item{root, 0.0f, 0.0f, 1.0f};
  int visited = 0;
  while (sp > 0) {
    Item it = stack[--sp];
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
          u1[nr] = it.s1a + it.w * s1;
          u2[nr] = it.s2a + it.w * s2;
          ++nr;
        }
        continue;
      } else if (st == -1) {
        continue;
      } else if (it.w < 1.0f / 1024.0f || sp > 28 || visited > 1024) {
        ++*fails;
        continue;
      }
      // not converged: split further (sub-patches have smaller q)
    } else if (it.w < 1.0f / 1024.0f || sp > 28 || visited > 1024) {
      // depth limit without an injectivity proof (tangency): Newton from the centre
      float s1 = 0.5f, s2 = 0.5f;
      if (patch_newton(it.p, s1, s2, tol / it.w, max_it) && s1 >= -1e-3f && s1 <= 1.001f && s2 >= -1e-3f &&
          s2 <= 1.001f && nr < cap) {
        u1[nr] = it.s1a + it.w * s1;
        u2[nr] = it.s2a + it.w * s2;
        ++nr;
      }
      continue;
    }
    Patch a, b, aa, ab, ba, bb;
    patch_split(it.p, 0, a, b);
    patch_split(a, 1, aa, ab);
    patch_split(b, 1, ba, bb);
    float h = 0.5f * it.w;
    stack[sp++] = Item{aa, it.s1a, it.s2a, h};
    stack[sp++] = Item{ab, it.s1a, it.s2a + h, h};
    stack[sp++] = Item{ba, it.s1a + h, it.s2a, h};
    stack[sp++] = Item{bb, it.s1a + h, it.s2a + h, h};
  }
  return nr;
}

}  // namespace

template <int P, int N>
__global__ void __launch_bounds__(WARPS * 32, 4) k_cast_curved(CamConst cc, const TreeConst* __restrict__ trees,
                                                               DevLeafView L, const int32_t* __restrict__ vis,
                                                               const Rect16* __restrict__ vrect,
                                                               const int64_t* __restrict__ chunk_off,
                                                               const int32_t* __restrict__ chunk_elem, int64_t nchunks,
                                                               uint32_t key_base, rc_seg* __restrict__ segs,
                                                               int64_t seg_cap, int32_t* __restrict__ hits_pp,
                                                               int64_t* __restrict__ counters) {
  constexpr int NF = (P + 1) * (P + 1) * (P + 1);
  __shared__ double sD[WARPS][2][81];
  __shared__ __align__(16) float sBall[WARPS][84];
  __shared__ float sFall[WARPS][28];
  __shared__ double sOrg[WARPS][3];
  __shared__ float sProj[WARPS][54 * 32];   // projected control points, [m*2+c][lane]
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  float* sB = sBall[warp];
  float* sF = sFall[warp];
  int local_hits = 0, local_fail = 0, face_fail = 0;
  const float tol = cc.newton_tol;
  const int max_it = cc.newton_max;

  for (;;) {
    int64_t c = 0;
    if (lane == 0) c = (int64_t)atomicAdd((unsigned long long*)&counters[CNT_WORK], 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= nchunks) break;
    const int v = chunk_elem[c];
    const int e = vis[v];
    const Rect16 r = vrect[v];
    const int rw = r.i1 - r.i0 + 1, rh = r.j1 - r.j0 + 1;
    const int p = (int)(c - chunk_off[v]) * RC_CHUNK + (int)lane;
    const bool active = p < rw * rh;
    const int i = r.i0 + p % rw, j = r.j0 + p / rw;
    const int lvl = L.level[e];
    const double h = ldexp(1.0, -lvl);

    // ---- 1. element prep: Bernstein restriction, 27 lanes, fp64 ----------
    __syncwarp();
    if (lane < 27) {
      const TreeConst& T = trees[L.tree[e]];
      const int m1 = lane % 3, m2 = (lane / 3) % 3, m3 = lane / 9;
      const int mm[3] = {m1, m2, m3};
      double M[3][3];   // blossom weights of output index mm[k] along axis k
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double u = ldexp((double)L.anchor[3 * (int64_t)e + k], -RC_MAXLEVEL);
        double w = u + h;
        double x = mm[k] == 2 ? w : u, y = mm[k] == 0 ? u : w;
        M[k][0] = (1 - x) * (1 - y);
        M[k][1] = (1 - x) * y + x * (1 - y);
        M[k][2] = x * y;
      }
      double o[3];
      // axis 1: in[m3][m2][q]
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc = fma(M[0][q], T.Bw[((m3 * 3 + m2) * 3 + q) * 3 + q3], acc);
        o[q3] = acc;
      }
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) sD[warp][0][lane * 3 + q3] = o[q3];
      __syncwarp(0x07ffffffu);
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc = fma(M[1][q], sD[warp][0][((m3 * 3 + q) * 3 + m1) * 3 + q3], acc);
        o[q3] = acc;
      }
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) sD[warp][1][lane * 3 + q3] = o[q3];
      __syncwarp(0x07ffffffu);
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) acc = fma(M[2][q], sD[warp][1][((q * 3 + m2) * 3 + m1) * 3 + q3], acc);
        o[q3] = acc;
      }
      if (lane == 13) {
        sOrg[warp][0] = o[0];
        sOrg[warp][1] = o[1];
        sOrg[warp][2] = o[2];
      }
      __syncwarp(0x07ffffffu);
#pragma unroll
      for (int q3 = 0; q3 < 3; ++q3) sB[lane * 3 + q3] = (float)(o[q3] - sOrg[warp][q3]);
      if (lane < NF) sF[lane] = __ldg(&L.field[(int64_t)e * NF + lane]);
    }
    __syncwarp();
    const double org0 = sOrg[warp][0], org1 = sOrg[warp][1], org2 = sOrg[warp][2];

    // ---- 2. ray of pixel (i,j), re-based near the element (fp64) ---------
    const double di = (double)i - 0.5 * (cc.W - 1), dj = (double)j - 0.5 * (cc.H - 1);
    double Rw[3], D[3];
    const double orgv[3] = {org0, org1, org2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      Rw[k] = fma(dj, cc.Ru[k], fma(di, cc.Rt[k], cc.R0[k]));
      double O = fma(dj, cc.Ou[k], fma(di, cc.Ot[k], cc.O0[k]));
      D[k] = orgv[k] - O;
    }
    float rf[3] = {(float)Rw[0], (float)Rw[1], (float)Rw[2]};
    const float rr = rf[0] * rf[0] + rf[1] * rf[1] + rf[2] * rf[2];
    const float alpha0 = ((float)D[0] * rf[0] + (float)D[1] * rf[1] + (float)D[2] * rf[2]) / rr;
    float P0[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) P0[k] = (float)fma((double)alpha0, Rw[k], -D[k]);
    const float rn = sqrtf(rr);

    int nroots = 0;
    RootRec roots[MAX_ROOTS];
    if (active) {
      // projection basis d1, d2 perpendicular to r
      float ax[3] = {0.f, 0.f, 0.f};
      {
        float a0 = fabsf(rf[0]), a1 = fabsf(rf[1]), a2 = fabsf(rf[2]);
        int im = (a0 <= a1 && a0 <= a2) ? 0 : (a1 <= a2 ? 1 : 2);
        ax[im] = 1.0f;
      }
      float d1[3] = {rf[1] * ax[2] - rf[2] * ax[1], rf[2] * ax[0] - rf[0] * ax[2], rf[0] * ax[1] - rf[1] * ax[0]};
      float n1 = rsqrtf(d1[0] * d1[0] + d1[1] * d1[1] + d1[2] * d1[2]);
      d1[0] *= n1; d1[1] *= n1; d1[2] *= n1;
      float d2[3] = {rf[1] * d1[2] - rf[2] * d1[1], rf[2] * d1[0] - rf[0] * d1[2], rf[0] * d1[1] - rf[1] * d1[0]};
      float n2 = rsqrtf(d2[0] * d2[0] + d2[1] * d2[1] + d2[2] * d2[2]);
      d2[0] *= n2; d2[1] *= n2; d2[2] *= n2;
      const float o1 = d1[0] * P0[0] + d1[1] * P0[1] + d1[2] * P0[2];
      const float o2 = d2[0] * P0[0] + d2[1] * P0[1] + d2[2] * P0[2];
      float* sp = sProj[warp] + lane;
#pragma unroll 9
      for (int m = 0; m < 27; ++m) {
        float bx = sB[3 * m], by = sB[3 * m + 1], bz = sB[3 * m + 2];
        sp[(2 * m) * 32] = fmaf(d1[0], bx, fmaf(d1[1], by, fmaf(d1[2], bz, -o1)));
        sp[(2 * m + 1) * 32] = fmaf(d2[0], bx, fmaf(d2[1], by, fmaf(d2[2], bz, -o2)));
      }
      // ---- 3. face roots ------------------------------------------------
#pragma unroll 1
      for (int f = 0; f < 6; ++f) {
        const int k = f >> 1, side = f & 1;
        const int a = (k + 1) % 3, b = (k + 2) % 3;
        Patch pt;
#pragma unroll
        for (int jb = 0; jb < 3; ++jb)
#pragma unroll
          for (int ia = 0; ia < 3; ++ia) {
            int mm[3];
            mm[k] = 2 * side;
            mm[a] = ia;
            mm[b] = jb;
            int m = (mm[2] * 3 + mm[1]) * 3 + mm[0];
            pt.gx[3 * jb + ia] = sp[(2 * m) * 32];
            pt.gy[3 * jb + ia] = sp[(2 * m + 1) * 32];
          }
        if (hull_excludes_origin(pt)) continue;
        float u1[4], u2[4];
        int nf = 0;
        float A11, A12, A21, A22, gcx, gcy;
        float q = injectivity_bound(pt, A11, A12, A21, A22, gcx, gcy);
        if (q < 1.0f) {
          float s1, s2;
          int st = chord_root(pt, A11, A12, A21, A22, gcx, gcy, q, tol, max_it, s1, s2);
          if (st == 1) {
            if (s1 >= -FACE_TOL && s1 <= 1.0f + FACE_TOL && s2 >= -FACE_TOL && s2 <= 1.0f + FACE_TOL) {
              u1[0] = s1;
              u2[0] = s2;
              nf = 1;
            }
          } else if (st == 0) {
            nf = face_roots_subdiv(pt, tol, max_it, u1, u2, 4, &face_fail);   // Newton wandered: split
          }
        } else {
          nf = face_roots_subdiv(pt, tol, max_it, u1, u2, 4, &face_fail);
        }
        if (nroots + nf > MAX_ROOTS) ++face_fail;
        for (int t = 0; t < nf && nroots < MAX_ROOTS; ++t) {
          float xi[3];
          xi[k] = (float)side;
          xi[a] = fminf(fmaxf(u1[t], 0.0f), 1.0f);
          xi[b] = fminf(fmaxf(u2[t], 0.0f), 1.0f);
          float X[3];
          eval_X(sB, xi, X);
          float beta = ((X[0] - P0[0]) * rf[0] + (X[1] - P0[1]) * rf[1] + (X[2] - P0[2]) * rf[2]) / rr;
          // insertion by beta
          int pos = nroots;
          while (pos > 0 && roots[pos - 1].beta > beta) {
            roots[pos] = roots[pos - 1];
            --pos;
          }
          roots[pos].beta = beta;
          roots[pos].xi[0] = xi[0];
          roots[pos].xi[1] = xi[1];
          roots[pos].xi[2] = xi[2];
          ++nroots;
        }
      }
      // dedupe roots found on two faces at a shared edge / vertex
      const float hw = fabsf(sB[3 * 26] - sB[0]) + fabsf(sB[3 * 26 + 1] - sB[1]) + fabsf(sB[3 * 26 + 2] - sB[2]);
      const float dtol = 4e-6f * hw / rn;   // edge roots found on two faces (>= 2x FACE_TOL)
      int m = 0;
      for (int t = 0; t < nroots; ++t) {
        if (m > 0 && roots[t].beta - roots[m - 1].beta < dtol) continue;
        roots[m++] = roots[t];
      }
      nroots = m & ~1;   // entry/exit pairs; an odd leftover is a tangency
    }

    // ---- 4. segments: GL rule with the inverse map per node ---------------
    const int nseg = nroots / 2;
    const float bmin = (float)(cc.amin - (double)alpha0), bmax = (float)(cc.amax - (double)alpha0);
    const int wseg = __reduce_max_sync(0xffffffffu, (unsigned)nseg);
    bool any_out = false;
    const uint32_t pix = (uint32_t)(j * cc.W + i);
    for (int s = 0; s < wseg; ++s) {
      bool have = false;
      float a = 1.0f, bb[3] = {0.f, 0.f, 0.f}, an = 0.f, af = 0.f;
      if (s < nseg) {
        const RootRec& ra = roots[2 * s];
        const RootRec& rb = roots[2 * s + 1];
        float b0 = fmaxf(ra.beta, bmin), b1 = fminf(rb.beta, bmax);
        if (b1 > b0) {
          have = true;
          const float db = b1 - b0;
          const float Lseg = db * rn;
          float xin[3] = {ra.xi[0], ra.xi[1], ra.xi[2]};
          float dxi[3] = {rb.xi[0] - ra.xi[0], rb.xi[1] - ra.xi[1], rb.xi[2] - ra.xi[2]};
          float xm[3] = {xin[0] + 0.5f * dxi[0], xin[1] + 0.5f * dxi[1], xin[2] + 0.5f * dxi[2]};
          float Xm[3], Jm[3][3], Ji[3][3];
          eval_XJ(sB, xm, Xm, Jm);
          bool okJ = inv3(Jm, Ji);
          float ft[N];
#pragma unroll
          for (int q = 0; q < N; ++q) {
            const float bq = fmaf(cc.u[q], db, b0);
            const float tx = fmaf(bq, rf[0], P0[0]), ty = fmaf(bq, rf[1], P0[1]), tz = fmaf(bq, rf[2], P0[2]);
            float xi[3] = {fmaf(cc.u[q], dxi[0], xin[0]), fmaf(cc.u[q], dxi[1], xin[1]),
                           fmaf(cc.u[q], dxi[2], xin[2])};
            bool conv = false;
            float last = 3.4e38f;
            for (int it = 0; okJ && it < max_it; ++it) {
              float X[3];
              float Jc[3][3], Jci[3][3];
              const bool full = it >= 3;   // simplified Newton first, full Newton if it stalls
              if (full) {
                eval_XJ(sB, xi, X, Jc);
                if (!inv3(Jc, Jci)) break;
              } else {
                eval_X(sB, xi, X);
              }
              const float(*A)[3] = full ? Jci : Ji;
              float rx = tx - X[0], ry = ty - X[1], rz = tz - X[2];
              float s0 = A[0][0] * rx + A[0][1] * ry + A[0][2] * rz;
              float s1 = A[1][0] * rx + A[1][1] * ry + A[1][2] * rz;
              float s2 = A[2][0] * rx + A[2][1] * ry + A[2][2] * rz;
              xi[0] += s0;
              xi[1] += s1;
              xi[2] += s2;
              float step = fmaxf(fabsf(s0), fmaxf(fabsf(s1), fabsf(s2)));
              if (step < tol) {
                conv = true;
                break;
              }
              last = step;
            }
            (void)last;
            if (!conv) ++local_fail;
            // the node lies inside the element: clamp against rounding (and
            // against divergence, which is counted above)
            xi[0] = fminf(fmaxf(xi[0], 0.0f), 1.0f);
            xi[1] = fminf(fmaxf(xi[1], 0.0f), 1.0f);
            xi[2] = fminf(fmaxf(xi[2], 0.0f), 1.0f);
            ft[q] = field_at<P>(sF, xi[0], xi[1], xi[2]) * cc.inv_F;
          }
          gl_rule<N>(cc, ft, Lseg, a, bb);
          an = alpha0 + b0;
          af = alpha0 + b1;
        }
      }
      int64_t slot = warp_append(&counters[CNT_SEGS], have ? 1 : 0);
      if (have) {
        any_out = true;
        if (slot < seg_cap) store_seg(segs + slot, pix, an, af, a, bb, key_base + (uint32_t)e);
        else atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
      }
    }
    if (any_out) {
      ++local_hits;
      atomicAdd(&hits_pp[pix], 1);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    local_hits += __shfl_down_sync(0xffffffffu, local_hits, off);
    local_fail += __shfl_down_sync(0xffffffffu, local_fail, off);
    face_fail += __shfl_down_sync(0xffffffffu, face_fail, off);
  }
  if (lane == 0) {
    if (local_hits) atomicAdd((unsigned long long*)&counters[CNT_HITPAIRS], (unsigned long long)local_hits);
    if (local_fail + face_fail)
      atomicAdd((unsigned long long*)&counters[CNT_NEWTON_FAIL], (unsigned long long)(local_fail + face_fail));
    if (face_fail) atomicAdd((unsigned long long*)&counters[CNT_FACE_FAIL], (unsigned long long)face_fail);
  }
}

template <int P>
static void curved_P(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                     const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem, int64_t nchunks,
                     uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp, int64_t* counters, int grid,
                     cudaStream_t s) {
#define CASE(N)                                                                                                     \
  case N:                                                                                                           \
    k_cast_curved<P, N><<<grid, WARPS * 32, 0, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks,      \
                                                    key_base, segs, seg_cap, hits_pp, counters);                    \
    break;
  switch (cc.N) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) }
#undef CASE
}

cudaError_t launch_cast_curved(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                               int64_t* counters, int grid, cudaStream_t s) {
  if (P == 1)
    curved_P<1>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base, segs, seg_cap, hits_pp, counters,
                grid, s);
  else
    curved_P<2>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base, segs, seg_cap, hits_pp, counters,
                grid, s);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace rc
