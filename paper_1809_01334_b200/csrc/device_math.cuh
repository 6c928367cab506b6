// device_math.cuh -- device helpers of the segment kernels: nodal field
// interpolation, the nested Gauss-Legendre segment rule, record output.
#pragma once
#include "rc_internal.cuh"
#include "geom.cuh"

namespace rc {

// Lagrange basis on the GLL nodes {0, 1/2, 1} (Eq. nodal)
__device__ __forceinline__ void lag2(float t, float& l0, float& l1, float& l2) {
  float tm = 1.0f - t;
  l0 = tm * (1.0f - 2.0f * t);
  l1 = 4.0f * t * tm;
  l2 = t * (2.0f * t - 1.0f);
}

// Field at element reference point xi from the element's nodal values
// (node order [k3][k2][k1]).  P = 1: trilinear; P = 2: triquadratic.
template <int P>
__device__ __forceinline__ float field_at(const float* f, float x1, float x2, float x3);

template <>
__device__ __forceinline__ float field_at<1>(const float* f, float x1, float x2, float x3) {
  float a00 = fmaf(x1, f[1] - f[0], f[0]);
  float a10 = fmaf(x1, f[3] - f[2], f[2]);
  float a01 = fmaf(x1, f[5] - f[4], f[4]);
  float a11 = fmaf(x1, f[7] - f[6], f[6]);
  float b0 = fmaf(x2, a10 - a00, a00);
  float b1 = fmaf(x2, a11 - a01, a01);
  return fmaf(x3, b1 - b0, b0);
}

template <>
__device__ __forceinline__ float field_at<2>(const float* f, float x1, float x2, float x3) {
  float p0, p1, p2, q0, q1, q2, r0, r1, r2;
  lag2(x1, p0, p1, p2);
  lag2(x2, q0, q1, q2);
  lag2(x3, r0, r1, r2);
  float out = 0.0f;
  float rr[3] = {r0, r1, r2};
#pragma unroll
  for (int k3 = 0; k3 < 3; ++k3) {
    const float* g = f + 9 * k3;
    float s0 = fmaf(p2, g[2], fmaf(p1, g[1], p0 * g[0]));
    float s1 = fmaf(p2, g[5], fmaf(p1, g[4], p0 * g[3]));
    float s2 = fmaf(p2, g[8], fmaf(p1, g[7], p0 * g[6]));
    out = fmaf(rr[k3], fmaf(q2, s2, fmaf(q1, s1, q0 * s0)), out);
  }
  return out;
}

// SURVEY R13 nested GL rule: a = exp(-L sum w kappa), tau_j = L sum_k S_jk kappa_k,
// b_c = L sum_j w_j q_cj exp(-tau_j), with q = q0((1+f~)/2, (1-f~)/2, 1/2).
// Inputs: fn[j] = f~ at the N nodes (ordered from the near end).
template <int N>
__device__ __forceinline__ void gl_rule(const CamConst& cc, const float* ft, float L, float& a, float b[3]) {
  float kap[N];
  float sumk = 0.0f;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    kap[j] = cc.kappa0 * ft[j] * ft[j];
    sumk = fmaf(cc.w[j], kap[j], sumk);
  }
  a = __expf(-L * sumk);
  float E0 = 0.0f, E1 = 0.0f;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    float t = 0.0f;
#pragma unroll
    for (int k = 0; k < N; ++k) t = fmaf(cc.S[j * RC_MAX_N + k], kap[k], t);
    float e = cc.w[j] * __expf(-L * t);
    E0 += e;
    E1 = fmaf(e, ft[j], E1);
  }
  float s = 0.5f * L * cc.q0;
  b[0] = s * (E0 + E1);
  b[1] = s * (E0 - E1);
  b[2] = s * E0;
}

// ---------------------------------------------------------------------------
// The paper's per-segment integrators with the adaptive recursion of Alg. 1
// (SURVEY §8(f) NEXT(1), NEXT(2)), selected by
// rc_camera.scheme.  Positions: t = fraction of the segment from its
// upstream (far) end x1, so the near-end parameter of the media
// callbacks is u = 1 - t.  Alg. 1's recursion runs without a stack: the
// sub-intervals are dyadic (k 2^-lev, 2^-lev) and are visited downstream
// first (near to far), so the pieces fold as acc (+) piece; after an accepted
// piece the walk climbs while it was a far (even) child and moves to the far
// sibling.  An attempted step is abandoned when it evaluates dx beta > c_RK
// at one of its nodes; at max_depth the step is taken anyway and counted.
// ---------------------------------------------------------------------------
struct MediumSample {
  float beta, g0, g1, g2;   // kappa and q (RGB) at one point
};

__device__ __forceinline__ MediumSample medium_from_f(const CamConst& cc, float ft) {
  MediumSample m;
  m.beta = cc.kappa0 * ft * ft;
  m.g0 = cc.q0 * 0.5f * (1.0f + ft);
  m.g1 = cc.q0 * 0.5f * (1.0f - ft);
  m.g2 = cc.q0 * 0.5f;
  return m;
}

// One attempted step on [t1, t1 + d] (fractions of the segment, length dx
// physical).  Returns false when the Alg. 1 test asks for a split.
template <class Med>
__device__ __forceinline__ bool scheme_step(const CamConst& cc, const Med& med, float t1, float d, float dx, bool force,
                                            float& A, float B[3]) {
  const float crk = force ? 0.0f : cc.c_rk;
  auto over = [&](float beta) { return crk > 0.0f && dx * beta > crk; };
  auto at = [&](float t) { return med(1.0f - t); };   // near-end parameter u = 1 - t
  if (cc.scheme == RC_SCHEME_GAUSS2) {   // Eq. gaussAB / gaussABab, xi = 1/2 -+ sqrt(3)/6 from x1
    const MediumSample m0 = at(t1 + 0.21132486540518713f * d), m1 = at(t1 + 0.78867513459481287f * d);
    if (over(m0.beta) || over(m1.beta)) return false;
    const float a1 = dx * (m0.beta + m1.beta) * 0.25f, a2 = dx * dx * m0.beta * m1.beta * (1.0f / 12.0f);
    const float den = 1.0f / (1.0f + a1 + a2);
    A = (1.0f - a1 + a2) * den;
    const float k2 = dx * dx * 0.14433756729740644f;   // sqrt(3)/12
    B[0] = (dx * 0.5f * (m0.g0 + m1.g0) + k2 * (m0.beta * m1.g0 - m1.beta * m0.g0)) * den;
    B[1] = (dx * 0.5f * (m0.g1 + m1.g1) + k2 * (m0.beta * m1.g1 - m1.beta * m0.g1)) * den;
    B[2] = (dx * 0.5f * (m0.g2 + m1.g2) + k2 * (m0.beta * m1.g2 - m1.beta * m0.g2)) * den;
    return true;
  }
  if (cc.scheme == RC_SCHEME_SIMPSON) {   // Eq. simpson, nodes x1, x1 + dx/2, x2
    const MediumSample m0 = at(t1), m1 = at(t1 + 0.5f * d), m2 = at(t1 + d);
    if (over(m0.beta) || over(m1.beta) || over(m2.beta)) return false;
    A = __expf(-dx * (m0.beta + 4.0f * m1.beta + m2.beta) * (1.0f / 6.0f));
    const float sA = sqrtf(A);
    B[0] = dx * (A * m0.g0 + 4.0f * sA * m1.g0 + m2.g0) * (1.0f / 6.0f);
    B[1] = dx * (A * m0.g1 + 4.0f * sA * m1.g1 + m2.g1) * (1.0f / 6.0f);
    B[2] = dx * (A * m0.g2 + 4.0f * sA * m1.g2 + m2.g2) * (1.0f / 6.0f);
    return true;
  }
  if (cc.scheme == RC_SCHEME_GL) {   // SURVEY R13 on the sub-interval, nodes u_j from its near end
    float kap[RC_MAX_N], g[RC_MAX_N][3];
    for (int j = 0; j < cc.N; ++j) {
      const MediumSample m = at(t1 + d - cc.u[j] * d);
      if (over(m.beta)) return false;
      kap[j] = m.beta;
      g[j][0] = m.g0;
      g[j][1] = m.g1;
      g[j][2] = m.g2;
    }
    float sumk = 0.0f;
    for (int j = 0; j < cc.N; ++j) sumk = fmaf(cc.w[j], kap[j], sumk);
    A = __expf(-dx * sumk);
    B[0] = B[1] = B[2] = 0.0f;
    for (int j = 0; j < cc.N; ++j) {
      float tau = 0.0f;
      for (int k = 0; k < cc.N; ++k) tau = fmaf(cc.S[j * RC_MAX_N + k], kap[k], tau);
      const float e = dx * cc.w[j] * __expf(-dx * tau);
      B[0] = fmaf(e, g[j][0], B[0]);
      B[1] = fmaf(e, g[j][1], B[1]);
      B[2] = fmaf(e, g[j][2], B[2]);
    }
    return true;
  }
  // explicit RK (Eq. RKresultAB; subdiagonal stages, a_Mj = b_j for the final values)
  int M;
  float c[4], asub[4], bw[4];
  switch (cc.scheme) {
    case RC_SCHEME_EULER: M = 1; c[0] = 0.f; bw[0] = 1.f; break;
    case RC_SCHEME_HEUN2: M = 2; c[0] = 0.f; c[1] = 1.f; asub[1] = 1.f; bw[0] = bw[1] = 0.5f; break;
    case RC_SCHEME_HEUN3:
      M = 3; c[0] = 0.f; c[1] = 1.f / 3; c[2] = 2.f / 3; asub[1] = 1.f / 3; asub[2] = 2.f / 3;
      bw[0] = 0.25f; bw[1] = 0.f; bw[2] = 0.75f; break;
    default:   // RC_SCHEME_RK4
      M = 4; c[0] = 0.f; c[1] = c[2] = 0.5f; c[3] = 1.f; asub[1] = asub[2] = 0.5f; asub[3] = 1.f;
      bw[0] = bw[3] = 1.f / 6; bw[1] = bw[2] = 1.f / 3; break;
  }
  // stage i: Ab_i = 1 + dx a_{i,i-1} (-beta_{i-1} Ab_{i-1}), Bb_i = dx a_{i,i-1} (g_{i-1} - beta_{i-1} Bb_{i-1});
  // final values accumulated as A = 1 + dx sum_j b_j (-beta_j Ab_j), B = dx sum_j b_j (g_j - beta_j Bb_j)
  MediumSample mprev = at(t1 + c[0] * d);
  float Ab = 1.0f, Bb[3] = {0.f, 0.f, 0.f};
  float Af = 1.0f - dx * bw[0] * mprev.beta;
  float Bf[3] = {dx * bw[0] * mprev.g0, dx * bw[0] * mprev.g1, dx * bw[0] * mprev.g2};
  for (int i = 1; i < M; ++i) {
    if (over(mprev.beta)) return false;   // Alg. 1: stage i evaluated dx beta(xi_{i-1})
    const float Ai = 1.0f + dx * asub[i] * (-mprev.beta * Ab);
    const float B0 = dx * asub[i] * (mprev.g0 - mprev.beta * Bb[0]);
    const float B1 = dx * asub[i] * (mprev.g1 - mprev.beta * Bb[1]);
    const float B2 = dx * asub[i] * (mprev.g2 - mprev.beta * Bb[2]);
    Ab = Ai;
    Bb[0] = B0;
    Bb[1] = B1;
    Bb[2] = B2;
    mprev = at(t1 + c[i] * d);
    Af += dx * bw[i] * (-mprev.beta * Ab);
    Bf[0] += dx * bw[i] * (mprev.g0 - mprev.beta * Bb[0]);
    Bf[1] += dx * bw[i] * (mprev.g1 - mprev.beta * Bb[1]);
    Bf[2] += dx * bw[i] * (mprev.g2 - mprev.beta * Bb[2]);
  }
  if (over(mprev.beta)) return false;     // the final values evaluated dx beta(xi_{M-1})
  A = Af;
  B[0] = Bf[0];
  B[1] = Bf[1];
  B[2] = Bf[2];
  return true;
}

// Alg. 1 over the whole segment of physical length L: (a, b) of the segment.
template <class Med>
__device__ __noinline__ void segment_scheme(const CamConst& cc, float L, const Med& med, float& a_out, float b_out[3],
                                            int& capped) {
  float A = 1.0f, B0 = 0.0f, B1 = 0.0f, B2 = 0.0f;   // fold of the accepted pieces, nearest first
  int k = 0, lev = 0;
  for (;;) {
    const float d = ldexpf(1.0f, -lev), t1 = (float)k * d;
    float pa, pb[3];
    bool ok = scheme_step(cc, med, t1, d, d * L, false, pa, pb);
    if (!ok && lev < cc.max_depth) {   // Alg. 1: split, downstream half first
      k = 2 * k + 1;
      ++lev;
      continue;
    }
    if (!ok) {
      ++capped;
      scheme_step(cc, med, t1, d, d * L, true, pa, pb);
    }
    B0 = fmaf(A, pb[0], B0);   // acc (+) piece (Eq. aggregate)
    B1 = fmaf(A, pb[1], B1);
    B2 = fmaf(A, pb[2], B2);
    A *= pa;
    while (lev > 0 && (k & 1) == 0) {   // finished a far half: its parent is done
      k >>= 1;
      --lev;
    }
    if (lev == 0) break;
    --k;   // the far sibling
  }
  a_out = A;
  b_out[0] = B0;
  b_out[1] = B1;
  b_out[2] = B2;
}


__device__ __forceinline__ void store_seg(rc_seg* dst, uint32_t pixel, float an, float af, float a, const float b[3],
                                          uint32_t key) {
  float4 lo = make_float4(__uint_as_float(pixel), an, af, a);
  float4 hi = make_float4(b[0], b[1], b[2], __uint_as_float(key));
  float4* d = reinterpret_cast<float4*>(dst);
  d[0] = lo;
  d[1] = hi;
}

// warp-aggregated append of `want` records per lane; returns this lane's first slot
__device__ __forceinline__ int64_t warp_append(int64_t* counter, int want) {
  unsigned lane = threadIdx.x & 31;
  int incl = want;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, off);
    if ((int)lane >= off) incl += y;
  }
  int total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total > 0) base = atomicAdd((unsigned long long*)counter, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return (int64_t)base + incl - want;
}

}  // namespace rc
