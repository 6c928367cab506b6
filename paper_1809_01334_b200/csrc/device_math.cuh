// device_math.cuh -- device helpers of the segment kernels: nodal field
// interpolation, the nested Gauss-Legendre segment rule, record output.
#pragma once
#include "rc_internal.cuh"

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
