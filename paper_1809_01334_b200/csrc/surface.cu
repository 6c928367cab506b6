// surface.cu -- surface forests: cull and point
// intersection of quadtree leaves on bilinear tree patches.
//
// PAPER.md:780-808 (§2.8, Eq. ABphi): a surface meets a ray in points; each
// point is a zero-length record with A = A_s^(1/cos phi) and b = I_s (1 - A)
// (Eq. BIrelation), phi the angle between the ray and the surface normal.
// PAPER.md:1473-1514 (App. A.1): with d1, d2 perpendicular to the ray, the
// projected patch is the 2D bilinear map g(s) = a + b s1 + c s2 + d s1 s2 and
// g(s) = 0 is a quadratic in s2 after eliminating s1 (at most two points).
//
// The records enter the volume path's rows unchanged: the pair work list
// (a3), aggregation (a7, zero-length records touch only at equal alpha) and
// the composite (a9).  Geometry is fp64 (B200 runs fp64 at half the fp32
// rate; a pair costs ~200 flops against a 32-byte record), the transfer fp32.
#include <cuda_runtime.h>
#include <math.h>

#include "device_math.cuh"
#include "kernels.cuh"

namespace rc {


// a2 (surfaces): camera-space AABB of the leaf patch's four corners (a
// bilinear patch lies in their convex hull) -> pixel-centre rectangle.
__global__ void __launch_bounds__(256) k_cull_surface(CamConst cc, const TreeConst* __restrict__ trees,
                                                      DevLeafView L, int64_t n, int32_t* __restrict__ flag,
                                                      Rect16* __restrict__ rect) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const TreeConst& T = trees[L.tree[e]];
  const double h = ldexp(1.0, -(int)L.level[e]);
  const double t1 = ldexp((double)L.anchor[3 * e], -RC_MAXLEVEL), t2 = ldexp((double)L.anchor[3 * e + 1], -RC_MAXLEVEL);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double X[3];
    patch_point(T.Bc, t1 + h * (q & 1), t2 + h * (q >> 1), X);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], X[c]);
      hi[c] = fmax(hi[c], X[c]);
    }
  }
  Rect16 rc{0, -1, 0, -1};
  const bool v = project_rect(cc, lo, hi, rc);
  flag[e] = v ? 1 : 0;
  rect[e] = rc;
}

// a4 + a5 (surfaces): one warp = one 32-pixel chunk of one visible leaf
// (the affine kernel's work list and dynamic chunk scheduling).
__global__ void __launch_bounds__(256) k_cast_surface(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L,
                                                      const int32_t* __restrict__ vis, const Rect16* __restrict__ vrect,
                                                      const int64_t* __restrict__ chunk_off,
                                                      const int32_t* __restrict__ chunk_elem, int64_t nchunks,
                                                      uint32_t key_base, rc_seg* __restrict__ segs, int64_t seg_cap,
                                                      int32_t* __restrict__ hits_pp, int64_t* __restrict__ counters) {
  const unsigned lane = threadIdx.x & 31;
  int local_pairs = 0;
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

    const TreeConst& T = trees[L.tree[e]];
    const double h = ldexp(1.0, -(int)L.level[e]);
    const double t1 = ldexp((double)L.anchor[3 * (int64_t)e], -RC_MAXLEVEL);
    const double t2 = ldexp((double)L.anchor[3 * (int64_t)e + 1], -RC_MAXLEVEL);
    const float4 fv = __ldg(reinterpret_cast<const float4*>(L.field) + e);   // corner values [k2][k1]

    // ray of pixel (i,j) and the leaf's corners relative to its origin
    const double di = (double)i - 0.5 * (cc.W - 1), dj = (double)j - 0.5 * (cc.H - 1);
    double O[3], R[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      O[k] = fma(dj, cc.Ou[k], fma(di, cc.Ot[k], cc.O0[k]));
      R[k] = fma(dj, cc.Ru[k], fma(di, cc.Rt[k], cc.R0[k]));
    }
    double P[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      patch_point(T.Bw, t1 + h * (q & 1), t2 + h * (q >> 1), P[q]);
#pragma unroll
      for (int k = 0; k < 3; ++k) P[q][k] -= O[k];
    }
    // d1 = R x axis (the coordinate axis least aligned with R), d2 = R x d1
    const double ax = fabs(R[0]), ay = fabs(R[1]), az = fabs(R[2]);
    const int m = (ax <= ay && ax <= az) ? 0 : (ay <= az ? 1 : 2);
    double d1[3] = {m == 0 ? 0.0 : (m == 1 ? -R[2] : R[1]), m == 0 ? R[2] : (m == 1 ? 0.0 : -R[0]),
                    m == 0 ? -R[1] : (m == 1 ? R[0] : 0.0)};
    double d2[3] = {R[1] * d1[2] - R[2] * d1[1], R[2] * d1[0] - R[0] * d1[2], R[0] * d1[1] - R[1] * d1[0]};
    double g[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      g[q][0] = d1[0] * P[q][0] + d1[1] * P[q][1] + d1[2] * P[q][2];
      g[q][1] = d2[0] * P[q][0] + d2[1] * P[q][1] + d2[2] * P[q][2];
    }
    double A2[2], B2[2], C2[2], D2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      A2[k] = g[0][k];
      B2[k] = g[1][k] - g[0][k];
      C2[k] = g[2][k] - g[0][k];
      D2[k] = g[3][k] - g[2][k] - g[1][k] + g[0][k];
    }
    // (a + c s2) x (b + d s2) = 0:  qq s2^2 + q1 s2 + q0 = 0
    const double q0 = A2[0] * B2[1] - A2[1] * B2[0];
    const double q1 = A2[0] * D2[1] - A2[1] * D2[0] + C2[0] * B2[1] - C2[1] * B2[0];
    const double qq = C2[0] * D2[1] - C2[1] * D2[0];
    double root[2];
    int nr = 0;
    if (fabs(qq) <= 1e-14 * (fabs(q0) + fabs(q1) + fabs(qq))) {
      if (q1 != 0.0) root[nr++] = -q0 / q1;
    } else {
      const double disc = q1 * q1 - 4.0 * qq * q0;
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        const double t = -0.5 * (q1 + (q1 >= 0.0 ? sq : -sq));   // stable quadratic formula
        root[nr++] = t / qq;
        if (t != 0.0) root[nr++] = q0 / t;
      }
    }
    float ra[2], rA[2], rb[2][3];
    int nh = 0;
    const double rr = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
    for (int k = 0; k < nr && active; ++k) {
      const double s2 = root[k];
      if (!(s2 >= 0.0 && s2 < 1.0)) continue;
      const double u0 = B2[0] + D2[0] * s2, u1 = B2[1] + D2[1] * s2;
      const double w0 = A2[0] + C2[0] * s2, w1 = A2[1] + C2[1] * s2;
      const double uu = u0 * u0 + u1 * u1;
      if (!(uu > 0.0)) continue;
      const double s1 = -(w0 * u0 + w1 * u1) / uu;
      if (!(s1 >= 0.0 && s1 < 1.0)) continue;
      double X[3], e1[3], e2[3];
#pragma unroll
      for (int c3 = 0; c3 < 3; ++c3) {
        X[c3] = (1.0 - s2) * ((1.0 - s1) * P[0][c3] + s1 * P[1][c3]) + s2 * ((1.0 - s1) * P[2][c3] + s1 * P[3][c3]);
        e1[c3] = (1.0 - s2) * (P[1][c3] - P[0][c3]) + s2 * (P[3][c3] - P[2][c3]);
        e2[c3] = (1.0 - s1) * (P[2][c3] - P[0][c3]) + s1 * (P[3][c3] - P[1][c3]);
      }
      const double alpha = (X[0] * R[0] + X[1] * R[1] + X[2] * R[2]) / rr;
      if (!(alpha >= cc.amin && alpha <= cc.amax)) continue;
      const double nx = e1[1] * e2[2] - e1[2] * e2[1], ny = e1[2] * e2[0] - e1[0] * e2[2],
                   nz = e1[0] * e2[1] - e1[1] * e2[0];
      const double cphi = fabs(nx * R[0] + ny * R[1] + nz * R[2]) / sqrt((nx * nx + ny * ny + nz * nz) * rr);
      // Eq. ABphi on the bilinearly interpolated corner value
      const float fs1 = (float)s1, fs2 = (float)s2;
      const float val = (1.0f - fs2) * ((1.0f - fs1) * fv.x + fs1 * fv.y) + fs2 * ((1.0f - fs1) * fv.z + fs1 * fv.w);
      const float As = fminf(1.0f, fmaxf(0.0f, fmaf(cc.surf.a[1], val, cc.surf.a[0])));
      const float wk = (1.0f - val) * cc.surf.k;
      const float wgt = expf(-0.5f * wk * wk);
      const float Aphi = As == 0.0f ? 0.0f : powf(As, (float)(1.0 / cphi));
      ra[nh] = (float)alpha;
      rA[nh] = Aphi;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
        rb[nh][ch] = fmaf(cc.surf.i[ch][2], wgt, fmaf(cc.surf.i[ch][1], val, cc.surf.i[ch][0])) * (1.0f - Aphi);
      ++nh;
    }
    int64_t slot = warp_append(&counters[CNT_SEGS], nh);
    if (nh > 0) {
      const uint32_t pix = (uint32_t)(j * cc.W + i);
      for (int k = 0; k < nh; ++k, ++slot) {
        if (slot < seg_cap) store_seg(segs + slot, pix, ra[k], ra[k], rA[k], rb[k], key_base + (uint32_t)e);
        else atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
      }
      atomicAdd(&hits_pp[pix], 1);
      ++local_pairs;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) local_pairs += __shfl_down_sync(0xffffffffu, local_pairs, off);
  if (lane == 0 && local_pairs) atomicAdd((unsigned long long*)&counters[CNT_HITPAIRS], (unsigned long long)local_pairs);
}

cudaError_t launch_cull_surface(const CamConst& cc, const TreeConst* trees, DevLeafView L, int64_t n, int32_t* flag,
                                Rect16* rect, cudaStream_t s) {
  k_cull_surface<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cc, trees, L, n, flag, rect);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_cast_surface(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                                const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                                int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                                int64_t* counters, int grid, cudaStream_t s) {
  k_cast_surface<<<grid, 256, 0, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base, segs,
                                      seg_cap, hits_pp, counters);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace rc
