// kernels.cu -- cull, pair generation, affine segment kernel, composite.
//
// Hot-path rows: a2 cull (k_cull_*), a3 pair generation
// (k_chunk_count, k_expand), a4+a5 ray-element intersection + GL segment
// integration for affine trees (k_cast_affine), a8 pack (k_pack_*), a9 tile
// composite (k_hist, k_scatter, k_fold).  Curved R=2 segments: cast_curved.cu.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "device_math.cuh"
#include "kernels.cuh"

namespace rc {

// ---------------------------------------------------------------------------
// a2: cull.  Camera-space AABB of the element's Bernstein-Bezier points ->
// pixel-centre rectangle.  fp64 so that the decision differs
// from the fp64 oracle only for eps-ambiguous leaves.
// ---------------------------------------------------------------------------
__device__ bool project_rect(const CamConst& cc, const double lo[3], const double hi[3], Rect16& rc) {
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

__global__ void k_cull_affine(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L, int64_t n,
                              int32_t* __restrict__ flag, Rect16* __restrict__ rect) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const TreeConst& T = trees[L.tree[e]];
  double h = ldexp(1.0, -(int)L.level[e]);
  double t[3];
  for (int k = 0; k < 3; ++k) t[k] = ldexp((double)L.anchor[3 * e + k], -RC_MAXLEVEL) + 0.5 * h;
  double lo[3], hi[3];
  for (int c = 0; c < 3; ++c) {
    double X = T.bcam[c], ext = 0.0;
    for (int k = 0; k < 3; ++k) {
      X = fma(T.Acam[3 * c + k], t[k], X);
      ext += fabs(T.Acam[3 * c + k]);
    }
    ext *= 0.5 * h;
    lo[c] = X - ext;
    hi[c] = X + ext;
  }
  Rect16 rc{0, -1, 0, -1};
  bool v = project_rect(cc, lo, hi, rc);
  flag[e] = v ? 1 : 0;
  rect[e] = rc;
}

// Restriction of a degree-R Bernstein polynomial (along one axis) to [u,v]:
// new control points are blossom values P(u..u, v..v) (de Casteljau).
template <int R>
__device__ __forceinline__ void bz_restrict_row(double u, double v, double M[R + 1][R + 1]);

template <>
__device__ __forceinline__ void bz_restrict_row<1>(double u, double v, double M[2][2]) {
  M[0][0] = 1 - u; M[0][1] = u;
  M[1][0] = 1 - v; M[1][1] = v;
}
template <>
__device__ __forceinline__ void bz_restrict_row<2>(double u, double v, double M[3][3]) {
  // blossom P(x,y) = (1-x)(1-y) p0 + ((1-x)y + x(1-y)) p1 + x y p2
  double x[3] = {u, u, v}, y[3] = {u, v, v};
  for (int r = 0; r < 3; ++r) {
    M[r][0] = (1 - x[r]) * (1 - y[r]);
    M[r][1] = (1 - x[r]) * y[r] + x[r] * (1 - y[r]);
    M[r][2] = x[r] * y[r];
  }
}

// Element Bernstein points from the tree's (index [m3][m2][m1][xyz]).
template <int R>
__device__ void element_bezier(const double* __restrict__ Btree, const double t0[3], double h, double* B) {
  constexpr int n1 = R + 1;
  double M[3][n1][n1];
  for (int k = 0; k < 3; ++k) bz_restrict_row<R>(t0[k], t0[k] + h, M[k]);
  double tmp[n1 * n1 * n1 * 3];
  // axis 1
  for (int m3 = 0; m3 < n1; ++m3)
    for (int m2 = 0; m2 < n1; ++m2)
      for (int r = 0; r < n1; ++r)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int m1 = 0; m1 < n1; ++m1) s = fma(M[0][r][m1], Btree[((m3 * n1 + m2) * n1 + m1) * 3 + c], s);
          tmp[((m3 * n1 + m2) * n1 + r) * 3 + c] = s;
        }
  // axis 2
  for (int m3 = 0; m3 < n1; ++m3)
    for (int r = 0; r < n1; ++r)
      for (int m1 = 0; m1 < n1; ++m1)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int m2 = 0; m2 < n1; ++m2) s = fma(M[1][r][m2], tmp[((m3 * n1 + m2) * n1 + m1) * 3 + c], s);
          B[((m3 * n1 + r) * n1 + m1) * 3 + c] = s;
        }
  // axis 3
  for (int r = 0; r < n1; ++r)
    for (int m2 = 0; m2 < n1; ++m2)
      for (int m1 = 0; m1 < n1; ++m1)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int m3 = 0; m3 < n1; ++m3) s = fma(M[2][r][m3], B[((m3 * n1 + m2) * n1 + m1) * 3 + c], s);
          tmp[((r * n1 + m2) * n1 + m1) * 3 + c] = s;
        }
  for (int q = 0; q < n1 * n1 * n1 * 3; ++q) B[q] = tmp[q];
}

#ifndef CULL_ROWWISE
#define CULL_ROWWISE 0   // 1: R = 2 cull restricts row by row with min / max on the fly (A/B: 17.0 -> 19.1 ms, spills; rejected)
#endif
template <int R>
__global__ void __launch_bounds__(128, CULL_ROWWISE ? 4 : 1) k_cull_curved(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L, int64_t n,
                              int32_t* __restrict__ flag, Rect16* __restrict__ rect) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  constexpr int NP = (R + 1) * (R + 1) * (R + 1);
  const TreeConst& T = trees[L.tree[e]];
  double h = ldexp(1.0, -(int)L.level[e]);
  double t0[3];
  for (int k = 0; k < 3; ++k) t0[k] = ldexp((double)L.anchor[3 * e + k], -RC_MAXLEVEL);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#if CULL_ROWWISE
  if constexpr (R == 2) {
    // the same restriction row by row (axis 3, then 2, then 1), min / max on
    // the fly: ~100 registers instead of two 81-double arrays
    double M0[3][3];   // axis 1; the rows of axes 2 and 3 are formed when used
    bz_restrict_row<2>(t0[0], t0[0] + h, M0);
    const double* __restrict__ Bt = T.Bc;
    auto row = [&](int k, int r, double m[3]) {   // blossom row r of axis k (bz_restrict_row<2>)
      const double u = t0[k], v = t0[k] + h;
      const double x = r == 2 ? v : u, y = r == 0 ? u : v;
      m[0] = (1 - x) * (1 - y);
      m[1] = (1 - x) * y + x * (1 - y);
      m[2] = x * y;
    };
#pragma unroll 1
    for (int r3 = 0; r3 < 3; ++r3) {
      double m3[3];
      row(2, r3, m3);
      double T2[9][3];
#pragma unroll
      for (int q21 = 0; q21 < 9; ++q21)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int q3 = 0; q3 < 3; ++q3) acc = fma(m3[q3], Bt[(q3 * 9 + q21) * 3 + c], acc);
          T2[q21][c] = acc;
        }
#pragma unroll 1
      for (int r2 = 0; r2 < 3; ++r2) {
        double m2[3];
        row(1, r2, m2);
        double T1[3][3];
#pragma unroll
        for (int q1 = 0; q1 < 3; ++q1)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < 3; ++q2) acc = fma(m2[q2], T2[q2 * 3 + q1][c], acc);
            T1[q1][c] = acc;
          }
#pragma unroll
        for (int r1 = 0; r1 < 3; ++r1)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < 3; ++q1) acc = fma(M0[r1][q1], T1[q1][c], acc);
            lo[c] = fmin(lo[c], acc);
            hi[c] = fmax(hi[c], acc);
          }
      }
    }
  } else
#endif
  {
    double B[NP * 3];
    element_bezier<R>(T.Bc, t0, h, B);
    for (int m = 0; m < NP; ++m)
      for (int c = 0; c < 3; ++c) {
        lo[c] = fmin(lo[c], B[3 * m + c]);
        hi[c] = fmax(hi[c], B[3 * m + c]);
      }
  }
  Rect16 rc{0, -1, 0, -1};
  bool v = project_rect(cc, lo, hi, rc);
  flag[e] = v ? 1 : 0;
  rect[e] = rc;
}


__global__ void k_compact(const int32_t* __restrict__ flag, const Rect16* __restrict__ rect,
                          const int64_t* __restrict__ pos, int64_t n, int32_t* __restrict__ vis,
                          Rect16* __restrict__ vis_rect) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n || !flag[e]) return;
  int64_t p = pos[e];
  vis[p] = (int32_t)e;
  vis_rect[p] = rect[e];
}

// ---------------------------------------------------------------------------
// a3: pair generation.  Per visible leaf: rect area -> ceil(area/32) warp
// chunks; exclusive scan -> chunk offsets; expand -> chunk -> leaf map.
// ---------------------------------------------------------------------------
__global__ void k_chunk_count(const Rect16* __restrict__ vis_rect, const int64_t* __restrict__ nvis_p,
                              int64_t* __restrict__ cnt, int64_t* __restrict__ counters) {
  int64_t nvis = *nvis_p;
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t area = 0;
  if (v < nvis) {
    Rect16 r = vis_rect[v];
    area = (int64_t)(r.i1 - r.i0 + 1) * (int64_t)(r.j1 - r.j0 + 1);
    cnt[v] = (area + RC_CHUNK - 1) / RC_CHUNK;
  }
  // block-reduce the candidate count
  unsigned long long s = (unsigned long long)area;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  __shared__ unsigned long long ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0 && s) atomicAdd((unsigned long long*)&counters[CNT_CANDIDATES], s);
  }
}

__global__ void k_expand(const int64_t* __restrict__ off, const int64_t* __restrict__ nvis_p,
                         int32_t* __restrict__ chunk_elem) {
  int64_t nvis = *nvis_p;
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvis) return;
  for (int64_t c = off[v]; c < off[v + 1]; ++c) chunk_elem[c] = (int32_t)v;
}

// Fold units of the curved segment kernel (row a6): the visible leaves of
// every node of the fold level (contiguous in the visible list, SFC order)
// are cut into <= RC_UNIT_LEAVES-leaf windows, and each window into
// <= RC_UNIT_CHUNKS-chunk pieces of about equal size.  Without folding
// (leaf_node == nullptr) the windows are 64 consecutive visible leaves.
struct NodeRun {
  int64_t v0, v1;   // visible range of the node
};

__device__ __forceinline__ NodeRun node_run(const int32_t* __restrict__ vis, const int32_t* __restrict__ leaf_node,
                                            int64_t nvis, int64_t v, bool& start) {
  if (!leaf_node) {
    start = (v % RC_UNIT_LEAVES) == 0;
    return NodeRun{v, min(nvis, v + RC_UNIT_LEAVES)};
  }
  const int32_t nd = leaf_node[vis[v]];
  start = v == 0 || leaf_node[vis[v - 1]] != nd;
  if (!start) return NodeRun{v, v};
  int64_t lo = v, hi = nvis;   // leaf_node[vis[lo]] == nd, hi is past the run
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (leaf_node[vis[mid]] == nd) lo = mid;
    else hi = mid;
  }
  return NodeRun{v, hi};
}

__global__ void k_unit_count(const int32_t* __restrict__ vis, const int64_t* __restrict__ nvis_p,
                             const int32_t* __restrict__ leaf_node, const int64_t* __restrict__ chunk_off,
                             int32_t* __restrict__ ucnt, int32_t* __restrict__ uend) {
  const int64_t nvis = *nvis_p;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvis) return;
  bool start;
  const NodeRun r = node_run(vis, leaf_node, nvis, v, start);
  if (!start) {
    ucnt[v] = 0;
    return;
  }
  uend[v] = (int32_t)r.v1;
  const int64_t nl = r.v1 - r.v0, nw = (nl + RC_UNIT_LEAVES - 1) / RC_UNIT_LEAVES;
  int64_t nu = 0;
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t a = r.v0 + nl * w / nw, b = r.v0 + nl * (w + 1) / nw;
    nu += (chunk_off[b] - chunk_off[a] + RC_UNIT_CHUNKS - 1) / RC_UNIT_CHUNKS;
  }
  ucnt[v] = (int32_t)nu;
}

__global__ void k_unit_emit(const int32_t* __restrict__ vis, const int64_t* __restrict__ nvis_p,
                            const int32_t* __restrict__ leaf_node, const int32_t* __restrict__ node_first,
                            const int64_t* __restrict__ chunk_off, const int32_t* __restrict__ ucnt,
                            const int64_t* __restrict__ uoff, const int32_t* __restrict__ uend, uint32_t key_base,
                            Unit* __restrict__ units) {
  const int64_t nvis = *nvis_p;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvis) return;
  if (ucnt[v] == 0) return;
  const int64_t v1 = uend[v], nl = v1 - v, nw = (nl + RC_UNIT_LEAVES - 1) / RC_UNIT_LEAVES;
  const uint32_t key = leaf_node ? key_base + (uint32_t)node_first[leaf_node[vis[v]]] : 0u;
  int64_t out = uoff[v];
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t a = v + nl * w / nw, b = v + nl * (w + 1) / nw;
    const int64_t c0 = chunk_off[a], nch = chunk_off[b] - c0;
    const int64_t nu = (nch + RC_UNIT_CHUNKS - 1) / RC_UNIT_CHUNKS;
    for (int64_t k = 0; k < nu; ++k) {
      const int64_t ca = c0 + nch * k / nu, cb = c0 + nch * (k + 1) / nu;
      units[out++] = Unit{ca, (int32_t)(cb - ca), key, (int32_t)a, (int32_t)(b - a), 0};
    }
  }
}

// ---------------------------------------------------------------------------
// a4 + a5 (affine trees): slab test in element reference coordinates and the
// N-point GL rule.  One warp = one 32-pixel chunk of one element; dynamic
// chunk scheduling over a persistent grid.
//
// Precision: the ray is re-based at alpha0 near the element
// centre with a few fp64 operations, P0 = T(alpha0) - C_E; everything after
// that is fp32 on quantities of the element's size.
// ---------------------------------------------------------------------------
template <int P, int N>
__global__ void __launch_bounds__(256) k_cast_affine(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L,
                                                     const int32_t* __restrict__ vis, const Rect16* __restrict__ vrect,
                                                     const int64_t* __restrict__ chunk_off,
                                                     const int32_t* __restrict__ chunk_elem, int64_t nchunks,
                                                     uint32_t key_base, rc_seg* __restrict__ segs, int64_t seg_cap,
                                                     int32_t* __restrict__ hits_pp, int64_t* __restrict__ counters) {
  constexpr int NF = (P + 1) * (P + 1) * (P + 1);
  const unsigned lane = threadIdx.x & 31;
  const float half_w = 0.5f * (cc.W - 1), half_h = 0.5f * (cc.H - 1);
  int local_hits = 0;
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
    const int lvl = L.level[e];
    const double h = ldexp(1.0, -lvl);
    const float hf = (float)h, inv_h = 1.0f / hf;
    float f[NF];
#pragma unroll
    for (int q = 0; q < NF; ++q) f[q] = __ldg(&L.field[(int64_t)e * NF + q]);

    // tree-reference ray of pixel (i,j) in fp64, re-based near the element centre
    const double di = (double)i - 0.5 * (cc.W - 1), dj = (double)j - 0.5 * (cc.H - 1);
    double TR[3], D[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      TR[k] = fma(dj, T.TRu[k], fma(di, T.TRt[k], T.TR0[k]));
      double TO = fma(dj, T.TOu[k], fma(di, T.TOt[k], T.TO0[k]));
      double C = ldexp((double)L.anchor[3 * (int64_t)e + k], -RC_MAXLEVEL) + 0.5 * h;
      D[k] = C - TO;
    }
    const float trf[3] = {(float)TR[0], (float)TR[1], (float)TR[2]};
    const float alpha0 = ((float)D[0] * trf[0] + (float)D[1] * trf[1] + (float)D[2] * trf[2]) /
                         (trf[0] * trf[0] + trf[1] * trf[1] + trf[2] * trf[2]);
    float P0[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) P0[k] = (float)fma((double)alpha0, TR[k], -D[k]);

    // slab: xi_k(beta) = 1/2 + (P0_k + beta TR_k)/h in [0,1]
    float b_in = (float)(cc.amin - (double)alpha0), b_out = (float)(cc.amax - (double)alpha0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float inv = 1.0f / trf[k];   // +-inf for axis-parallel rays: handled by IEEE min/max
      float t0 = (-0.5f * hf - P0[k]) * inv, t1 = (0.5f * hf - P0[k]) * inv;
      if (trf[k] == 0.0f) {
        t0 = (fabsf(P0[k]) <= 0.5f * hf) ? -INFINITY : INFINITY;
        t1 = (fabsf(P0[k]) <= 0.5f * hf) ? INFINITY : -INFINITY;
      }
      b_in = fmaxf(b_in, fminf(t0, t1));
      b_out = fminf(b_out, fmaxf(t0, t1));
    }
    const bool hit = active && (b_out > b_in);

    float a = 1.0f, b[3] = {0.0f, 0.0f, 0.0f};
    if (hit) {
      // physical length: |R_world(i,j)|
      float rw0 = (float)fma(dj, cc.Ru[0], fma(di, cc.Rt[0], cc.R0[0]));
      float rw1 = (float)fma(dj, cc.Ru[1], fma(di, cc.Rt[1], cc.R0[1]));
      float rw2 = (float)fma(dj, cc.Ru[2], fma(di, cc.Rt[2], cc.R0[2]));
      const float rn = sqrtf(rw0 * rw0 + rw1 * rw1 + rw2 * rw2);
      const float db = b_out - b_in;
      const float Lseg = db * rn;
      float xin[3], dx[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        xin[k] = 0.5f + (P0[k] + b_in * trf[k]) * inv_h;
        dx[k] = db * trf[k] * inv_h;
      }
      float ft[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        float x1 = fmaf(cc.u[q], dx[0], xin[0]);
        float x2 = fmaf(cc.u[q], dx[1], xin[1]);
        float x3 = fmaf(cc.u[q], dx[2], xin[2]);
        ft[q] = field_at<P>(f, x1, x2, x3) * cc.inv_F;
      }
      gl_rule<N>(cc, ft, Lseg, a, b);
    }
    int64_t slot = warp_append(&counters[CNT_SEGS], hit ? 1 : 0);
    if (hit) {
      ++local_hits;
      uint32_t pix = (uint32_t)(j * cc.W + i);
      if (slot < seg_cap) {
        store_seg(segs + slot, pix, alpha0 + b_in, alpha0 + b_out, a, b, key_base + (uint32_t)e);
      } else {
        atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
      }
      atomicAdd(&hits_pp[pix], 1);
    }
  }
  // hit-pair count (one segment per pair for convex affine elements)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) local_hits += __shfl_down_sync(0xffffffffu, local_hits, off);
  if (lane == 0 && local_hits) atomicAdd((unsigned long long*)&counters[CNT_HITPAIRS], (unsigned long long)local_hits);
}

// ---------------------------------------------------------------------------
// a8: pack records by tile-owner rank (owner = (tx+ty) mod P).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int owner_of(uint32_t pix, int W, int tw, int th, int tiles_x, int nranks) {
  int i = pix % W, j = pix / W;
  return ((i / tw) + (j / th)) % nranks;
}

__global__ void k_pack_count(const rc_seg* __restrict__ segs, const int64_t* __restrict__ nseg_p, int W, int tw,
                             int th, int tiles_x, int nranks, int64_t* __restrict__ counts) {
  __shared__ unsigned long long c[64];
  if (threadIdx.x < 64) c[threadIdx.x] = 0;
  __syncthreads();
  int64_t n = *nseg_p;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&c[owner_of(segs[s].pixel, W, tw, th, tiles_x, nranks)], 1ull);
  __syncthreads();
  if (threadIdx.x < nranks && c[threadIdx.x]) atomicAdd((unsigned long long*)&counts[threadIdx.x], c[threadIdx.x]);
}

__global__ void k_pack_scatter(const rc_seg* __restrict__ segs, const int64_t* __restrict__ nseg_p, int W, int tw,
                               int th, int tiles_x, int nranks, const int64_t* __restrict__ dest_off,
                               int64_t* __restrict__ cursor, rc_seg* __restrict__ out) {
  __shared__ unsigned long long c[64], base[64];
  int64_t n = *nseg_p;
  int64_t per = ((n + gridDim.x - 1) / gridDim.x + 255) / 256 * 256;
  int64_t lo = (int64_t)blockIdx.x * per, hi = min(n, lo + per);
  if (threadIdx.x < 64) c[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t s = lo + threadIdx.x; s < hi; s += blockDim.x)
    atomicAdd(&c[owner_of(segs[s].pixel, W, tw, th, tiles_x, nranks)], 1ull);
  __syncthreads();
  if (threadIdx.x < nranks) {
    base[threadIdx.x] = c[threadIdx.x] ? atomicAdd((unsigned long long*)&cursor[threadIdx.x], c[threadIdx.x]) : 0;
    c[threadIdx.x] = 0;
  }
  __syncthreads();
  for (int64_t s = lo + threadIdx.x; s < hi; s += blockDim.x) {
    rc_seg rec = segs[s];
    int d = owner_of(rec.pixel, W, tw, th, tiles_x, nranks);
    unsigned long long k = atomicAdd(&c[d], 1ull);
    out[dest_off[d] + base[d] + k] = rec;
  }
}

// ---------------------------------------------------------------------------
// a9: composite.  Bucket records by pixel (histogram, scan, scatter), then one
// warp per pixel: order by (alpha_near, key) with a bitonic sort in shared
// memory, check for overlaps, fold nearest-first with Eq. aggregate in fp64
// (a warp-parallel ordered reduction: the group is associative,
// PAPER.md:395-427), overlaps resolved sequentially by Eq. segsplit /
// Eq. segaverage.
// ---------------------------------------------------------------------------
__global__ void k_hist(const rc_seg* __restrict__ segs, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[segs[s].pixel], 1);
}

// bucket by pixel as a permutation (record indices, 4 bytes each) instead of
// a sorted copy of the 32-byte records
__global__ void k_scatter(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ off,
                          int32_t* __restrict__ cursor, uint32_t* __restrict__ out) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pix = segs[s].pixel;
    int k = atomicAdd(&cursor[pix], 1);
    out[off[pix] + k] = (uint32_t)s;
  }
}

// pixel-bucketed copy of the records (the composite then reads each pixel's
// records contiguously instead of gathering them through a permutation)
#ifndef SCATTER_ILP
#define SCATTER_ILP 1   // records in flight per thread in k_scatter_rec (A/B: 4 -> 17.9 ms vs 1 -> 16.0 ms bucketing, rejected)
#endif
__global__ void k_scatter_rec(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ off,
                              int32_t* __restrict__ cursor, rc_seg* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#if SCATTER_ILP > 1
  for (; s + (SCATTER_ILP - 1) * stride < n; s += SCATTER_ILP * stride) {
    float4 lo[SCATTER_ILP], hi[SCATTER_ILP];
#pragma unroll
    for (int u = 0; u < SCATTER_ILP; ++u) {
      const float4* src = reinterpret_cast<const float4*>(segs + s + u * stride);
      lo[u] = __ldcs(src);
      hi[u] = __ldcs(src + 1);
    }
    int64_t dst[SCATTER_ILP];
#pragma unroll
    for (int u = 0; u < SCATTER_ILP; ++u) {
      const uint32_t pix = __float_as_uint(lo[u].x);
      dst[u] = off[pix] + atomicAdd(&cursor[pix], 1);
    }
#pragma unroll
    for (int u = 0; u < SCATTER_ILP; ++u) {
      float4* d = reinterpret_cast<float4*>(out + dst[u]);
      d[0] = lo[u];
      d[1] = hi[u];
    }
  }
#endif
  for (; s < n; s += stride) {
    const float4* src = reinterpret_cast<const float4*>(segs + s);
    const float4 lo = __ldcs(src), hi = __ldcs(src + 1);
    const uint32_t pix = __float_as_uint(lo.x);
    const int k = atomicAdd(&cursor[pix], 1);
    float4* dst = reinterpret_cast<float4*>(out + off[pix] + k);
    dst[0] = lo;
    dst[1] = hi;
  }
}

struct Acc {
  double A, B0, B1, B2;
};
__device__ __forceinline__ void acc_push(Acc& acc, double a, double b0, double b1, double b2) {
  // acc (nearer) (+) seg (farther): (A a, B + A b)
  acc.B0 = fma(acc.A, b0, acc.B0);
  acc.B1 = fma(acc.A, b1, acc.B1);
  acc.B2 = fma(acc.A, b2, acc.B2);
  acc.A *= a;
}

__device__ __forceinline__ uint64_t sort_key(const rc_seg& s) {
  uint32_t u = __float_as_uint(s.alpha_near);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | s.key;
}

struct Piece {
  double an, af, a, b0, b1, b2;
};
__device__ __forceinline__ Piece piece_of(const rc_seg& s) {
  return Piece{s.alpha_near, s.alpha_far, s.a, s.b[0], s.b[1], s.b[2]};
}
// Eq. segsplit at alpha = at: returns near piece, far piece in *farp
__device__ Piece split_piece(const Piece& s, double at, Piece* farp) {
  double d = s.af - s.an, d1 = at - s.an, d2 = s.af - at;
  Piece n1 = s, f1 = s;
  n1.af = at;
  f1.an = at;
  if (s.a == 1.0 || d <= 0.0) {
    double r1 = d > 0 ? d1 / d : 0.5, r2 = d > 0 ? d2 / d : 0.5;
    n1.b0 = s.b0 * r1; n1.b1 = s.b1 * r1; n1.b2 = s.b2 * r1;
    f1.b0 = s.b0 * r2; f1.b1 = s.b1 * r2; f1.b2 = s.b2 * r2;
  } else {
    double la = log(s.a);
    double a1 = exp(la * d1 / d), a2 = exp(la * d2 / d);
    double q1 = (1.0 - a1) / (1.0 - s.a), q2 = (1.0 - a2) / (1.0 - s.a);
    n1.a = a1; f1.a = a2;
    n1.b0 = s.b0 * q1; n1.b1 = s.b1 * q1; n1.b2 = s.b2 * q1;
    f1.b0 = s.b0 * q2; f1.b1 = s.b1 * q2; f1.b2 = s.b2 * q2;
  }
  *farp = f1;
  return n1;
}
__device__ __forceinline__ Piece avg_piece(const Piece& x, const Piece& y) {   // Eq. segaverage
  return Piece{x.an, x.af, sqrt(x.a * y.a), 0.5 * (x.b0 + y.b0), 0.5 * (x.b1 + y.b1), 0.5 * (x.b2 + y.b2)};
}

// Sequential sweep with overlap resolution (single lane).
struct Sweep {
  Acc acc;
  Piece cur;
  bool have = false;
  double tau;
  __device__ void emit(const Piece& p) { acc_push(acc, p.a, p.b0, p.b1, p.b2); }
  __device__ void push(Piece nx) {
    if (!have) { cur = nx; have = true; return; }
    double tol = tau * fmax(1.0, fabs(nx.an));
    if (nx.an >= cur.af - tol) { emit(cur); cur = nx; return; }
    Piece B;
    if (nx.an > cur.an) { Piece A = split_piece(cur, nx.an, &B); emit(A); }
    else B = cur;
    if (nx.af < B.af) {
      Piece B2;
      Piece B1 = split_piece(B, nx.af, &B2);
      emit(avg_piece(B1, nx));
      cur = B2;
    } else {
      Piece C2;
      Piece C1 = (nx.af > B.af) ? split_piece(nx, B.af, &C2) : nx;
      if (!(nx.af > B.af)) { C2 = nx; C2.an = C2.af; C2.a = 1.0; C2.b0 = C2.b1 = C2.b2 = 0.0; }
      emit(avg_piece(B, C1));
      cur = C2;
    }
  }
  __device__ void finish() { if (have) emit(cur); have = false; }
};

constexpr int FOLD_WARPS = 4;
constexpr int FOLD_CAP = 2048;   // records per pixel sorted in shared memory

// Warp bitonic sort of 32 E (key, id) pairs held in registers in the blocked
// layout i = lane E + e, ascending.  Stage loops are not unrolled (code size:
// the per-pixel kernels were instruction-cache bound); only the element loops
// and the in-register distances (j < E) are static.
#ifndef FOLD_E4
#define FOLD_E4 1   // 1: a 128-record register bucket in k_fold / k_coarsen (C4's pixels hold ~115 records)
#endif
template <int E>
__device__ __forceinline__ void warp_sort_blocked(uint64_t (&key)[E], uint32_t (&id)[E]) {
  const unsigned lane = threadIdx.x & 31;
  constexpr int NN = 32 * E;
#pragma unroll 1
  for (int k = 2; k <= NN; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j >= E; j >>= 1) {   // partners in other lanes
      const int lj = j / E;
      const bool lower = (lane & lj) == 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lj);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, id[e], lj);
        const bool up = ((((int)lane * E + e) & k) == 0);
        const bool take = (lower == up) ? (ok < key[e]) : (ok > key[e]);
        if (take) {
          key[e] = ok;
          id[e] = oi;
        }
      }
    }
#pragma unroll
    for (int j = E >> 1; j > 0; j >>= 1) {     // partners in the same lane
      if (j < k) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e ^ j;
          if (p > e) {
            const bool up = ((((int)lane * E + e) & k) == 0);
            if ((key[e] > key[p]) == up) {
              const uint64_t tk = key[e]; key[e] = key[p]; key[p] = tk;
              const uint32_t ti = id[e]; id[e] = id[p]; id[p] = ti;
            }
          }
        }
      }
    }
  }
}


// Aggregation fast path (n <= 32 E): register sort, then per sorted record
// its index, alpha_near, alpha_far and target-level node cached in shared
// memory, so that run detection needs no dependent global loads.
struct RunCache {
  uint32_t* rid;
  float* an;
  float* af;
  int32_t* anc;
};

template <int E>
__device__ __forceinline__ void sort_pixel_cache(const rc_seg* __restrict__ recs, const uint32_t* __restrict__ S,
                                                 int n, const int32_t* __restrict__ leaf_node, uint32_t key_base,
                                                 RunCache C) {
  const unsigned lane = threadIdx.x & 31;
  constexpr int NN = 32 * E;
  uint64_t key[E];
  uint32_t id[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = (int)lane * E + e;
    id[e] = i < n ? S[i] : 0u;
    key[e] = i < n ? sort_key(recs[id[e]]) : ~0ull;
  }
  warp_sort_blocked<E>(key, id);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = (int)lane * E + e;
    if (i < n) {
      const rc_seg& r = recs[id[e]];
      C.rid[i] = id[e];
      C.an[i] = r.alpha_near;
      C.af[i] = r.alpha_far;
      C.anc[i] = leaf_node[r.key - key_base];
    }
  }
  __syncwarp();
}

// Common case of the per-pixel fold: up to 32 E records sorted by
// (alpha_near, key) in registers (warp bitonic network over the blocked
// layout i = lane E + e: in-register exchanges for distances < E, shuffles
// beyond), then each lane folds its E consecutive records and the lanes are
// combined by an ordered tree reduction (Eq. aggregate is associative,
// PAPER.md:395-427).  Returns false when consecutive records overlap beyond
// tau (the caller then cuts and averages in the sequential sweep).
template <int E>
__device__ __forceinline__ bool fold_pixel_reg(const rc_seg* __restrict__ recs, const uint32_t* __restrict__ S,
                                               int64_t base, int n, float tau, Acc& acc) {
  const unsigned lane = threadIdx.x & 31;
  constexpr int NN = 32 * E;
  uint64_t key[E];
  uint32_t id[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = (int)lane * E + e;
    id[e] = i < n ? (S ? S[i] : (uint32_t)(base + i)) : 0xffffffffu;   // S == nullptr: pixel-sorted copy
    key[e] = i < n ? sort_key(recs[id[e]]) : ~0ull;
  }
  warp_sort_blocked<E>(key, id);
  // overlap check between consecutive records, then the lane's ordered fold
  float prev_af = __shfl_up_sync(0xffffffffu, id[E - 1] != 0xffffffffu ? recs[id[E - 1]].alpha_far : -3.4e38f, 1);
  if (lane == 0) prev_af = -3.4e38f;
  bool ovl = false;
  Acc a{1.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (id[e] == 0xffffffffu) continue;
    const rc_seg& r = recs[id[e]];
    ovl |= (prev_af - r.alpha_near) > tau * fmaxf(1.0f, fabsf(r.alpha_near));
    prev_af = r.alpha_far;
    acc_push(a, r.a, r.b[0], r.b[1], r.b[2]);
  }
  if (__any_sync(0xffffffffu, ovl)) return false;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double A = __shfl_down_sync(0xffffffffu, a.A, o);
    const double B0 = __shfl_down_sync(0xffffffffu, a.B0, o);
    const double B1 = __shfl_down_sync(0xffffffffu, a.B1, o);
    const double B2 = __shfl_down_sync(0xffffffffu, a.B2, o);
    if ((lane & (2 * o - 1)) == 0) acc_push(a, A, B0, B1, B2);
  }
  acc = a;
  return true;
}

#ifndef FOLD_PACKED
#define FOLD_PACKED 0   // 1: sort one 64-bit word per record (alpha, low key bits, bucket position); A/B 25.4 -> 29.8 ms, rejected
#endif
// Keys only: the warp bitonic network of warp_sort_blocked without a payload.
template <int E>
__device__ __forceinline__ void warp_sort_keys(uint64_t (&key)[E]) {
  const unsigned lane = threadIdx.x & 31;
  constexpr int NN = 32 * E;
#pragma unroll 1
  for (int k = 2; k <= NN; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j >= E; j >>= 1) {
      const int lj = j / E;
      const bool lower = (lane & lj) == 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lj);
        const bool up = ((((int)lane * E + e) & k) == 0);
        const bool take = (lower == up) ? (ok < key[e]) : (ok > key[e]);
        key[e] = take ? ok : key[e];
      }
    }
#pragma unroll
    for (int j = E >> 1; j > 0; j >>= 1) {
      if (j < k) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e ^ j;
          if (p > e) {
            const bool up = ((((int)lane * E + e) & k) == 0);
            const uint64_t lo = key[e] < key[p] ? key[e] : key[p], hi = key[e] < key[p] ? key[p] : key[e];
            key[e] = up ? lo : hi;
            key[p] = up ? hi : lo;
          }
        }
      }
    }
  }
}

// fold_pixel_reg with the record's bucket position packed into the sort key
// (9 bits) below the low 23 bits of its node key: one word per exchange
// instead of key + index.  The order is (alpha_near, key) as in sort_key
// except between records of one pixel whose alpha_near are equal AND whose
// node keys agree in the low 23 bits (then bucket position).
template <int E>
__device__ __forceinline__ bool fold_pixel_packed(const rc_seg* __restrict__ recs, const uint32_t* __restrict__ S,
                                                  int64_t base, int n, float tau, Acc& acc) {
  const unsigned lane = threadIdx.x & 31;
  uint64_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = (int)lane * E + e;
    if (i < n) {
      const rc_seg& r = recs[S ? S[i] : (uint32_t)(base + i)];
      uint32_t u = __float_as_uint(r.alpha_near);
      u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
      key[e] = ((uint64_t)u << 32) | ((uint64_t)(r.key & 0x7FFFFFu) << 9) | (uint64_t)i;
    } else {
      key[e] = ~0ull;
    }
  }
  warp_sort_keys<E>(key);
  auto rid = [&](int e) -> uint32_t {
    const int pos = (int)(key[e] & 511u);
    return S ? S[pos] : (uint32_t)(base + pos);
  };
  const int last = (int)lane * E + E - 1;
  float prev_af = __shfl_up_sync(0xffffffffu, last < n ? recs[rid(E - 1)].alpha_far : -3.4e38f, 1);
  if (lane == 0) prev_af = -3.4e38f;
  bool ovl = false;
  Acc a{1.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((int)lane * E + e >= n) continue;
    const rc_seg& r = recs[rid(e)];
    ovl |= (prev_af - r.alpha_near) > tau * fmaxf(1.0f, fabsf(r.alpha_near));
    prev_af = r.alpha_far;
    acc_push(a, r.a, r.b[0], r.b[1], r.b[2]);
  }
  if (__any_sync(0xffffffffu, ovl)) return false;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double A = __shfl_down_sync(0xffffffffu, a.A, o);
    const double B0 = __shfl_down_sync(0xffffffffu, a.B0, o);
    const double B1 = __shfl_down_sync(0xffffffffu, a.B1, o);
    const double B2 = __shfl_down_sync(0xffffffffu, a.B2, o);
    if ((lane & (2 * o - 1)) == 0) acc_push(a, A, B0, B1, B2);
  }
  acc = a;
  return true;
}
#if FOLD_PACKED
#define FOLD_PIXEL fold_pixel_packed
#else
#define FOLD_PIXEL fold_pixel_reg
#endif

// Two passes: CAP = 512 over every pixel (registers, 16 warps per SM); the
// few pixels with more records are deferred to a list that the CAP = 2048
// pass (shared-memory bitonic, else selection order) works through.
#ifndef FOLD_MINB
#define FOLD_MINB 8   // resident k_fold<512> CTAs per SM the register budget is sized for (A/B: 4 -> 8 = 31.1 -> 25.4 ms at C4)
#endif
template <int CAP, bool FROM_LIST>
__global__ void __launch_bounds__(FOLD_WARPS * 32, CAP <= 512 ? FOLD_MINB : 1) k_fold(
    const rc_seg* __restrict__ recs, const uint32_t* __restrict__ perm, const int64_t* __restrict__ off, int W,
    int H, int tw, int th, const int32_t* __restrict__ my_tiles, int tiles_x, int64_t npix_out, float bg0, float bg1,
    float bg2, float tau, float* __restrict__ rgba, int32_t* __restrict__ defer, int64_t* __restrict__ counters) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * CAP;
  uint16_t* idxs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)FOLD_WARPS * CAP) +
                   (size_t)warp * CAP;
  const int64_t tile_px = (int64_t)tw * th;
  const int64_t nq = FROM_LIST ? counters[CNT_DEFER] : npix_out;
  for (int64_t qi = (int64_t)blockIdx.x * FOLD_WARPS + warp; qi < nq; qi += (int64_t)gridDim.x * FOLD_WARPS) {
    const int64_t q = FROM_LIST ? (int64_t)defer[qi] : qi;
    int t = (int)(q / tile_px);
    int rem = (int)(q - (int64_t)t * tile_px);
    int tile = my_tiles[t];
    int tx = tile % tiles_x, ty = tile / tiles_x;
    int i = tx * tw + rem % tw, j = ty * th + rem / tw;
    int64_t pix = (int64_t)j * W + i;
    int64_t base = off[pix];
    int n = (int)(off[pix + 1] - base);
    const uint32_t* S = perm ? perm + base : nullptr;   // S[k] = index of the pixel's k-th record
#define RI(k) (S ? S[(k)] : (uint32_t)(base + (k)))
    if (!FROM_LIST && n > CAP && defer) {
      if (lane == 0) defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)q;
      continue;
    }
    Acc acc{1.0, 0.0, 0.0, 0.0};
    bool done = false;
    if (n <= 64) done = FOLD_PIXEL<2>(recs, S, base, n, tau, acc);
#if FOLD_E4
    else if (n <= 128) done = FOLD_PIXEL<4>(recs, S, base, n, tau, acc);
#endif
    else if (n <= 256) done = FOLD_PIXEL<8>(recs, S, base, n, tau, acc);
    else if (n <= 512) done = FOLD_PIXEL<16>(recs, S, base, n, tau, acc);
    if (done) {
      // lane 0 holds the pixel's fold
    } else if (n <= CAP) {
      int m = 1;
      while (m < n) m <<= 1;
      for (int k = lane; k < m; k += 32) {
        keys[k] = k < n ? sort_key(recs[RI(k)]) : ~0ull;
        idxs[k] = (uint16_t)k;
      }
      __syncwarp();
      // bitonic sort of (key, idx), ascending
      for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int k = lane; k < m; k += 32) {
            int p = k ^ stride;
            if (p > k) {
              bool up = (k & size) == 0;
              uint64_t ka = keys[k], kb = keys[p];
              if ((ka > kb) == up) {
                keys[k] = kb; keys[p] = ka;
                uint16_t t2 = idxs[k]; idxs[k] = idxs[p]; idxs[p] = t2;
              }
            }
          }
          __syncwarp();
        }
      }
      // overlap detection between consecutive records
      bool ovl = false;
      for (int k = lane; k + 1 < n; k += 32) {
        const rc_seg& x = recs[RI(idxs[k])];
        const rc_seg& y = recs[RI(idxs[k + 1])];
        float tol = tau * fmaxf(1.0f, fabsf(y.alpha_near));
        ovl |= (x.alpha_far - y.alpha_near) > tol;
      }
      if (__any_sync(0xffffffffu, ovl)) {
        if (lane == 0) {
          Sweep sw;
          sw.acc = acc;
          sw.tau = tau;
          for (int k = 0; k < n; ++k) sw.push(piece_of(recs[RI(idxs[k])]));
          sw.finish();
          acc = sw.acc;
        }
      } else {
        // warp-parallel ordered fold: lane l folds the l-th contiguous run
        int per = (n + 31) / 32;
        int lo = min(n, (int)lane * per), hi = min(n, lo + per);
        for (int k = lo; k < hi; ++k) {
          const rc_seg& s = recs[RI(idxs[k])];
          acc_push(acc, s.a, s.b[0], s.b[1], s.b[2]);
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          double A = __shfl_down_sync(0xffffffffu, acc.A, o);
          double B0 = __shfl_down_sync(0xffffffffu, acc.B0, o);
          double B1 = __shfl_down_sync(0xffffffffu, acc.B1, o);
          double B2 = __shfl_down_sync(0xffffffffu, acc.B2, o);
          if ((lane & (2 * o - 1)) == 0) acc_push(acc, A, B0, B1, B2);
        }
      }
      __syncwarp();
    } else if (lane == 0) {
      // rare: more records than the shared-memory sort holds -> selection order
      Sweep sw;
      sw.acc = acc;
      sw.tau = tau;
      uint64_t last = 0;
      bool first = true;
      for (int cnt = 0; cnt < n; ++cnt) {
        uint64_t best = ~0ull;
        int bi = -1;
        for (int k = 0; k < n; ++k) {
          uint64_t kk = sort_key(recs[RI(k)]);
          if ((first || kk > last) && kk < best) { best = kk; bi = k; }
        }
        if (bi < 0) break;
        first = false;
        last = best;
        sw.push(piece_of(recs[RI(bi)]));
      }
      sw.finish();
      acc = sw.acc;
    }
    if (lane == 0) {
      float4 o = make_float4((float)(acc.B0 + acc.A * bg0), (float)(acc.B1 + acc.A * bg1),
                             (float)(acc.B2 + acc.A * bg2), (float)(1.0 - acc.A));
      reinterpret_cast<float4*>(rgba)[q] = o;
    }
  }
#undef RI
}


// ---------------------------------------------------------------------------
// a7: one pass of the aggregation cycles.
// Records are bucketed by pixel (k_hist / k_scatter); one warp per pixel
// orders them by (alpha_near, key) and combines every maximal run of touching
// records (|gap| <= tau max(1, alpha)) that lie in the same node of the target
// level (node_of of the record's key) with Eq. aggregate, nearest first.  The
// result is keyed by the node's first leaf.  Records of one node that do not
// touch stay separate (safe for non-convex curved nodes).
// ---------------------------------------------------------------------------
// Two passes (as k_fold): FROM_LIST = false takes every pixel with <= 512
// records (8 KB of shared memory per warp: 6 resident CTAs per SM instead of
// 2) and defers the others to a list that FROM_LIST = true works through.
constexpr int COARSEN_CACHE = 512;
#ifndef COARSEN_MINB
#define COARSEN_MINB 6
#endif
template <bool FROM_LIST>
__global__ void __launch_bounds__(FOLD_WARPS * 32, FROM_LIST ? 1 : COARSEN_MINB) k_coarsen(
    const rc_seg* __restrict__ recs, const uint32_t* __restrict__ perm, const int64_t* __restrict__ off, int64_t npix,
    const int32_t* __restrict__ node_first, const int32_t* __restrict__ leaf_node, uint32_t key_base, float tau,
    rc_seg* __restrict__ out, int64_t out_cap, int32_t* __restrict__ defer, int64_t* __restrict__ counters) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  constexpr int WCAP = FROM_LIST ? FOLD_CAP : COARSEN_CACHE * 2;   // uint64 words of keys per warp
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * WCAP;
  uint16_t* idxs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)FOLD_WARPS * WCAP) +
                   (size_t)warp * FOLD_CAP;
  const int64_t nq = FROM_LIST ? counters[CNT_DEFER] : npix;
  for (int64_t qi = (int64_t)blockIdx.x * FOLD_WARPS + warp; qi < nq; qi += (int64_t)gridDim.x * FOLD_WARPS) {
    const int64_t pix = FROM_LIST ? (int64_t)defer[qi] : qi;
    const int64_t base = off[pix];
    const int n = (int)(off[pix + 1] - base);
    if (n == 0) continue;
    const uint32_t* S = perm + base;
    if (!FROM_LIST && n > COARSEN_CACHE) {
      if (lane == 0) defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)pix;
      continue;
    }
    if (FROM_LIST && n > FOLD_CAP) {   // rare: pass through, re-keyed by the target node
      for (int k0 = 0; k0 < n; k0 += 32) {
        const int k = k0 + (int)lane;
        const int64_t slot = warp_append(&counters[CNT_AGG_OUT], k < n ? 1 : 0);
        if (k < n) {
          rc_seg r = recs[S[k]];
          r.key = key_base + (uint32_t)node_first[leaf_node[r.key - key_base]];
          if (slot < out_cap) out[slot] = r;
          else atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
        }
      }
      continue;
    }
    if (!FROM_LIST) {
      RunCache C{reinterpret_cast<uint32_t*>(keys), reinterpret_cast<float*>(keys) + 512,
                 reinterpret_cast<float*>(keys) + 1024, reinterpret_cast<int32_t*>(keys) + 1536};
      if (n <= 64) sort_pixel_cache<2>(recs, S, n, leaf_node, key_base, C);
#if FOLD_E4
      else if (n <= 128) sort_pixel_cache<4>(recs, S, n, leaf_node, key_base, C);
#endif
      else if (n <= 256) sort_pixel_cache<8>(recs, S, n, leaf_node, key_base, C);
      else sort_pixel_cache<16>(recs, S, n, leaf_node, key_base, C);
      auto head = [&](int k) -> bool {
        return k == 0 || fabsf(C.an[k] - C.af[k - 1]) > tau * fmaxf(1.0f, fabsf(C.an[k])) || C.anc[k] != C.anc[k - 1];
      };
      for (int k0 = 0; k0 < n; k0 += 32) {
        const int k = k0 + (int)lane;
        const bool h = k < n && head(k);
        const int64_t slot = warp_append(&counters[CNT_AGG_OUT], h ? 1 : 0);
        if (!h) continue;
        double A = 1.0, B0 = 0.0, B1 = 0.0, B2 = 0.0;
        int q = k;
        do {
          const rc_seg* sq = recs + C.rid[q];
          const float a = sq->a;
          const float4 hb = reinterpret_cast<const float4*>(sq)[1];   // b0, b1, b2, key
          B0 = fma(A, (double)hb.x, B0);
          B1 = fma(A, (double)hb.y, B1);
          B2 = fma(A, (double)hb.z, B2);
          A *= (double)a;
          ++q;
        } while (q < n && !head(q));
        if (slot < out_cap) {
          const float bb[3] = {(float)B0, (float)B1, (float)B2};
          store_seg(out + slot, (uint32_t)pix, C.an[k], C.af[q - 1], (float)A, bb,
                    key_base + (uint32_t)node_first[C.anc[k]]);
        } else {
          atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
        }
      }
      __syncwarp();
      continue;
    }
    {
      int m = 1;
      while (m < n) m <<= 1;
      for (int k = lane; k < m; k += 32) {
        keys[k] = k < n ? sort_key(recs[S[k]]) : ~0ull;
        idxs[k] = (uint16_t)k;
      }
      __syncwarp();
      for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int k = lane; k < m; k += 32) {
            const int p = k ^ stride;
            if (p > k) {
              const bool up = (k & size) == 0;
              const uint64_t ka = keys[k], kb = keys[p];
              if ((ka > kb) == up) {
                keys[k] = kb;
                keys[p] = ka;
                const uint16_t t2 = idxs[k];
                idxs[k] = idxs[p];
                idxs[p] = t2;
              }
            }
          }
          __syncwarp();
        }
      }
    }
    auto anc = [&](int k) -> int64_t {
      return (int64_t)leaf_node[recs[S[idxs[k]]].key - key_base];
    };
    auto is_head = [&](int k) -> bool {
      if (k == 0) return true;
      const rc_seg& x = recs[S[idxs[k - 1]]];
      const rc_seg& y = recs[S[idxs[k]]];
      if (fabsf(y.alpha_near - x.alpha_far) > tau * fmaxf(1.0f, fabsf(y.alpha_near))) return true;
      return anc(k) != anc(k - 1);
    };
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + (int)lane;
      const bool h = k < n && is_head(k);
      const int64_t slot = warp_append(&counters[CNT_AGG_OUT], h ? 1 : 0);
      if (!h) continue;
      const rc_seg& s0 = recs[S[idxs[k]]];
      double A = 1.0, B0 = 0.0, B1 = 0.0, B2 = 0.0;
      float af = s0.alpha_far;
      int q = k;
      do {
        const rc_seg& sq = recs[S[idxs[q]]];
        B0 = fma(A, (double)sq.b[0], B0);
        B1 = fma(A, (double)sq.b[1], B1);
        B2 = fma(A, (double)sq.b[2], B2);
        A *= (double)sq.a;
        af = sq.alpha_far;
        ++q;
      } while (q < n && !is_head(q));
      if (slot < out_cap) {
        const float bb[3] = {(float)B0, (float)B1, (float)B2};
        store_seg(out + slot, s0.pixel, s0.alpha_near, af, (float)A, bb,
                  key_base + (uint32_t)node_first[anc(k)]);
      } else {
        atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// host launchers (kernels are launched only from this translation unit)
// ---------------------------------------------------------------------------
static unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_cull(const CamConst& cc, const TreeConst* trees, DevLeafView L, int64_t n, int R, bool affine,
                        int32_t* flag, Rect16* rect, cudaStream_t s) {
  if (affine) k_cull_affine<<<nblk(n, 256), 256, 0, s>>>(cc, trees, L, n, flag, rect);
  else if (R == 2) k_cull_curved<2><<<nblk(n, 128), 128, 0, s>>>(cc, trees, L, n, flag, rect);
  else k_cull_curved<1><<<nblk(n, 128), 128, 0, s>>>(cc, trees, L, n, flag, rect);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_compact(const int32_t* flag, const Rect16* rect, const int64_t* pos, int64_t n, int32_t* vis,
                           Rect16* vis_rect, cudaStream_t s) {
  k_compact<<<nblk(n, 256), 256, 0, s>>>(flag, rect, pos, n, vis, vis_rect);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_chunk_count(const Rect16* vis_rect, const int64_t* nvis_p, int64_t n, int64_t* cnt,
                               int64_t* counters, cudaStream_t s) {
  k_chunk_count<<<nblk(n, 256), 256, 0, s>>>(vis_rect, nvis_p, cnt, counters);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_expand(const int64_t* off, const int64_t* nvis_p, int64_t nvis, int32_t* chunk_elem,
                          cudaStream_t s) {
  k_expand<<<nblk(nvis, 256), 256, 0, s>>>(off, nvis_p, chunk_elem);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_units(const int32_t* vis, const int64_t* nvis_p, int64_t nvis, const int32_t* leaf_node,
                         const int32_t* node_first, const int64_t* chunk_off, int32_t* ucnt, int64_t* uoff,
                         int32_t* uend, int64_t* scan_tmp, uint32_t key_base, Unit* units, bool emit,
                         cudaStream_t s) {
  if (!emit) {
    cudaError_t e = cudaMemsetAsync(ucnt, 0, sizeof(int32_t) * (nvis + 1), s);
    if (e != cudaSuccess) return e;
    if (nvis > 0) {
      k_unit_count<<<nblk(nvis, 256), 256, 0, s>>>(vis, nvis_p, leaf_node, chunk_off, ucnt, uend);
      ++g_launches;
    }
    return scan_exclusive<int32_t>(ucnt, uoff, nvis, scan_tmp, s);
  }
  if (nvis > 0) {
    k_unit_emit<<<nblk(nvis, 256), 256, 0, s>>>(vis, nvis_p, leaf_node, node_first, chunk_off, ucnt, uoff, uend,
                                                key_base, units);
    ++g_launches;
  }
  return cudaGetLastError();
}

template <int P>
static void cast_affine_P(const CamConst& cc, const TreeConst* trees, DevLeafView L, const int32_t* vis,
                          const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem, int64_t nchunks,
                          uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp, int64_t* counters,
                          int grid, cudaStream_t s) {
#define CASE(N)                                                                                                    \
  case N:                                                                                                          \
    k_cast_affine<P, N><<<grid, 256, 0, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base,   \
                                             segs, seg_cap, hits_pp, counters);                                    \
    break;
  switch (cc.N) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) }
#undef CASE
}

cudaError_t launch_cast_affine(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                               int64_t* counters, int grid, cudaStream_t s) {
  if (P == 1) cast_affine_P<1>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base, segs, seg_cap,
                               hits_pp, counters, grid, s);
  else cast_affine_P<2>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, key_base, segs, seg_cap, hits_pp,
                        counters, grid, s);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_pack(const rc_seg* segs, const int64_t* nseg_p, int W, int tw, int th, int tiles_x, int nranks,
                        int64_t* counts, const int64_t* dest_off, int64_t* cursor, rc_seg* out, int grid, bool count,
                        cudaStream_t s) {
  if (count) k_pack_count<<<grid, 256, 0, s>>>(segs, nseg_p, W, tw, th, tiles_x, nranks, counts);
  else k_pack_scatter<<<grid, 256, 0, s>>>(segs, nseg_p, W, tw, th, tiles_x, nranks, dest_off, cursor, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_hist(const rc_seg* segs, int64_t n, int32_t* cnt, int grid, cudaStream_t s) {
  k_hist<<<grid, 256, 0, s>>>(segs, n, cnt);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_scatter(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, uint32_t* out,
                           int grid, cudaStream_t s) {
  k_scatter<<<grid, 256, 0, s>>>(segs, n, off, cursor, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_scatter_rec(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, rc_seg* out,
                               int grid, cudaStream_t s) {
  k_scatter_rec<<<grid, 256, 0, s>>>(segs, n, off, cursor, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_coarsen(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int64_t npix,
                           const int32_t* node_first, const int32_t* leaf_node, uint32_t key_base, float tau, rc_seg* out,
                           int64_t out_cap, int32_t* defer, int64_t* counters, int max_grid, cudaStream_t s) {
  static bool attr = false;
  const size_t smem1 = (size_t)FOLD_WARPS * COARSEN_CACHE * 2 * sizeof(uint64_t);
  const size_t smem2 = (size_t)FOLD_WARPS * FOLD_CAP * (sizeof(uint64_t) + sizeof(uint16_t));
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_coarsen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaError_t e = cudaMemsetAsync(counters + CNT_DEFER, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  int grid = (int)std::min<int64_t>((npix + FOLD_WARPS - 1) / FOLD_WARPS, (int64_t)max_grid);
  k_coarsen<false><<<grid, FOLD_WARPS * 32, smem1, s>>>(recs, perm, off, npix, node_first, leaf_node, key_base, tau,
                                                        out, out_cap, defer, counters);
  k_coarsen<true><<<std::min(grid, 296), FOLD_WARPS * 32, smem2, s>>>(recs, perm, off, npix, node_first, leaf_node,
                                                                      key_base, tau, out, out_cap, defer, counters);
  g_launches += 2;
  return cudaGetLastError();
}

template <int CAP, bool FROM_LIST>
static cudaError_t fold_pass(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int W, int H, int tw,
                             int th, const int32_t* my_tiles, int tiles_x, int64_t npix_out, const float bg[3],
                             float tau, float* rgba, int32_t* defer, int64_t* counters, int grid, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = (size_t)FOLD_WARPS * CAP * (sizeof(uint64_t) + sizeof(uint16_t));
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_fold<CAP, FROM_LIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_fold<CAP, FROM_LIST><<<grid, FOLD_WARPS * 32, smem, s>>>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x,
                                                             npix_out, bg[0], bg[1], bg[2], tau, rgba, defer,
                                                             counters);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_fold(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int W, int H, int tw, int th,
                        const int32_t* my_tiles, int tiles_x, int64_t npix_out, const float bg[3], float tau,
                        float* rgba, int32_t* defer, int64_t* counters, int max_grid, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((npix_out + FOLD_WARPS - 1) / FOLD_WARPS, (int64_t)max_grid);
  cudaError_t e = cudaMemsetAsync(counters + CNT_DEFER, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  e = fold_pass<512, false>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x, npix_out, bg, tau, rgba, defer,
                            counters, grid, s);
  if (e != cudaSuccess) return e;
  // the deferred pixels (n > 512): a fixed grid reading the list length on the device
  return fold_pass<FOLD_CAP, true>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x, npix_out, bg, tau, rgba, defer,
                                   counters, std::min(grid, 296), s);
}

}  // namespace rc
