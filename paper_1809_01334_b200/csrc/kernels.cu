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


template <int R>
__global__ void __launch_bounds__(128) k_cull_curved(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L, int64_t n,
                              int32_t* __restrict__ flag, Rect16* __restrict__ rect) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  constexpr int NP = (R + 1) * (R + 1) * (R + 1);
  const TreeConst& T = trees[L.tree[e]];
  double h = ldexp(1.0, -(int)L.level[e]);
  double t0[3];
  for (int k = 0; k < 3; ++k) t0[k] = ldexp((double)L.anchor[3 * e + k], -RC_MAXLEVEL);
  double lo[3], hi[3];
  element_aabb<R>(T.Bc, t0, h, lo, hi);
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

// Partition weight of every leaf: pixel-centre rectangle area
// (0 when culled) + 1.
__global__ void k_leaf_weights(const int32_t* __restrict__ flag, const Rect16* __restrict__ rect, int64_t n,
                               int64_t* __restrict__ w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const Rect16 r = rect[e];
  w[e] = 1 + (flag[e] ? (int64_t)(r.i1 - r.i0 + 1) * (int64_t)(r.j1 - r.j0 + 1) : 0);
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
template <int P, int N, bool ADAPT>
__global__ void __launch_bounds__(256) k_cast_affine(CamConst cc, const TreeConst* __restrict__ trees, DevLeafView L,
                                                     const int32_t* __restrict__ vis, const Rect16* __restrict__ vrect,
                                                     const int64_t* __restrict__ chunk_off,
                                                     const int32_t* __restrict__ chunk_elem, int64_t nchunks,
                                                     const int64_t* __restrict__ d_nchunks,
                                                     uint32_t key_base, rc_seg* __restrict__ segs, int64_t seg_cap,
                                                     int32_t* __restrict__ hits_pp, int64_t* __restrict__ counters) {
  constexpr int NF = (P + 1) * (P + 1) * (P + 1);
  const unsigned lane = threadIdx.x & 31;
  const float half_w = 0.5f * (cc.W - 1), half_h = 0.5f * (cc.H - 1);
  if (d_nchunks) nchunks = min(nchunks, *d_nchunks);   // device-side count (CUDA-graph frames), nchunks = capacity
  int local_hits = 0, capped = 0;
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
      if constexpr (!ADAPT) {
        float ft[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          float x1 = fmaf(cc.u[q], dx[0], xin[0]);
          float x2 = fmaf(cc.u[q], dx[1], xin[1]);
          float x3 = fmaf(cc.u[q], dx[2], xin[2]);
          ft[q] = field_at<P>(f, x1, x2, x3) * cc.inv_F;
        }
        gl_rule<N>(cc, ft, Lseg, a, b);
      } else {
        // the paper's integrators with Alg. 1 (the medium is affine in the element: xi(u) = xin + u dx)
        struct Med {
          float f[NF], xin[3], dx[3], inv_F;
          const CamConst* cc;
          __device__ MediumSample operator()(float u) const {
            return medium_from_f(*cc, field_at<P>(f, fmaf(u, dx[0], xin[0]), fmaf(u, dx[1], xin[1]),
                                                  fmaf(u, dx[2], xin[2])) * inv_F);
          }
        } med;
#pragma unroll
        for (int q = 0; q < NF; ++q) med.f[q] = f[q];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          med.xin[k] = xin[k];
          med.dx[k] = dx[k];
        }
        med.inv_F = cc.inv_F;
        med.cc = &cc;
        segment_scheme(cc, Lseg, med, a, b, capped);
      }
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
  if (capped) atomicAdd((unsigned long long*)&counters[CNT_DEPTH_CAP], (unsigned long long)capped);
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

// exclusive prefix of the per-owner counts (<= 64 ranks) on the device
__global__ void k_pack_offsets(const int64_t* __restrict__ counts, int nranks, int64_t* __restrict__ dest_off) {
  if (threadIdx.x != 0) return;
  int64_t run = 0;
  for (int r = 0; r < nranks; ++r) {
    dest_off[r] = run;
    run += counts[r];
  }
  dest_off[nranks] = run;
}

// ---------------------------------------------------------------------------
// a9: composite.  Bucket records by pixel (histogram, scan, scatter), then one
// warp per pixel: order by (alpha_near, key) with a bitonic sort in shared
// memory, check for overlaps, fold nearest-first with Eq. aggregate in fp64
// (a warp-parallel ordered reduction: the group is associative,
// PAPER.md:395-427), overlaps resolved sequentially by Eq. segsplit /
// Eq. segaverage.
// ---------------------------------------------------------------------------
__global__ void k_hist(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ d_n,
                       int32_t* __restrict__ cnt) {
  if (d_n) n = min(n, *d_n);   // device-side count (CUDA-graph frames), n = capacity
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[segs[s].pixel], 1);
}

// bucket by pixel as a permutation (record indices, 4 bytes each) instead of
// a sorted copy of the 32-byte records
__global__ void k_scatter(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ d_n,
                          const int64_t* __restrict__ off, int32_t* __restrict__ cursor, uint32_t* __restrict__ out) {
  if (d_n) n = min(n, *d_n);
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pix = segs[s].pixel;
    int k = atomicAdd(&cursor[pix], 1);
    out[off[pix] + k] = (uint32_t)s;
  }
}

// Banded pixel bucketing of the aggregation pass (row a7): a permutation
// grouping the records by pixel, built without scattered 4-byte writes into
// the 4-byte-per-record permutation (each would cost a DRAM read-modify-write
// of its 32-byte sector).  Bands of RC_BAND pixels: (1) band counts with
// warp-aggregated atomics, (2) record indices appended to their band's range
// of a scratch array in warp runs (a warp's records are mostly one band: its
// 32 pixels are one chunk of one leaf's rectangle row), (3) one CTA per band
// counts its pixels in shared memory, writes their offsets and places the
// indices within the band's range (an L2-resident window).
constexpr int BAND_SH = 5;   // 32 pixels per band (the scan in k_band_sort assumes 32)
constexpr int BAND_SMEM = 9216;    // entries cached in shared memory per band (index + local pixel; static smem < 48 KB)

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void k_band_count(const rc_seg* __restrict__ segs, int64_t n, int32_t* __restrict__ bcnt) {
  const unsigned lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const int64_t s = base + lane;
    const int b = s < n ? (int)(__ldcs(&segs[s].pixel) >> BAND_SH) : -1;
    const unsigned m = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && lane == (unsigned)(__ffs(m) - 1)) atomicAdd(&bcnt[b], __popc(m));
  }
}

__global__ void k_band_scatter(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ boff,
                               int32_t* __restrict__ bcur, uint64_t* __restrict__ tmp) {
  const unsigned lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const int64_t s = base + lane;
    const uint32_t pix = s < n ? __ldcs(&segs[s].pixel) : 0u;
    const int b = s < n ? (int)(pix >> BAND_SH) : -1;
    const unsigned m = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(m) - 1;
    int first = 0;
    if (b >= 0 && (int)lane == leader) first = atomicAdd(&bcur[b], __popc(m));
    first = __shfl_sync(0xffffffffu, first, leader);
    if (b >= 0) {
      // index and band-local pixel in one 8-byte entry (full-sector runs; no gather in k_band_sort)
      const int64_t slot = boff[b] + first + __popc(m & lanemask_lt());
      RC_DCHECK(slot < boff[b + 1]);
      tmp[slot] = ((uint64_t)(pix & ((1u << BAND_SH) - 1)) << 32) | (uint64_t)(uint32_t)s;
    }
  }
}

__global__ void __launch_bounds__(512) k_band_sort(const uint64_t* __restrict__ tmp,
                                                   const int64_t* __restrict__ boff, int64_t nbands, int64_t npix,
                                                   uint32_t* __restrict__ perm, int64_t* __restrict__ off) {
  __shared__ int32_t hist[1 << BAND_SH];
  __shared__ uint32_t sidx[BAND_SMEM];
  __shared__ uint8_t spix[BAND_SMEM];
  constexpr int NB = 1 << BAND_SH;
  for (int64_t b = blockIdx.x; b < nbands; b += gridDim.x) {
    const int64_t e0 = boff[b], ne = boff[b + 1] - e0;
    if (threadIdx.x < NB) hist[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < ne; i += blockDim.x) {
      const uint64_t t = tmp[e0 + i];
      const uint32_t sidx_i = (uint32_t)t;
      const int p = (int)(t >> 32);
      if (i < BAND_SMEM) {
        sidx[i] = sidx_i;
        spix[i] = (uint8_t)p;
      }
      atomicAdd(&hist[p], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the NB = 32 counts, one per lane
      const int lane = threadIdx.x;
      const int c0 = hist[lane];
      int incl = c0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      hist[lane] = incl - c0;
      const int64_t p0 = b * NB + lane;
      if (p0 < npix) off[p0] = e0 + incl - c0;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < ne; i += blockDim.x) {
      uint32_t sidx_i;
      int p;
      if (i < BAND_SMEM) {
        sidx_i = sidx[i];
        p = spix[i];
      } else {
        const uint64_t t = tmp[e0 + i];
        sidx_i = (uint32_t)t;
        p = (int)(t >> 32);
      }
      const int pos = atomicAdd(&hist[p], 1);
      RC_DCHECK(p < NB && pos < ne);
      perm[e0 + pos] = sidx_i;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) off[npix] = boff[nbands];
}

// pixel-bucketed copy of the records (the composite then reads each pixel's
// records contiguously instead of gathering them through a permutation)
__global__ void k_scatter_rec(const rc_seg* __restrict__ segs, int64_t n, const int64_t* __restrict__ d_n,
                              const int64_t* __restrict__ off, int32_t* __restrict__ cursor, rc_seg* __restrict__ out) {
  if (d_n) n = min(n, *d_n);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; s < n; s += stride) {
    const float4* src = reinterpret_cast<const float4*>(segs + s);
    const float4 lo = __ldcs(src), hi = __ldcs(src + 1);
    const uint32_t pix = __float_as_uint(lo.x);
    const int k = atomicAdd(&cursor[pix], 1);
    RC_DCHECK(off[pix] + k < off[pix + 1]);
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

// Total order of the records of one pixel, so that every fold is
// deterministic: the sort key (alpha_near, key), then alpha_far,
// a, b (float bits in order-preserving integer form), then the caller's
// index (records equal in every field are interchangeable).
__device__ __forceinline__ uint32_t ord_bits(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ bool rec_tail_less(const rc_seg& x, const rc_seg& y, uint32_t ix, uint32_t iy) {
  const float fx[5] = {x.alpha_far, x.a, x.b[0], x.b[1], x.b[2]};
  const float fy[5] = {y.alpha_far, y.a, y.b[0], y.b[1], y.b[2]};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const uint32_t ox = ord_bits(fx[t]), oy = ord_bits(fy[t]);
    if (ox != oy) return ox < oy;
  }
  return ix < iy;
}

// Overlap clusters, one lane ("cutting the segments into
// pieces to isolate the overlapping section and then averaging"; DESIGN.md
// D14).  at(k) is the k-th record in order.  A cluster is a run of records
// each starting more than tol = tau max(1,|alpha|) before the largest far end
// of the run so far.  Inside a cluster the elementary intervals [x, y] are
// visited left to right (y = the smallest member end point above x); every
// member covering [x, y] contributes its piece in closed form -- Eq. segsplit
// with the length fraction phi = (y - x)/(af - an): A^phi and
// B (1 - A^phi)/(1 - A), or B phi when A = 1 -- and the m pieces are averaged
// as in Eq. segaverage: exp(mean ln A), mean B.  Uncovered intervals are
// empty gaps (identity).
template <class At>
__device__ void fold_clusters(At at, int n, float tau, Acc& acc) {
  int k = 0;
  while (k < n) {
    const rc_seg& s0 = at(k);
    double far = s0.alpha_far;
    int j = k + 1;
    while (j < n) {
      const rc_seg& r = at(j);
      if (!((double)r.alpha_near < far - (double)tau * fmax(1.0, fabs((double)r.alpha_near)))) break;
      far = fmax(far, (double)r.alpha_far);
      ++j;
    }
    if (j == k + 1) {
      acc_push(acc, s0.a, s0.b[0], s0.b[1], s0.b[2]);
      k = j;
      continue;
    }
    double x = s0.alpha_near;   // the cluster's first start (records are in alpha_near order)
    for (;;) {
      double y = INFINITY;
      for (int t = k; t < j; ++t) {
        const rc_seg& r = at(t);
        if (r.alpha_near > x) y = fmin(y, (double)r.alpha_near);
        if (r.alpha_far > x) y = fmin(y, (double)r.alpha_far);
      }
      if (!(y < INFINITY)) break;
      int m = 0;
      bool opaque = false;
      double lnA = 0.0, B0 = 0.0, B1 = 0.0, B2 = 0.0;
      for (int t = k; t < j; ++t) {
        const rc_seg& r = at(t);
        if (!(r.alpha_near <= x && y <= r.alpha_far)) continue;
        const double phi = (y - x) / ((double)r.alpha_far - (double)r.alpha_near);
        const double a = r.a;
        double ap, qb;
        if (a == 1.0) {
          ap = 1.0;
          qb = phi;
        } else if (a <= 0.0) {
          ap = 0.0;
          qb = 1.0;
        } else {
          ap = exp(phi * log(a));
          qb = (1.0 - ap) / (1.0 - a);
        }
        if (ap > 0.0) lnA += log(ap);
        else opaque = true;
        B0 = fma(qb, (double)r.b[0], B0);
        B1 = fma(qb, (double)r.b[1], B1);
        B2 = fma(qb, (double)r.b[2], B2);
        ++m;
      }
      if (m > 0) {
        const double im = 1.0 / m;
        acc_push(acc, opaque ? 0.0 : exp(lnA * im), B0 * im, B1 * im, B2 * im);
      }
      x = y;
    }
    k = j;
  }
}

// Warp fold of one pixel's records in order: lane l takes the l-th
// contiguous range; a running far end (exclusive prefix max across lanes)
// detects overlaps beyond the tolerance.  Without overlaps the lanes fold
// their ranges and an ordered tree reduction combines them (Eq. aggregate is
// associative); with overlaps lane 0 resolves the clusters.
// The result is in lane 0's acc.
template <class At>
__device__ void fold_sorted(At at, int n, float tau, Acc& acc) {
  const unsigned lane = threadIdx.x & 31;
  const int per = (n + 31) / 32;
  const int lo = min(n, (int)lane * per), hi = min(n, lo + per);
  float lmax = -3.4e38f;
  for (int k = lo; k < hi; ++k) lmax = fmaxf(lmax, at(k).alpha_far);
  float run = -3.4e38f;   // exclusive prefix max of the lanes' far ends
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, lmax, o);
    if ((int)lane >= o) lmax = fmaxf(lmax, y);
  }
  run = __shfl_up_sync(0xffffffffu, lmax, 1);
  if (lane == 0) run = -3.4e38f;
  bool ovl = false;
  Acc a{1.0, 0.0, 0.0, 0.0};
  for (int k = lo; k < hi; ++k) {
    const rc_seg& r = at(k);
    ovl |= (run - r.alpha_near) > tau * fmaxf(1.0f, fabsf(r.alpha_near));
    run = fmaxf(run, r.alpha_far);
    acc_push(a, r.a, r.b[0], r.b[1], r.b[2]);
  }
  if (__any_sync(0xffffffffu, ovl)) {
    if (lane == 0) fold_clusters(at, n, tau, acc);
    __syncwarp();
    return;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double A = __shfl_down_sync(0xffffffffu, a.A, o);
    const double B0 = __shfl_down_sync(0xffffffffu, a.B0, o);
    const double B1 = __shfl_down_sync(0xffffffffu, a.B1, o);
    const double B2 = __shfl_down_sync(0xffffffffu, a.B2, o);
    if ((lane & (2 * o - 1)) == 0) acc_push(a, A, B0, B1, B2);
  }
  acc = a;
}

// Warp bitonic sort of m (power of two) (key, idx) pairs in shared memory
// under the total order above; entries with idx >= n are padding (+inf).
template <class Rec>
__device__ void warp_sort_smem(uint64_t* keys, uint16_t* idxs, int n, int m, Rec rec) {
  const unsigned lane = threadIdx.x & 31;
  auto less = [&](uint64_t ka, uint16_t ia, uint64_t kb, uint16_t ib) -> bool {
    if (ia >= n) return false;
    if (ib >= n) return true;
    if (ka != kb) return ka < kb;
    return rec_tail_less(rec(ia), rec(ib), ia, ib);
  };
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = lane; k < m; k += 32) {
        const int p = k ^ stride;
        if (p > k) {
          const bool up = (k & size) == 0;
          const uint64_t ka = keys[k], kb = keys[p];
          const uint16_t ia = idxs[k], ib = idxs[p];
          if (less(kb, ib, ka, ia) == up) {
            keys[k] = kb;
            keys[p] = ka;
            idxs[k] = ib;
            idxs[p] = ia;
          }
        }
      }
      __syncwarp();
    }
  }
}

constexpr int FOLD_WARPS = 4;
constexpr int FOLD_CAP = 2048;   // records per pixel sorted in shared memory

// Warp bitonic sort of 32 E (key, id) pairs held in registers in the blocked
// layout i = lane E + e, ascending.  Stage loops are not unrolled (code size:
// the per-pixel kernels were instruction-cache bound); only the element loops
// and the in-register distances (j < E) are static.
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
      for (int e = 0; e < E; ++e) {   // branch-free: selects, no divergent swaps
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, key[e], lj);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, id[e], lj);
        const bool up = ((((int)lane * E + e) & k) == 0);
        const bool take = (lower == up) ? (ok < key[e]) : (ok > key[e]);
        key[e] = take ? ok : key[e];
        id[e] = take ? oi : id[e];
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
            const bool sw = (key[e] > key[p]) == up;
            const uint64_t ke = key[e], kp = key[p];
            const uint32_t ie = id[e], ip = id[p];
            key[e] = sw ? kp : ke;
            key[p] = sw ? ke : kp;
            id[e] = sw ? ip : ie;
            id[p] = sw ? ie : ip;
          }
        }
      }
    }
  }
}


// Common case of the per-pixel fold: up to 32 E records sorted by
// (alpha_near, key) in registers (warp bitonic network over the blocked
// layout i = lane E + e: in-register exchanges for distances < E, shuffles
// beyond), then each lane folds its E consecutive records and the lanes are
// combined by an ordered tree reduction (Eq. aggregate is associative,
// PAPER.md:395-427).  Returns false when records overlap beyond tau or two
// records share the sort key (the caller then sorts under the total order
// and resolves the overlap clusters).
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
  // overlaps beyond tau against the running far end (lane prefix max) and
  // equal sort keys (order not total): both go to the caller's slow path
  float lmax = -3.4e38f;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (id[e] != 0xffffffffu) lmax = fmaxf(lmax, recs[id[e]].alpha_far);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, lmax, o);
    if ((int)lane >= o) lmax = fmaxf(lmax, y);
  }
  float run = __shfl_up_sync(0xffffffffu, lmax, 1);
  uint64_t prev_key = __shfl_up_sync(0xffffffffu, key[E - 1], 1);
  if (lane == 0) {
    run = -3.4e38f;
    prev_key = ~0ull;
  }
  bool ovl = false;
  Acc a{1.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (id[e] == 0xffffffffu) continue;
    const rc_seg& r = recs[id[e]];
    ovl |= (run - r.alpha_near) > tau * fmaxf(1.0f, fabsf(r.alpha_near)) || key[e] == prev_key;
    run = fmaxf(run, r.alpha_far);
    prev_key = key[e];
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

// Two passes: CAP = 512 over every pixel with FOLD_WARPS warps per CTA
// (register sort; a shared-memory sort under the total order when records
// overlap or tie); the few pixels with more records are deferred to a list
// that the second pass (one warp per CTA, CAP = FOLD_CAP_LIST records in
// shared memory) works through.
#ifndef RC_FOLD_MINB
#define RC_FOLD_MINB 8   // A/B at C4 (s8): 8 = 23.2, 6 = 25.2 ms of composite fold per frame
#endif
constexpr int FOLD_MINB = RC_FOLD_MINB;   // resident k_fold<512> CTAs per SM the register budget is sized for (A/B: 4 -> 8 = 31.1 -> 25.4 ms at C4)
constexpr int FOLD_CAP_LIST = 16384;   // records per pixel the composite can order (more: NaN pixel, counted)
template <int CAP, bool FROM_LIST, int NW>
__global__ void __launch_bounds__(NW * 32, CAP <= 512 ? FOLD_MINB : 1) k_fold(
    const rc_seg* __restrict__ recs, const uint32_t* __restrict__ perm, const int64_t* __restrict__ off, int W,
    int H, int tw, int th, const int32_t* __restrict__ my_tiles, int tiles_x, int64_t npix_out, float bg0, float bg1,
    float bg2, float tau, float* __restrict__ rgba, int32_t* __restrict__ defer, int64_t* __restrict__ counters,
    int pps) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * CAP;
  uint16_t* idxs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)NW * CAP) +
                   (size_t)warp * CAP;
  const int64_t tile_px = (int64_t)tw * th;
  const int64_t nq = FROM_LIST ? counters[CNT_DEFER] : npix_out;
  auto locate = [&](int64_t q) -> int64_t {   // output slot q -> image pixel
    const int t = (int)(q / tile_px);
    const int rem = (int)(q - (int64_t)t * tile_px);
    const int tile = my_tiles[t];
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    return (int64_t)(ty * th + rem / tw) * W + (tx * tw + rem % tw);
  };
  // pps (32, or 1 for small images) output pixels per warp step: a lane
  // finishes its pixel alone when it has at most one record (no ordering
  // needed); the others are folded one at a time by the whole warp below
  const int64_t nsteps = FROM_LIST ? nq : (nq + pps - 1) / pps;
  for (int64_t st = (int64_t)blockIdx.x * NW + warp; st < nsteps; st += (int64_t)gridDim.x * NW) {
    unsigned todo = 1u;
    int64_t my_q = 0, my_pix = 0, my_base = 0;
    int my_n = 0;
    if (!FROM_LIST) {
      my_q = st * pps + lane;
      if ((int)lane < pps && my_q < nq) {
        my_pix = locate(my_q);
        my_base = off[my_pix];
        my_n = (int)(off[my_pix + 1] - my_base);
        if (my_n <= 1) {
          Acc a1{1.0, 0.0, 0.0, 0.0};
          if (my_n == 1) {
            const rc_seg& r = recs[perm ? perm[my_base] : (uint32_t)my_base];
            acc_push(a1, r.a, r.b[0], r.b[1], r.b[2]);
          }
          reinterpret_cast<float4*>(rgba)[my_q] =
              make_float4((float)(a1.B0 + a1.A * bg0), (float)(a1.B1 + a1.A * bg1), (float)(a1.B2 + a1.A * bg2),
                          (float)(1.0 - a1.A));
        }
      }
      todo = __ballot_sync(0xffffffffu, (int)lane < pps && my_q < nq && my_n > 1);
    }
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    int64_t q, pix, base;
    int n;
    if (FROM_LIST) {
      q = (int64_t)defer[st];
      pix = locate(q);
      base = off[pix];
      n = (int)(off[pix + 1] - base);
    } else {
      q = __shfl_sync(0xffffffffu, my_q, src);
      pix = __shfl_sync(0xffffffffu, my_pix, src);
      base = __shfl_sync(0xffffffffu, my_base, src);
      n = __shfl_sync(0xffffffffu, my_n, src);
    }
    (void)pix;
    const uint32_t* S = perm ? perm + base : nullptr;   // S[k] = index of the pixel's k-th record (else contiguous copy)
    auto rec = [&](int k) -> const rc_seg& { return recs[S ? S[k] : (uint32_t)(base + k)]; };
    if (!FROM_LIST && n > CAP) {
      if (lane == 0) defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)q;
      continue;
    }
    Acc acc{1.0, 0.0, 0.0, 0.0};
    bool done = false, bad = false;
    if (!FROM_LIST) {
      if (n <= 64) done = fold_pixel_reg<2>(recs, S, base, n, tau, acc);
      else if (n <= 128) done = fold_pixel_reg<4>(recs, S, base, n, tau, acc);
      else if (n <= 256) done = fold_pixel_reg<8>(recs, S, base, n, tau, acc);
      else done = fold_pixel_reg<16>(recs, S, base, n, tau, acc);
    }
    if (!done) {
      if (n <= CAP) {
        int m = 1;
        while (m < n) m <<= 1;
        for (int k = lane; k < m; k += 32) {
          keys[k] = k < n ? sort_key(rec(k)) : ~0ull;
          idxs[k] = (uint16_t)k;
        }
        __syncwarp();
        warp_sort_smem(keys, idxs, n, m, rec);
        fold_sorted([&](int k) -> const rc_seg& { return rec(idxs[k]); }, n, tau, acc);
        __syncwarp();
      } else {
        bad = true;   // more records than one warp can order (FOLD_CAP_LIST): loud NaN pixel
        if (lane == 0) atomicAdd((unsigned long long*)&counters[CNT_BIGPIX], 1ull);
      }
    }
    if (lane == 0) {
      const float4 o = bad ? make_float4(NAN, NAN, NAN, NAN)
                           : make_float4((float)(acc.B0 + acc.A * bg0), (float)(acc.B1 + acc.A * bg1),
                                         (float)(acc.B2 + acc.A * bg2), (float)(1.0 - acc.A));
      reinterpret_cast<float4*>(rgba)[q] = o;
    }
  }
  }
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
// Two passes (as k_fold): k_coarsen_fast takes every pixel with <= 512
// records; the others (and pixels with tied sort keys) are deferred to a list
// that k_coarsen_list works through with a shared-memory sort under the total
// order (FOLD_CAP records; more are passed through re-keyed, unmerged).
__global__ void __launch_bounds__(FOLD_WARPS * 32, 1) k_coarsen_list(
    const rc_seg* __restrict__ recs, const uint32_t* __restrict__ perm, const int64_t* __restrict__ off,
    const int32_t* __restrict__ node_first, const int32_t* __restrict__ leaf_node, uint32_t key_base, float tau,
    rc_seg* __restrict__ out, int64_t out_cap, const int32_t* __restrict__ defer, int64_t* __restrict__ counters) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * FOLD_CAP;
  uint16_t* idxs = reinterpret_cast<uint16_t*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)FOLD_WARPS * FOLD_CAP) +
                   (size_t)warp * FOLD_CAP;
  const int64_t nq = counters[CNT_DEFER];
  for (int64_t qi = (int64_t)blockIdx.x * FOLD_WARPS + warp; qi < nq; qi += (int64_t)gridDim.x * FOLD_WARPS) {
    const int64_t pix = (int64_t)defer[qi];
    const int64_t base = off[pix];
    const int n = (int)(off[pix + 1] - base);
    if (n == 0) continue;
    const uint32_t* S = perm + base;
    if (n > FOLD_CAP) {   // rare: pass through, re-keyed by the target node
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
    {
      int m = 1;
      while (m < n) m <<= 1;
      for (int k = lane; k < m; k += 32) {
        keys[k] = k < n ? sort_key(recs[S[k]]) : ~0ull;
        idxs[k] = (uint16_t)k;
      }
      __syncwarp();
      warp_sort_smem(keys, idxs, n, m, [&](int k) -> const rc_seg& { return recs[S[k]]; });
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

// Fast path of the aggregation pass: pixels with <= COARSEN_FAST_CAP records
// (C5: ~240 records per covered pixel after the on-chip fold).  Each record is
// gathered ONCE (32 bytes, through the pixel-bucketed permutation) into the
// warp's shared memory (structure of arrays: no bank-aligned record stride)
// together with its record key and target-level node; a register bitonic sort
// of (sort key, local index) leaves sorted positions l E .. l E + E - 1 in
// lane l; the maximal runs of touching records of one node are folded nearest
// first (Eq. aggregate) by the whole warp: per-lane partial folds and a
// segmented scan of the open run across the lanes, so long runs (deep
// coarsening: a ray crossing one big node) do not serialise on one lane.
// Pixels with tied sort keys or more records go to the list pass.
constexpr int COARSEN_FAST_CAP = 512;
constexpr int COARSEN_MAIN_CAP = 256;   // main pass; 256 < n <= 512 go to a second pass over a list
constexpr int COARSEN_FAST_WARPS = 2;
struct Acc;
__device__ __forceinline__ void acc_push(Acc& acc, double a, double b0, double b1, double b2);
template <int CAP>
struct CoarsenSmemT {                   // per warp, structure of arrays
  float an[CAP], af[CAP], a[CAP], b0[CAP], b1[CAP], b2[CAP];
  int32_t node[CAP];
  __device__ __forceinline__ void push(Acc& x, uint32_t i) const { acc_push(x, a[i], b0[i], b1[i], b2[i]); }
};

// Warp bitonic sort of 32 E 32-bit keys in the blocked layout i = lane E + e,
// ascending (as warp_sort_blocked, one register per element: the aggregation
// pass embeds the local index in the key's low bits).
template <int E>
__device__ __forceinline__ void warp_sort32(uint32_t (&key)[E]) {
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
        const uint32_t ok = __shfl_xor_sync(0xffffffffu, key[e], lj);
        const bool up = ((((int)lane * E + e) & k) == 0);
        key[e] = (lower == up) ? min(ok, key[e]) : max(ok, key[e]);
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
            const uint32_t lo = min(key[e], key[p]), hi = max(key[e], key[p]);
            key[e] = up ? lo : hi;
            key[p] = up ? hi : lo;
          }
        }
      }
    }
  }
}

// returns false when two records' alpha_near cannot be told apart by the
// 22-bit sort key (their order-preserving bits agree after the pixel's range
// shift; the caller defers the pixel to the list pass, which sorts under the
// total order)
template <int E, class Smem>
__device__ __forceinline__ bool coarsen_pixel(const Smem& C, int n, int64_t pix,
                                              const int32_t* __restrict__ node_first, uint32_t key_base, float tau,
                                              rc_seg* __restrict__ out, int64_t out_cap,
                                              int64_t* __restrict__ counters, const uint16_t* list = nullptr,
                                              int* agree = nullptr) {
  // list: the local indices of the n records to fold (nullptr: 0 .. n-1);
  // agree: the CTA's warps fold disjoint groups of one pixel and emit only if
  // none of them found a tie (two shared-memory flags, CTA barriers)
  const unsigned lane = threadIdx.x & 31;
  // sort key: alpha_near's order-preserving bits relative to the pixel's
  // smallest, shifted into 22 bits (exact while the pixel's alpha range spans
  // < 2^22 ulps), above the 9-bit local index; < 2^31, below the 0xffffffff pad
  uint32_t key[E];
  uint32_t omin = 0xffffffffu, omax = 0u;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int pos = (int)lane * E + e;
    const int i = pos < n ? (list ? (int)list[pos] : pos) : 0;
    key[e] = pos < n ? ord_bits(C.an[i]) : 0u;
    if (pos < n) {
      omin = min(omin, key[e]);
      omax = max(omax, key[e]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    omin = min(omin, __shfl_xor_sync(0xffffffffu, omin, o));
    omax = max(omax, __shfl_xor_sync(0xffffffffu, omax, o));
  }
  const uint32_t range = omax - omin;
  const int sh = max(0, 32 - __clz((int)range) - 22);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int pos = (int)lane * E + e;
    const uint32_t i = pos < n ? (list ? (uint32_t)list[pos] : (uint32_t)pos) : 0u;
    key[e] = pos < n ? ((((key[e] - omin) >> sh) << 9) | i) : 0xffffffffu;
  }
  warp_sort32<E>(key);
  uint32_t id[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    id[e] = key[e] & 0x1FFu;
    RC_DCHECK((int)lane * E + e >= n || (int)id[e] < (list ? COARSEN_FAST_CAP : n));
  }
  {
    uint32_t prev_key = __shfl_up_sync(0xffffffffu, key[E - 1], 1);
    bool tie = false;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = (int)lane * E + e;
      tie |= k > 0 && k < n && (key[e] >> 9) == (prev_key >> 9);
      prev_key = key[e];
    }
    bool any = __any_sync(0xffffffffu, tie);
    if (agree) {
      if (lane == 0) agree[threadIdx.x >> 5] = any ? 1 : 0;
      __syncthreads();
      any = false;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) any |= agree[w] != 0;
      __syncthreads();
    }
    if (any) return false;
  }
  // head flags of this lane's positions (a run starts at a gap / overlap or a new node)
  const int lo = (int)lane * E;
  uint32_t prev = __shfl_up_sync(0xffffffffu, id[E - 1], 1);
  uint32_t heads = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = lo + e;
    if (k < n) {
      bool h = k == 0;
      if (!h) {
        const float an = C.an[id[e]];
        h = fabsf(an - C.af[prev]) > tau * fmaxf(1.0f, fabsf(an)) || C.node[id[e]] != C.node[prev];
      }
      heads |= (h ? 1u : 0u) << e;
    }
    prev = id[e];
  }
  // pass 1: the lane's open tail (from its last head, or its start)
  bool F = false;
  uint32_t HID = 0;   // local index of the lane's last head record
  Acc X{1.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (lo + e < n) {   // predicated, no early exit (positions >= n are the tail)
      if ((heads >> e) & 1u) {
        F = true;
        HID = id[e];
        X = Acc{1.0, 0.0, 0.0, 0.0};
      }
      C.push(X, id[e]);
    }
  }
  const int hi = min(n, lo + E);
  int nemit = __popc(heads & ~(lo == 0 ? 1u : 0u)) + ((lo < hi && hi == n) ? 1 : 0);
  // exclusive segmented scan across lanes: the run entering this lane
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool Fo = __shfl_up_sync(0xffffffffu, F, o);
    const uint32_t HIDo = __shfl_up_sync(0xffffffffu, HID, o);
    const double Ao = __shfl_up_sync(0xffffffffu, X.A, o), B0o = __shfl_up_sync(0xffffffffu, X.B0, o);
    const double B1o = __shfl_up_sync(0xffffffffu, X.B1, o), B2o = __shfl_up_sync(0xffffffffu, X.B2, o);
    if ((int)lane >= o && !F) {   // (nearer lanes) (+) (this one)
      Acc y{Ao, B0o, B1o, B2o};
      acc_push(y, X.A, X.B0, X.B1, X.B2);
      X = y;
      F = Fo;
      HID = HIDo;
    }
  }
  Acc acc{__shfl_up_sync(0xffffffffu, X.A, 1), __shfl_up_sync(0xffffffffu, X.B0, 1),
          __shfl_up_sync(0xffffffffu, X.B1, 1), __shfl_up_sync(0xffffffffu, X.B2, 1)};
  uint32_t start_id = __shfl_up_sync(0xffffffffu, HID, 1);   // head of the run entering this lane
  if (lane == 0) {
    acc = Acc{1.0, 0.0, 0.0, 0.0};
    start_id = id[0];
  }
  // pass 2: emit every run that ends in this lane's positions
  int64_t slot = warp_append(&counters[CNT_AGG_OUT], nemit);
  auto emit = [&](uint32_t i0, uint32_t i1, const Acc& v) {
    if (slot < out_cap) {
      const float bb[3] = {(float)v.B0, (float)v.B1, (float)v.B2};
      store_seg(out + slot, (uint32_t)pix, C.an[i0], C.af[i1], (float)v.A, bb,
                key_base + (uint32_t)node_first[C.node[i0]]);
    } else {
      atomicAdd((unsigned long long*)&counters[CNT_OVERFLOW], 1ull);
    }
    ++slot;
  };
  uint32_t last_id = __shfl_up_sync(0xffffffffu, id[E - 1], 1);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = lo + e;
    if (k < n) {
      if (k > 0 && ((heads >> e) & 1u)) {
        emit(start_id, last_id, acc);
        acc = Acc{1.0, 0.0, 0.0, 0.0};
        start_id = id[e];
      }
      C.push(acc, id[e]);
      last_id = id[e];
    }
  }
  if (lo < hi && hi == n) emit(start_id, last_id, acc);
  return true;
}

// Main pass (CAP = 256): one warp per pixel (grid-stride over all pixels);
// 256 < n <= 512 go to the mid list, larger ones to the defer list.  The
// record gathers and the target-node lookups are separate loops (independent
// loads in flight).
__global__ void __launch_bounds__(COARSEN_FAST_WARPS * 32, 10) k_coarsen_fast(
    const rc_seg* __restrict__ recs, int64_t nrec, int64_t nleaf, const uint32_t* __restrict__ perm,
    const int64_t* __restrict__ off, int64_t npix,
    const int32_t* __restrict__ node_first, const int32_t* __restrict__ leaf_node, uint32_t key_base, float tau,
    rc_seg* __restrict__ out, int64_t out_cap, int32_t* __restrict__ defer, int32_t* __restrict__ mid,
    int64_t* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  CoarsenSmemT<COARSEN_MAIN_CAP>& C = reinterpret_cast<CoarsenSmemT<COARSEN_MAIN_CAP>*>(smem_raw)[warp];
  const float4* recs4 = reinterpret_cast<const float4*>(recs);
  for (int64_t pix = (int64_t)blockIdx.x * COARSEN_FAST_WARPS + warp; pix < npix;
       pix += (int64_t)gridDim.x * COARSEN_FAST_WARPS) {
    const int64_t base = off[pix];
    const int n = (int)(off[pix + 1] - base);
    if (n == 0) continue;
    if (n > COARSEN_MAIN_CAP) {
      if (lane == 0) {
        if (n <= COARSEN_FAST_CAP) mid[atomicAdd((unsigned long long*)&counters[CNT_MID], 1ull)] = (int32_t)pix;
        else defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)pix;
      }
      continue;
    }
    const uint32_t* S = perm + base;
    // 1. one gather per record; the record key parks in node[] ...
#pragma unroll 4
    for (int k = lane; k < n; k += 32) {
      const uint32_t id = S[k];
      RC_DCHECK((int64_t)id < nrec);
      const float4 lo = recs4[2 * (size_t)id], hi = recs4[2 * (size_t)id + 1];
      C.an[k] = lo.y;
      C.af[k] = lo.z;
      C.a[k] = lo.w;
      C.b0[k] = hi.x;
      C.b1[k] = hi.y;
      C.b2[k] = hi.z;
      C.node[k] = (int32_t)(__float_as_uint(hi.w) - key_base);
    }
    // ... 2. and becomes its node at the target level (independent lookups)
#pragma unroll 8
    for (int k = lane; k < n; k += 32) {
      RC_DCHECK(C.node[k] >= 0 && C.node[k] < nleaf);
      C.node[k] = leaf_node[C.node[k]];
    }
    __syncwarp();
    bool ok;
    if (n <= 64) ok = coarsen_pixel<2>(C, n, pix, node_first, key_base, tau, out, out_cap, counters);
    else if (n <= 128) ok = coarsen_pixel<4>(C, n, pix, node_first, key_base, tau, out, out_cap, counters);
    else ok = coarsen_pixel<8>(C, n, pix, node_first, key_base, tau, out, out_cap, counters);
    if (!ok && lane == 0) defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)pix;
    __syncwarp();
  }
}

// Mid pass: 256 < n <= 512.  Runs never cross target nodes, so the records
// split into two independent groups by one bit of the node id (of the lowest
// four, the one with the most even split): one CTA per pixel, warp g folds
// group g (<= 256 records, else the pixel is deferred) with the main pass's
// warp code; the warps emit only if neither met a tie (shared-memory flags
// between CTA barriers).  (A/B at C5: this kernel 106 ms; four warps and
// groups by node id mod 4 133 ms; a 16-byte layout re-reading (a, b) from
// L1/L2 158 ms; one warp per (pixel, parity) with the main pass's layout
// 132 ms + 20 ms more in the list pass.)
constexpr int MID_WARPS = 2;
struct CoarsenMidSmem {
  CoarsenSmemT<COARSEN_FAST_CAP> C;
  uint16_t list[MID_WARPS][COARSEN_MAIN_CAP];
  int ng[MID_WARPS];
  int agree[MID_WARPS];
};

__global__ void __launch_bounds__(MID_WARPS * 32, 8) k_coarsen_mid(
    const rc_seg* __restrict__ recs, int64_t nrec, int64_t nleaf, const uint32_t* __restrict__ perm,
    const int64_t* __restrict__ off, const int32_t* __restrict__ node_first, const int32_t* __restrict__ leaf_node,
    uint32_t key_base, float tau, rc_seg* __restrict__ out, int64_t out_cap, int32_t* __restrict__ defer,
    const int32_t* __restrict__ mid, int64_t* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CoarsenMidSmem& M = *reinterpret_cast<CoarsenMidSmem*>(smem_raw);
  CoarsenSmemT<COARSEN_FAST_CAP>& C = M.C;
  const int warp = threadIdx.x >> 5;
  const unsigned lane = threadIdx.x & 31;
  const float4* recs4 = reinterpret_cast<const float4*>(recs);
  const int64_t nq = counters[CNT_MID];
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    const int64_t pix = mid[q];
    const int64_t base = off[pix];
    const int n = (int)(off[pix + 1] - base);
    const uint32_t* S = perm + base;
#pragma unroll 4
    for (int k = threadIdx.x; k < n; k += MID_WARPS * 32) {
      const uint32_t id = S[k];
      RC_DCHECK((int64_t)id < nrec);
      const float4 lo = recs4[2 * (size_t)id], hi = recs4[2 * (size_t)id + 1];
      C.an[k] = lo.y;
      C.af[k] = lo.z;
      C.a[k] = lo.w;
      C.b0[k] = hi.x;
      C.b1[k] = hi.y;
      C.b2[k] = hi.z;
      C.node[k] = (int32_t)(__float_as_uint(hi.w) - key_base);
    }
#pragma unroll 8
    for (int k = threadIdx.x; k < n; k += MID_WARPS * 32) {
      RC_DCHECK(C.node[k] >= 0 && C.node[k] < nleaf);
      C.node[k] = leaf_node[C.node[k]];
    }
    __syncthreads();
    int c1[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + (int)lane;
      const int nd = k < n ? C.node[k] : 0;
#pragma unroll
      for (int bit = 0; bit < 4; ++bit) c1[bit] += __popc(__ballot_sync(0xffffffffu, k < n && ((nd >> bit) & 1)));
    }
    int sbit = 0, best = n;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
      const int worst = max(c1[bit], n - c1[bit]);
      if (worst < best) {
        best = worst;
        sbit = bit;
      }
    }
    // warp g lists the records of group g, in index order
    int ng = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + (int)lane;
      const bool mine = k < n && ((C.node[k] >> sbit) & 1) == warp;
      const unsigned bal = __ballot_sync(0xffffffffu, mine);
      const int pos = ng + __popc(bal & lanemask_lt());
      if (mine && pos < COARSEN_MAIN_CAP) M.list[warp][pos] = (uint16_t)k;
      ng += __popc(bal);
    }
    if (lane == 0) M.ng[warp] = ng;
    __syncthreads();
    const int ngmax = max(M.ng[0], M.ng[1]);
    bool ok = ngmax <= COARSEN_MAIN_CAP;
    if (ok) {   // uniform over the CTA: the same instantiation in both warps
      if (ngmax <= 64) ok = coarsen_pixel<2>(C, ng, pix, node_first, key_base, tau, out, out_cap, counters, M.list[warp], M.agree);
      else if (ngmax <= 128) ok = coarsen_pixel<4>(C, ng, pix, node_first, key_base, tau, out, out_cap, counters, M.list[warp], M.agree);
      else ok = coarsen_pixel<8>(C, ng, pix, node_first, key_base, tau, out, out_cap, counters, M.list[warp], M.agree);
    }
    if (!ok && threadIdx.x == 0) defer[atomicAdd((unsigned long long*)&counters[CNT_DEFER], 1ull)] = (int32_t)pix;
    __syncthreads();
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
                          const int64_t* d_nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap,
                          int32_t* hits_pp, int64_t* counters, int grid, cudaStream_t s) {
  const bool adapt = cc.scheme != RC_SCHEME_GL || cc.c_rk > 0.0f;   // separate instantiation (see cast_curved.cu)
#define CASE(N)                                                                                                    \
  case N:                                                                                                          \
    if (adapt)                                                                                                     \
      k_cast_affine<P, N, true><<<grid, 256, 0, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks,     \
                                                     d_nchunks, key_base, segs, seg_cap, hits_pp, counters);       \
    else                                                                                                           \
      k_cast_affine<P, N, false><<<grid, 256, 0, s>>>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks,    \
                                                      d_nchunks, key_base, segs, seg_cap, hits_pp, counters);      \
    break;
  switch (cc.N) { CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) }
#undef CASE
}

cudaError_t launch_cast_affine(const CamConst& cc, const TreeConst* trees, DevLeafView L, int P, const int32_t* vis,
                               const Rect16* vrect, const int64_t* chunk_off, const int32_t* chunk_elem,
                               int64_t nchunks, uint32_t key_base, rc_seg* segs, int64_t seg_cap, int32_t* hits_pp,
                               int64_t* counters, int grid, cudaStream_t s, const int64_t* d_nchunks) {
  if (P == 1) cast_affine_P<1>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, d_nchunks, key_base, segs,
                               seg_cap, hits_pp, counters, grid, s);
  else cast_affine_P<2>(cc, trees, L, vis, vrect, chunk_off, chunk_elem, nchunks, d_nchunks, key_base, segs, seg_cap,
                        hits_pp, counters, grid, s);
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

cudaError_t launch_leaf_weights(const int32_t* flag, const Rect16* rect, int64_t n, int64_t* w, cudaStream_t s) {
  k_leaf_weights<<<nblk(n, 256), 256, 0, s>>>(flag, rect, n, w);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_pack_offsets(const int64_t* counts, int nranks, int64_t* dest_off, cudaStream_t s) {
  k_pack_offsets<<<1, 32, 0, s>>>(counts, nranks, dest_off);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_hist(const rc_seg* segs, int64_t n, int32_t* cnt, int grid, cudaStream_t s, const int64_t* d_n) {
  k_hist<<<grid, 256, 0, s>>>(segs, n, d_n, cnt);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_scatter(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, uint32_t* out,
                           int grid, cudaStream_t s, const int64_t* d_n) {
  k_scatter<<<grid, 256, 0, s>>>(segs, n, d_n, off, cursor, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_band_bucket(const rc_seg* segs, int64_t n, int64_t npix, int32_t* bcnt, int64_t* boff,
                               int64_t* scan_tmp, void* scratch, uint32_t* perm, int64_t* off, int grid,
                               cudaStream_t s) {
  uint64_t* tmp = reinterpret_cast<uint64_t*>(scratch);
  const int64_t nb = (npix + (1 << BAND_SH) - 1) >> BAND_SH;
  cudaError_t e = cudaMemsetAsync(bcnt, 0, sizeof(int32_t) * (nb + 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0) k_band_count<<<grid, 256, 0, s>>>(segs, n, bcnt);
  e = scan_exclusive<int32_t>(bcnt, boff, nb, scan_tmp, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(bcnt, 0, sizeof(int32_t) * (nb + 1), s);   // reused as cursors
  if (e != cudaSuccess) return e;
  if (n > 0) k_band_scatter<<<grid, 256, 0, s>>>(segs, n, boff, bcnt, tmp);
  k_band_sort<<<(unsigned)std::min<int64_t>(nb, 148 * 4), 512, 0, s>>>(tmp, boff, nb, npix, perm, off);
  g_launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_scatter_rec(const rc_seg* segs, int64_t n, const int64_t* off, int32_t* cursor, rc_seg* out,
                               int grid, cudaStream_t s, const int64_t* d_n) {
  k_scatter_rec<<<grid, 256, 0, s>>>(segs, n, d_n, off, cursor, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_coarsen(const rc_seg* recs, int64_t nrec, int64_t nleaf, const uint32_t* perm, const int64_t* off,
                           int64_t npix,
                           const int32_t* node_first, const int32_t* leaf_node, uint32_t key_base, float tau, rc_seg* out,
                           int64_t out_cap, int32_t* defer, int32_t* mid, int64_t* counters, int max_grid,
                           cudaStream_t s) {
  static bool attr = false;
  const size_t smem_main = sizeof(CoarsenSmemT<COARSEN_MAIN_CAP>) * COARSEN_FAST_WARPS;
  const size_t smem_mid = sizeof(CoarsenMidSmem);
  const size_t smeml = (size_t)FOLD_WARPS * FOLD_CAP * (sizeof(uint64_t) + sizeof(uint16_t));
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_coarsen_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_main);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_coarsen_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mid);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_coarsen_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smeml);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaError_t e = cudaMemsetAsync(counters + CNT_DEFER, 0, sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(counters + CNT_MID, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>((npix + COARSEN_FAST_WARPS - 1) / COARSEN_FAST_WARPS, (int64_t)max_grid);
  k_coarsen_fast<<<grid, COARSEN_FAST_WARPS * 32, smem_main, s>>>(recs, nrec, nleaf, perm, off, npix, node_first, leaf_node,
                                                                  key_base, tau, out, out_cap, defer, mid, counters);
  k_coarsen_mid<<<grid, MID_WARPS * 32, smem_mid, s>>>(recs, nrec, nleaf, perm, off, node_first, leaf_node, key_base,
                                                       tau, out, out_cap, defer, mid, counters);
  k_coarsen_list<<<std::min(grid, 296), FOLD_WARPS * 32, smeml, s>>>(recs, perm, off, node_first, leaf_node, key_base,
                                                                     tau, out, out_cap, defer, counters);
  g_launches += 3;
  return cudaGetLastError();
}

template <int CAP, bool FROM_LIST, int NW>
static cudaError_t fold_pass(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int W, int H, int tw,
                             int th, const int32_t* my_tiles, int tiles_x, int64_t npix_out, const float bg[3],
                             float tau, float* rgba, int32_t* defer, int64_t* counters, int grid, int pps,
                             cudaStream_t s) {
  static bool attr = false;
  const size_t smem = (size_t)NW * CAP * (sizeof(uint64_t) + sizeof(uint16_t));
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_fold<CAP, FROM_LIST, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_fold<CAP, FROM_LIST, NW><<<grid, NW * 32, smem, s>>>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x, npix_out,
                                                         bg[0], bg[1], bg[2], tau, rgba, defer, counters, pps);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_fold(const rc_seg* recs, const uint32_t* perm, const int64_t* off, int W, int H, int tw, int th,
                        const int32_t* my_tiles, int tiles_x, int64_t npix_out, const float bg[3], float tau,
                        float* rgba, int32_t* defer, int64_t* counters, int max_grid, cudaStream_t s) {
  // small images (C1: 4096 pixels) get one pixel per warp step, so that every
  // pixel's fold runs in its own warp (32 per step left most of the GPU idle)
  const int pps = npix_out < ((int64_t)1 << 17) ? 1 : 32;
  const int grid = (int)std::min<int64_t>((npix_out + (int64_t)FOLD_WARPS * pps - 1) / ((int64_t)FOLD_WARPS * pps),
                                          (int64_t)max_grid);
  cudaError_t e = cudaMemsetAsync(counters + CNT_DEFER, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  e = fold_pass<512, false, FOLD_WARPS>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x, npix_out, bg, tau, rgba,
                                        defer, counters, grid, pps, s);
  if (e != cudaSuccess) return e;
  // the deferred pixels (n > 512): a fixed grid reading the list length on the device
  return fold_pass<FOLD_CAP_LIST, true, 1>(recs, perm, off, W, H, tw, th, my_tiles, tiles_x, npix_out, bg, tau, rgba,
                                           defer, counters, std::min(grid, 296), 1, s);
}

}  // namespace rc
