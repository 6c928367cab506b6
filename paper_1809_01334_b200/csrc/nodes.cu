// nodes.cu -- the coarsening hierarchy of the local forest (PAPER.md:956-994,
// §3 "coarsening": "complete local sibling families" are replaced by their
// parent, one level per cycle).
//
// Level 0 is the SFC-ordered leaf array itself.  Level c+1 is level c with
// every complete family of 8 same-level siblings (4 for the quadtrees of surface forests; 8 consecutive nodes with
// the same tree, level l >= 1 and parent, child ids 0..7 in Morton order)
// replaced by its parent.  Families split across ranks are incomplete
// locally and stay.  A node is stored by the local index
// of its first leaf; node k of level c owns leaves [first[k], first[k+1]).
// The tables depend on the forest only (not on the camera) and are built once
// in rc_forest_create.  They define the fold units of the segment kernel
// (row a6) and the parents of rc_aggregate (row a7).
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace rc {

namespace {

struct NodeView {
  const int32_t* tree;
  const int32_t* anchor;   // [n][3]
  const int8_t* level;
  const int32_t* first;    // nullptr at level 0 (identity)
};

__device__ __forceinline__ int child_id(const int32_t* a, int lvl) {
  const int b = RC_MAXLEVEL - lvl;
  return ((a[0] >> b) & 1) | (((a[1] >> b) & 1) << 1) | (((a[2] >> b) & 1) << 2);
}

// flag[k] = 1 iff nodes k..k+fam-1 form a complete family (k is child 0);
// fam = 8 (octrees) or 4 (quadtrees of surface forests: z anchors are 0)
__global__ void k_family_start(NodeView V, int64_t n, int fam, int32_t* __restrict__ flag) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int f = 0;
  const int lvl = V.level[k];
  if (k + fam - 1 < n && lvl >= 1 && child_id(V.anchor + 3 * k, lvl) == 0) {
    const int t = V.tree[k];
    const int32_t pm = ~((1 << (RC_MAXLEVEL - lvl + 1)) - 1);
    const int32_t p0 = V.anchor[3 * k] & pm, p1 = V.anchor[3 * k + 1] & pm, p2 = V.anchor[3 * k + 2] & pm;
    f = 1;
    for (int j = 1; j < fam && f; ++j) {
      const int64_t q = k + j;
      const int32_t* a = V.anchor + 3 * q;
      if (V.tree[q] != t || V.level[q] != lvl || (a[0] & pm) != p0 || (a[1] & pm) != p1 || (a[2] & pm) != p2 ||
          child_id(a, lvl) != j)
        f = 0;
    }
  }
  flag[k] = f;
}

// keep[k] = 1 unless k is a non-first member of a family
__global__ void k_family_keep(const int32_t* __restrict__ start, int64_t n, int fam, int32_t* __restrict__ keep) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int in_family = 0;
  for (int j = 1; j < fam; ++j)
    if (k - j >= 0 && start[k - j]) in_family = 1;
  keep[k] = in_family ? 0 : 1;
}

__global__ void k_family_emit(NodeView V, int64_t n, const int32_t* __restrict__ start,
                              const int32_t* __restrict__ keep, const int64_t* __restrict__ pos,
                              int32_t* __restrict__ o_tree, int32_t* __restrict__ o_anchor, int8_t* __restrict__ o_level,
                              int32_t* __restrict__ o_first) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || !keep[k]) return;
  const int64_t p = pos[k];
  int lvl = V.level[k];
  int32_t a0 = V.anchor[3 * k], a1 = V.anchor[3 * k + 1], a2 = V.anchor[3 * k + 2];
  if (start[k]) {   // child 0 carries the parent's anchor already
    --lvl;
  }
  o_tree[p] = V.tree[k];
  o_anchor[3 * p] = a0;
  o_anchor[3 * p + 1] = a1;
  o_anchor[3 * p + 2] = a2;
  o_level[p] = (int8_t)lvl;
  o_first[p] = V.first ? V.first[k] : (int32_t)k;
}

__global__ void k_set_sentinel(int32_t* first, int64_t n, int32_t value) { first[n] = value; }

// per-leaf node index at one level: the node k with first[k] <= e < first[k+1]
__global__ void k_leaf_node(const int32_t* __restrict__ first, int64_t nnodes, int64_t n,
                            int32_t* __restrict__ leaf_node) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  leaf_node[e] = (int32_t)node_of(first, nnodes, (int32_t)e);
}

unsigned nb(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// Builds f->d_node_first[1..RC_NODE_LEVELS] and f->n_nodes[] (one level per
// coarsening cycle; a level that coarsens nothing repeats the previous one).
cudaError_t build_node_levels(rc_forest* f, cudaStream_t s) {
  const int64_t n = f->n;
  int32_t *tree[2] = {nullptr, nullptr}, *anchor[2] = {nullptr, nullptr}, *first[2] = {nullptr, nullptr};
  int8_t* level[2] = {nullptr, nullptr};
  int32_t *start = nullptr, *keep = nullptr;
  int64_t* pos = nullptr;
  cudaError_t e = cudaSuccess;
#define TRY(x)                      \
  if ((e = (x)) != cudaSuccess) { \
    goto done;                      \
  }
  TRY(dmalloc((void**)&start, sizeof(int32_t) * (n + 1), s));
  TRY(dmalloc((void**)&keep, sizeof(int32_t) * (n + 1), s));
  TRY(dmalloc((void**)&pos, sizeof(int64_t) * (n + 1), s));
  for (int b = 0; b < 2; ++b) {
    TRY(dmalloc((void**)&tree[b], sizeof(int32_t) * (n + 8), s));
    TRY(dmalloc((void**)&anchor[b], sizeof(int32_t) * 3 * (n + 8), s));
    TRY(dmalloc((void**)&level[b], sizeof(int8_t) * (n + 8), s));
    TRY(dmalloc((void**)&first[b], sizeof(int32_t) * (n + 8), s));
  }
  {
    f->n_nodes[0] = n;
    NodeView V{f->d_tree, f->d_anchor, f->d_level, nullptr};
    int64_t cur = n;
    int out = 0;
    const int fam = f->surface ? 4 : 8;   // complete sibling families
    for (int c = 1; c <= RC_NODE_LEVELS; ++c) {
      k_family_start<<<nb(cur, 256), 256, 0, s>>>(V, cur, fam, start);
      k_family_keep<<<nb(cur, 256), 256, 0, s>>>(start, cur, fam, keep);
      g_launches += 2;
      TRY(scan_exclusive<int32_t>(keep, pos, cur, f->d_scan_tmp, s));
      int64_t next = 0;
      TRY(cudaMemcpyAsync(&next, pos + cur, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      TRY(cudaStreamSynchronize(s));
      int32_t* fo = nullptr;
      TRY(dmalloc((void**)&fo, sizeof(int32_t) * (next + 1), s));
      f->d_node_first[c] = fo;
      f->n_nodes[c] = next;
      k_family_emit<<<nb(cur, 256), 256, 0, s>>>(V, cur, start, keep, pos, tree[out], anchor[out], level[out],
                                                 first[out]);
      ++g_launches;
      TRY(cudaMemcpyAsync(fo, first[out], sizeof(int32_t) * next, cudaMemcpyDeviceToDevice, s));
      k_set_sentinel<<<1, 1, 0, s>>>(fo, next, (int32_t)n);
      ++g_launches;
      V = NodeView{tree[out], anchor[out], level[out], first[out]};
      cur = next;
      out ^= 1;
    }
    TRY(cudaStreamSynchronize(s));
  }
done:
#undef TRY
  dfree(start, s);
  dfree(keep, s);
  dfree(pos, s);
  for (int b = 0; b < 2; ++b) {
    dfree(tree[b], s);
    dfree(anchor[b], s);
    dfree(level[b], s);
    dfree(first[b], s);
  }
  return e;
}

// Per-leaf node index at level c (c >= 1), cached for the last two levels
// asked for (the fold level of the cast and the target level of rc_aggregate).
cudaError_t build_leaf_node(rc_forest* f, int c, cudaStream_t s, const int32_t** out) {
  for (int k = 0; k < 2; ++k)
    if (f->leaf_node_lv[k] == c && f->d_leaf_nodes[k]) {
      *out = f->d_leaf_nodes[k];
      return cudaSuccess;
    }
  const int k = f->leaf_node_next;
  f->leaf_node_next ^= 1;
  if (!f->d_leaf_nodes[k]) {
    cudaError_t e = dmalloc((void**)&f->d_leaf_nodes[k], sizeof(int32_t) * f->n, s);
    if (e != cudaSuccess) return e;
  }
  k_leaf_node<<<nb(f->n, 256), 256, 0, s>>>(f->d_node_first[c], f->n_nodes[c], f->n, f->d_leaf_nodes[k]);
  ++g_launches;
  f->leaf_node_lv[k] = c;
  *out = f->d_leaf_nodes[k];
  return cudaGetLastError();
}

}  // namespace rc
