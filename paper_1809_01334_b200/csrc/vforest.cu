// vforest.cu -- multiple image instances and the visualization forest
// ("Culling and pre-partition").
//
// Instances: the cull runs once per instance camera (rc_camera_set + rc_cull);
// rc_visible_area_add accumulates each instance's pixel-centre rectangle area
// per leaf into a caller buffer, so a leaf stays in as long as one instance
// sees it ("Top-down traversals of the forest will continue until the last of
// the instances considers a leaf or subtree invisible") and
// its weight is "proportional to its visible pixel count summed over all
// instances".  rc_vforest_create copies the leaves of
// positive weight -- keys and field, a stream compaction on the device --
// into a new forest: the paper's vforest ("copying only the data of the
// visible elements"), which is then repartitioned by those
// weights (dist.py) and rendered once per instance.  The input forest is read
// only ("We render non-destructively").
#include <cuda_runtime.h>
#include <string.h>

#include <vector>

#include "rc_internal.cuh"
#include "scan.cuh"

using namespace rc;

#define CU(call)                                                                                              \
  do {                                                                                                        \
    cudaError_t e_ = (call);                                                                                  \
    if (e_ != cudaSuccess)                                                                                    \
      return rc_fail(e_ == cudaErrorMemoryAllocation ? RC_ERR_OUT_OF_MEMORY : RC_ERR_CUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                                      \
  } while (0)

namespace {
__global__ void k_area_add(const int32_t* __restrict__ flag, const Rect16* __restrict__ rect, int64_t n,
                           int64_t* __restrict__ w) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n || !flag[e]) return;
  const Rect16 r = rect[e];
  w[e] += (int64_t)(r.i1 - r.i0 + 1) * (int64_t)(r.j1 - r.j0 + 1);
}

__global__ void k_keep_flag(const int64_t* __restrict__ w, int64_t n, int32_t* __restrict__ keep) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) keep[e] = w[e] > 0 ? 1 : 0;
}

// one thread per kept leaf: keys, weight and the (P+1)^3 (or 4) field values
__global__ void k_gather_leaves(const int32_t* __restrict__ keep, const int64_t* __restrict__ pos, int64_t n,
                                DevLeafView L, int nf, const int64_t* __restrict__ w, int32_t* __restrict__ anchor,
                                int32_t* __restrict__ tree, int8_t* __restrict__ level, float* __restrict__ field,
                                int64_t* __restrict__ w_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n || !keep[e]) return;
  const int64_t p = pos[e];
  for (int k = 0; k < 3; ++k) anchor[3 * p + k] = L.anchor[3 * e + k];
  tree[p] = L.tree[e];
  level[p] = L.level[e];
  if (field)
    for (int q = 0; q < nf; ++q) field[p * nf + q] = L.field[e * nf + q];
  if (w_out) w_out[p] = w[e];
}

unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }
}  // namespace

extern "C" rc_status rc_visible_area_add(rc_forest* f, int64_t* d_w, int64_t capacity, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !d_w) return rc_fail(RC_ERR_INVALID_ARG, "rc_visible_area_add: null argument");
  if (!f->have_cull) return rc_fail(RC_ERR_STATE, "rc_visible_area_add before rc_cull");
  if (capacity < f->n)
    return rc_fail(RC_ERR_CAPACITY, "rc_visible_area_add: capacity %lld < %lld leaves", (long long)capacity,
                   (long long)f->n);
  cudaStream_t s = (cudaStream_t)stream;
  k_area_add<<<blocks(f->n), 256, 0, s>>>(f->d_flag, f->d_rect_all, f->n, d_w);
  ++g_launches;
  CU(cudaGetLastError());
  return RC_OK;
}

extern "C" rc_status rc_vforest_create(rc_forest* f, const int64_t* d_w, int64_t first_global_leaf, void* stream,
                                       rc_forest** out, int64_t* h_count, int64_t* d_w_out) {
  RC_NVTX("rc_vforest_create");
  if (!f || !d_w || !out || !h_count) return rc_fail(RC_ERR_INVALID_ARG, "rc_vforest_create: null argument");
  *out = nullptr;
  *h_count = 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n;
  const int nf = f->surface ? 4 : (f->P + 1) * (f->P + 1) * (f->P + 1);
  int32_t* keep = nullptr;
  int64_t *pos = nullptr, *tmp = nullptr;
  int32_t *anchor = nullptr, *tree = nullptr;
  int8_t* level = nullptr;
  float* field = nullptr;
  rc_status st = RC_OK;
  auto release = [&]() {
    for (void* p : {(void*)keep, (void*)pos, (void*)tmp, (void*)anchor, (void*)tree, (void*)level, (void*)field})
      if (p) dfree(p, s);
  };
#define TRY(call)                                                                                     \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess) {                                                                          \
      st = rc_fail(e_ == cudaErrorMemoryAllocation ? RC_ERR_OUT_OF_MEMORY : RC_ERR_CUDA, "%s: %s", #call, \
                   cudaGetErrorString(e_));                                                           \
      release();                                                                                      \
      return st;                                                                                      \
    }                                                                                                 \
  } while (0)
  TRY(dmalloc((void**)&keep, sizeof(int32_t) * n, s));
  TRY(dmalloc((void**)&pos, sizeof(int64_t) * (n + 1), s));
  TRY(dmalloc((void**)&tmp, sizeof(int64_t) * scan_tmp_size(n), s));
  k_keep_flag<<<blocks(n), 256, 0, s>>>(d_w, n, keep);
  ++g_launches;
  TRY(cudaGetLastError());
  TRY(scan_exclusive<int32_t>(keep, pos, n, tmp, s));
  int64_t m = 0;
  TRY(cudaMemcpyAsync(&m, pos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TRY(cudaStreamSynchronize(s));
  *h_count = m;
  if (m == 0) {
    release();
    return RC_OK;
  }
  TRY(dmalloc((void**)&anchor, sizeof(int32_t) * 3 * m, s));
  TRY(dmalloc((void**)&tree, sizeof(int32_t) * m, s));
  TRY(dmalloc((void**)&level, m, s));
  if (f->has_field) TRY(dmalloc((void**)&field, sizeof(float) * nf * m, s));
  DevLeafView L{f->d_anchor, f->d_tree, f->d_level, f->d_field};
  k_gather_leaves<<<blocks(n), 256, 0, s>>>(keep, pos, n, L, nf, d_w, anchor, tree, level, field, d_w_out);
  ++g_launches;
  TRY(cudaGetLastError());
  // the vforest: same trees, transfer and kind; leaves on the device (subset of an SFC-ordered forest)
  const int nctrl = f->surface ? 12 : (f->R + 1) * (f->R + 1) * (f->R + 1) * 3;
  std::vector<double> ctrl((size_t)f->K * nctrl);
  for (int k = 0; k < f->K; ++k) memcpy(&ctrl[(size_t)k * nctrl], f->h_trees[k].lagr, sizeof(double) * nctrl);
  rc_forest_desc d;
  memset(&d, 0, sizeof d);
  d.num_trees = f->K;
  d.geom_degree = f->R;
  d.tree_ctrl = ctrl.data();
  d.field_degree = f->P;
  d.num_leaves = m;
  d.first_global_leaf = first_global_leaf;
  d.leaf_anchor = anchor;
  d.leaf_tree = tree;
  d.leaf_level = level;
  d.leaf_field = field;
  d.memory = RC_DEVICE_COPY;
  d.transfer = f->transfer;
  d.dim = f->surface ? 2 : 3;
  d.surface = f->surf;
  st = rc_forest_create(&d, stream, out);
  TRY(cudaStreamSynchronize(s));
  release();
  return st;
#undef TRY
}

extern "C" rc_status rc_forest_leaves(rc_forest* f, int32_t* d_anchor, int32_t* d_tree, int8_t* d_level,
                                      float* d_field, int64_t capacity, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f) return rc_fail(RC_ERR_INVALID_ARG, "rc_forest_leaves: null forest");
  if (capacity < f->n)
    return rc_fail(RC_ERR_CAPACITY, "rc_forest_leaves: capacity %lld < %lld leaves", (long long)capacity,
                   (long long)f->n);
  cudaStream_t s = (cudaStream_t)stream;
  const int nf = f->surface ? 4 : (f->P + 1) * (f->P + 1) * (f->P + 1);
  if (d_anchor) CU(cudaMemcpyAsync(d_anchor, f->d_anchor, sizeof(int32_t) * 3 * f->n, cudaMemcpyDeviceToDevice, s));
  if (d_tree) CU(cudaMemcpyAsync(d_tree, f->d_tree, sizeof(int32_t) * f->n, cudaMemcpyDeviceToDevice, s));
  if (d_level) CU(cudaMemcpyAsync(d_level, f->d_level, f->n, cudaMemcpyDeviceToDevice, s));
  if (d_field) {
    if (!f->has_field) return rc_fail(RC_ERR_STATE, "rc_forest_leaves: keys-only forest has no field");
    CU(cudaMemcpyAsync(d_field, f->d_field, sizeof(float) * nf * f->n, cudaMemcpyDeviceToDevice, s));
  }
  return RC_OK;
}
