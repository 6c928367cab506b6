// rc_api.cu -- host side of the C ABI declared in include/rc.h.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "rc_internal.cuh"

namespace rc {
std::atomic<int64_t> g_launches{0};
}
using namespace rc;

static thread_local char g_err[1024] = "";

namespace rc {
rc_status rc_fail(rc_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return st;
}
}  // namespace rc
#define fail rc_fail

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? RC_ERR_OUT_OF_MEMORY : RC_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                               \
  } while (0)

#define LAUNCHED() (++g_launches)

extern "C" const char* rc_last_error(void) { return g_err; }
extern "C" int32_t rc_version(void) { return 4; }
extern "C" int64_t rc_launch_count(int32_t reset) {
  const int64_t v = reset ? g_launches.exchange(0) : g_launches.load();
  return v;
}

template <typename T>
static cudaError_t grow(T** p, int64_t* cap, int64_t need, cudaStream_t s) {
  if (need <= *cap && *p) return cudaSuccess;
  if (*p) dfree(*p, s);
  *p = nullptr;
  int64_t c = std::max<int64_t>(need + std::min<int64_t>(need / 8, (int64_t)1 << 24), 64);   // bounded slack
  cudaError_t e = dmalloc((void**)p, sizeof(T) * (size_t)c, s);
  if (e == cudaSuccess) *cap = c;
  else *cap = 0;
  return e;
}

// ---------------------------------------------------------------------------
// forest
// ---------------------------------------------------------------------------
static uint64_t spread18(uint32_t v) {
  uint64_t x = v & 0x3FFFFu, r = 0;
  for (int b = 0; b < 18; ++b) r |= ((x >> b) & 1ull) << (3 * b);
  return r;
}

extern "C" rc_status rc_forest_create(const rc_forest_desc* d, void* stream, rc_forest** out) {
  RC_NVTX("rc_forest_create");
  if (!d || !out) return fail(RC_ERR_INVALID_ARG, "rc_forest_create: null argument");
  *out = nullptr;
  if (d->num_trees < 1 || d->num_trees > RC_MAX_TREES) return fail(RC_ERR_INVALID_ARG, "num_trees out of range");
  if (d->dim != 0 && d->dim != 2 && d->dim != 3) return fail(RC_ERR_INVALID_ARG, "dim must be 0, 2 or 3");
  const bool surface = d->dim == 2;
  if (surface && (d->geom_degree != 1 || d->field_degree != 1))
    return fail(RC_ERR_INVALID_ARG, "surface forests take geom_degree = field_degree = 1 (bilinear patches)");
  if (d->geom_degree < 1 || d->geom_degree > 2) return fail(RC_ERR_INVALID_ARG, "geom_degree must be 1 or 2");
  if (d->field_degree < 1 || d->field_degree > 2) return fail(RC_ERR_INVALID_ARG, "field_degree must be 1 or 2");
  if (d->num_leaves < 1 || d->num_leaves > (int64_t)INT32_MAX) return fail(RC_ERR_INVALID_ARG, "num_leaves out of range");
  if (!d->tree_ctrl || !d->leaf_anchor || !d->leaf_tree || !d->leaf_level)
    return fail(RC_ERR_INVALID_ARG, "rc_forest_create: null array");
  if (d->memory != RC_HOST_COPY && d->memory != RC_DEVICE_COPY && d->memory != RC_HOST_COPY_TRUSTED &&
      d->memory != RC_DEVICE_BORROW)
    return fail(RC_ERR_INVALID_ARG, "bad memory mode");
  if (d->first_global_leaf < 0 || d->first_global_leaf + d->num_leaves > (int64_t)UINT32_MAX)
    return fail(RC_ERR_INVALID_ARG, "global leaf index must fit 32 bits");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = d->num_leaves;
  const int NF = surface ? 4 : (d->field_degree + 1) * (d->field_degree + 1) * (d->field_degree + 1);
  int n1 = d->geom_degree + 1;
  const int nctrl = surface ? 12 : n1 * n1 * n1 * 3;   // doubles per tree
  for (int q = 0; q < d->num_trees * nctrl; ++q)
    if (!isfinite(d->tree_ctrl[q])) return fail(RC_ERR_NUMERIC, "non-finite control point");
  if (d->memory == RC_HOST_COPY) {
    // strict SFC order: (tree, Morton key) increasing; anchors aligned to their level
    uint64_t prev_key = 0;
    int prev_tree = -1;
    for (int64_t e = 0; e < n; ++e) {
      int t = d->leaf_tree[e], l = d->leaf_level[e];
      if (t < 0 || t >= d->num_trees || l < 0 || l > RC_MAXLEVEL)
        return fail(RC_ERR_INVALID_ARG, "leaf %lld: bad tree or level", (long long)e);
      uint32_t mask = (1u << (RC_MAXLEVEL - l)) - 1u;
      const int32_t* a = d->leaf_anchor + 3 * e;
      for (int k = 0; k < 3; ++k)
        if (a[k] < 0 || a[k] >= (1 << RC_MAXLEVEL) || ((uint32_t)a[k] & mask))
          return fail(RC_ERR_INVALID_ARG, "leaf %lld: anchor not aligned to its level", (long long)e);
      if (surface && a[2] != 0) return fail(RC_ERR_INVALID_ARG, "leaf %lld: quadtree leaf with z anchor != 0", (long long)e);
      uint64_t key = spread18(a[0]) | (spread18(a[1]) << 1) | (spread18(a[2]) << 2);
      if (t < prev_tree || (t == prev_tree && key <= prev_key))
        return fail(RC_ERR_NOT_SFC_SORTED, "leaf %lld breaks SFC order", (long long)e);
      // non-overlap: previous leaf's last descendant key must be below this key
      prev_tree = t;
      prev_key = key | (spread18(mask) | (spread18(mask) << 1) | (spread18(mask) << 2));
    }
    if (d->leaf_field)
      for (int64_t q = 0; q < n * NF; ++q)
        if (!isfinite(d->leaf_field[q])) return fail(RC_ERR_NUMERIC, "non-finite field value");
  }
  rc_forest* f = new rc_forest();
  f->K = d->num_trees;
  f->R = d->geom_degree;
  f->P = d->field_degree;
  f->n = n;
  f->first_global = d->first_global_leaf;
  f->transfer = d->transfer;
  f->has_field = d->leaf_field != nullptr;
  f->borrowed = d->memory == RC_DEVICE_BORROW;
  f->last_stream = s;
  f->surface = surface;
  if (surface) f->surf = d->surface;
  f->h_trees = new TreeConst[f->K];
  memset(f->h_trees, 0, sizeof(TreeConst) * f->K);
  cudaError_t e = cudaSuccess;
  auto cleanup = [&](rc_status st, const char* what) {
    rc_status r = fail(st, "%s: %s", what, cudaGetErrorString(e));
    rc_forest_destroy(f);
    return r;
  };
#define ALLOC(ptr, bytes)                                        \
  if ((e = dmalloc((void**)&(ptr), (bytes), s)) != cudaSuccess) \
    return cleanup(RC_ERR_OUT_OF_MEMORY, "cudaMalloc " #ptr);
  if (f->borrowed) {   // the caller's device arrays in place (they outlive the forest)
    f->d_anchor = const_cast<int32_t*>(d->leaf_anchor);
    f->d_tree = const_cast<int32_t*>(d->leaf_tree);
    f->d_field = const_cast<float*>(d->leaf_field);
  } else {
    ALLOC(f->d_anchor, sizeof(int32_t) * 3 * n);
    ALLOC(f->d_tree, sizeof(int32_t) * n);
    if (f->has_field) ALLOC(f->d_field, sizeof(float) * NF * n);
  }
  // the 1-byte levels are always copied: k_prep_slots stages them in whole 4-byte words
  ALLOC(f->d_level, sizeof(int8_t) * ((n + 3) & ~(int64_t)3));
  ALLOC(f->d_flag, sizeof(int32_t) * n);
  ALLOC(f->d_rect_all, sizeof(Rect16) * n);
  ALLOC(f->d_scan, sizeof(int64_t) * (n + 1));
  ALLOC(f->d_vis, sizeof(int32_t) * n);
  ALLOC(f->d_vis_rect, sizeof(Rect16) * n);
  ALLOC(f->d_chunk_off, sizeof(int64_t) * (n + 1));
  ALLOC(f->d_counters, sizeof(int64_t) * CNT_TOTAL);
  ALLOC(f->d_trees, sizeof(TreeConst) * f->K);
  ALLOC(f->d_cam, sizeof(CamConst));
  f->scan_tmp_cap = std::max<int64_t>((int64_t)scan_tmp_size(n + 1) + 64, 256);
  ALLOC(f->d_scan_tmp, sizeof(int64_t) * f->scan_tmp_cap);
#undef ALLOC
  cudaMemcpyKind kind = (d->memory == RC_DEVICE_COPY || f->borrowed) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if ((!f->borrowed && (e = cudaMemcpyAsync(f->d_anchor, d->leaf_anchor, sizeof(int32_t) * 3 * n, kind, s))) ||
      (!f->borrowed && (e = cudaMemcpyAsync(f->d_tree, d->leaf_tree, sizeof(int32_t) * n, kind, s))) ||
      (e = cudaMemcpyAsync(f->d_level, d->leaf_level, sizeof(int8_t) * n, kind, s)) ||
      (!f->borrowed && f->has_field &&
       (e = cudaMemcpyAsync(f->d_field, d->leaf_field, sizeof(float) * NF * n, kind, s))) ||
      (e = cudaMemsetAsync(f->d_counters, 0, sizeof(int64_t) * CNT_TOTAL, s)))
    return cleanup(RC_ERR_CUDA, "cudaMemcpyAsync leaves");
  // host copy of the tree control points for rc_camera_set
  for (int k = 0; k < f->K; ++k)
    memcpy(f->h_trees[k].lagr, d->tree_ctrl + (size_t)k * nctrl, sizeof(double) * nctrl);
  if ((e = cudaEventCreate(&f->ev0)) || (e = cudaEventCreate(&f->ev1))) return cleanup(RC_ERR_CUDA, "event");
  for (int k = 0; k < 3; ++k)
    if ((e = cudaEventCreate(&f->evc[k]))) return cleanup(RC_ERR_CUDA, "event");
  if ((e = cudaStreamSynchronize(s))) return cleanup(RC_ERR_CUDA, "sync");
  if ((e = build_node_levels(f, s))) return cleanup(RC_ERR_CUDA, "node levels");
  *out = f;
  return RC_OK;
}

extern "C" rc_status rc_forest_destroy(rc_forest* f) {
  if (!f) return RC_OK;
  // blocks go back to the caching pool: no kernel may still use them.  One forest is driven from
  // one stream at a time (rc.h), so its last stream holds all its pending work.
  if (f->last_stream) cudaStreamSynchronize(f->last_stream);
  else cudaDeviceSynchronize();
  if (f->borrowed) f->d_anchor = f->d_tree = nullptr, f->d_field = nullptr;   // the caller's
  void* ptrs[] = {f->d_anchor, f->d_tree, f->d_level, f->d_field, f->d_flag, f->d_rect_all, f->d_scan,
                  f->d_vis, f->d_vis_rect, f->d_chunk_off, f->d_counters, f->d_trees, f->d_cam,
                  f->d_scan_tmp, f->d_chunk_elem, f->d_segs, f->d_hits_pp, f->d_pix_cnt, f->d_pix_off,
                  f->d_perm, f->d_send, f->d_items, f->d_leaf_nodes[0], f->d_leaf_nodes[1], f->d_ucnt, f->d_uend, f->d_units,
                  f->d_scratch, f->d_segs2, f->d_uoff, f->d_defer, f->d_sorted, f->d_tiles, f->d_xcnt, f->d_recv, f->d_gslot, f->d_boff};
  for (void* p : ptrs)
    if (p) dfree(p, 0, true);
  for (int c = 0; c <= RC_NODE_LEVELS; ++c)
    if (f->d_node_first[c]) dfree(f->d_node_first[c], 0, true);
  if (f->ev0) cudaEventDestroy(f->ev0);
  if (f->ev1) cudaEventDestroy(f->ev1);
  for (int k = 0; k < 3; ++k)
    if (f->evc[k]) cudaEventDestroy(f->evc[k]);
  for (int k = 0; k < 4; ++k)
    if (f->evb[k]) cudaEventDestroy(f->evb[k]);
  for (cudaEvent_t ev : f->evk)
    if (ev) cudaEventDestroy(ev);
  if (f->h_tiles) cudaFreeHost(f->h_tiles);
  if (f->h_xcnt) cudaFreeHost(f->h_xcnt);
  if (f->h_trees_pin) cudaFreeHost(f->h_trees_pin);
  if (f->graph_exec) cudaGraphExecDestroy(f->graph_exec);
  if (f->cap_stream) cudaStreamDestroy(f->cap_stream);
  delete[] f->h_trees;
  delete f;
  return RC_OK;
}

// ---------------------------------------------------------------------------
// camera (host fp64 preprocessing)
// ---------------------------------------------------------------------------
// Gauss-Legendre nodes/weights on [0,1] and the table S_jk = int_0^{u_j} l_k
// (SURVEY R13), computed in long double: Newton on P_N from Tricomi's
// initial guess; S by exact integration of the monomial form of l_k.
static void gl_tables(int N, float* u, float* w, float* S) {
  long double x[RC_MAX_N], wx[RC_MAX_N];
  const long double PI = 3.141592653589793238462643383279502884L;
  for (int i = 1; i <= N; ++i) {
    long double z = (1.0L - (N - 1.0L) / (8.0L * N * N * N)) * cosl(PI * (4.0L * i - 1.0L) / (4.0L * N + 2.0L));
    long double dp = 1.0L;
    for (int it = 0; it < 200; ++it) {
      long double p0 = 1.0L, p1 = z;
      for (int k = 2; k <= N; ++k) {
        long double p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (N == 1) p0 = 1.0L;
      dp = N * (z * p1 - p0) / (z * z - 1.0L);
      long double dz = p1 / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    // z descends with i; map to ascending u = (1 + x)/2 with x = -z
    x[i - 1] = -z;
    wx[i - 1] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
  long double uu[RC_MAX_N];
  for (int j = 0; j < N; ++j) {
    uu[j] = 0.5L * (1.0L + x[j]);
    u[j] = (float)uu[j];
    w[j] = (float)(0.5L * wx[j]);
  }
  for (int k = 0; k < N; ++k) {
    long double c[RC_MAX_N + 1] = {1.0L};
    int deg = 0;
    long double denom = 1.0L;
    for (int m = 0; m < N; ++m) {
      if (m == k) continue;
      for (int q = deg + 1; q >= 1; --q) c[q] = c[q - 1] - uu[m] * c[q];
      c[0] = -uu[m] * c[0];
      ++deg;
      denom *= (uu[k] - uu[m]);
    }
    for (int j = 0; j < N; ++j) {
      long double acc = 0.0L, pw = uu[j];
      for (int q = 0; q <= deg; ++q) {
        acc += c[q] * pw / (q + 1);
        pw *= uu[j];
      }
      S[j * RC_MAX_N + k] = (float)(acc / denom);
    }
  }
}

static void mat3_inv(const double A[9], double inv[9], double* det_out) {
  double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
               A[2] * (A[3] * A[7] - A[4] * A[6]);
  *det_out = det;
  inv[0] = (A[4] * A[8] - A[5] * A[7]) / det;
  inv[1] = (A[2] * A[7] - A[1] * A[8]) / det;
  inv[2] = (A[1] * A[5] - A[2] * A[4]) / det;
  inv[3] = (A[5] * A[6] - A[3] * A[8]) / det;
  inv[4] = (A[0] * A[8] - A[2] * A[6]) / det;
  inv[5] = (A[2] * A[3] - A[0] * A[5]) / det;
  inv[6] = (A[3] * A[7] - A[4] * A[6]) / det;
  inv[7] = (A[1] * A[6] - A[0] * A[7]) / det;
  inv[8] = (A[0] * A[4] - A[1] * A[3]) / det;
}

extern "C" rc_status rc_camera_set(rc_forest* f, const rc_camera* cam, void* stream) {
  RC_NVTX("rc_camera_set");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !cam) return fail(RC_ERR_INVALID_ARG, "rc_camera_set: null argument");
  auto dot = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
  double n = sqrt(dot(cam->view, cam->view));
  if (cam->projection != RC_PERSPECTIVE && cam->projection != RC_ORTHOGRAPHIC)
    return fail(RC_ERR_INVALID_ARG, "bad projection");
  if (!(n > 0) || fabs(dot(cam->right, cam->right) - 1) > 1e-9 || fabs(dot(cam->up, cam->up) - 1) > 1e-9 ||
      fabs(dot(cam->right, cam->up)) > 1e-9 || fabs(dot(cam->right, cam->view)) > 1e-9 * n ||
      fabs(dot(cam->up, cam->view)) > 1e-9 * n)
    return fail(RC_ERR_INVALID_ARG, "camera frame (t,u,v) not orthonormal");
  if (cam->projection == RC_ORTHOGRAPHIC && fabs(n - 1.0) > 1e-9)
    return fail(RC_ERR_INVALID_ARG, "orthographic view direction must be a unit vector");
  if (!(cam->far_dist > (cam->projection == RC_PERSPECTIVE ? n : 0.0)))
    return fail(RC_ERR_INVALID_ARG, "far distance must exceed the near distance");
  if (cam->width < 1 || cam->height < 1 || cam->width > 32767 || cam->height > 32767)
    return fail(RC_ERR_INVALID_ARG, "image size out of range");
  if (cam->gl_points < 1 || cam->gl_points > RC_MAX_N) return fail(RC_ERR_INVALID_ARG, "gl_points must be 1..8");
  if (!(cam->pixel_size > 0)) return fail(RC_ERR_INVALID_ARG, "pixel_size must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  f->cam = *cam;
  CamConst& c = f->cc;
  memset(&c, 0, sizeof c);
  c.proj = cam->projection;
  c.W = cam->width;
  c.H = cam->height;
  c.N = cam->gl_points;
  c.newton_max = cam->newton_max_iter > 0 ? cam->newton_max_iter : 20;
  c.newton_tol = (float)(cam->newton_tol > 0 ? cam->newton_tol : 1e-6);
  if (cam->scheme < RC_SCHEME_GL || cam->scheme > RC_SCHEME_SIMPSON)
    return fail(RC_ERR_INVALID_ARG, "scheme must be one of RC_SCHEME_*");
  if (!(cam->c_rk >= 0.0) || cam->max_depth < 0 || cam->max_depth > 24)
    return fail(RC_ERR_INVALID_ARG, "c_rk must be >= 0 and max_depth in [0, 24]");
  c.scheme = cam->scheme;
  c.c_rk = (float)cam->c_rk;
  c.max_depth = cam->max_depth > 0 ? cam->max_depth : 24;
  c.n = n;
  c.ell = cam->pixel_size;
  c.far_dist = cam->far_dist;
  for (int k = 0; k < 3; ++k) {
    c.cam_rot[k] = cam->right[k];
    c.cam_rot[3 + k] = cam->up[k];
    c.cam_rot[6 + k] = cam->view[k] / n;
    c.cam_org[k] = cam->origin[k];
    if (cam->projection == RC_PERSPECTIVE) {
      c.O0[k] = cam->origin[k];
      c.Ot[k] = c.Ou[k] = 0.0;
      c.R0[k] = cam->view[k];
      c.Rt[k] = cam->pixel_size * cam->right[k];
      c.Ru[k] = cam->pixel_size * cam->up[k];
    } else {
      c.O0[k] = cam->origin[k];
      c.Ot[k] = cam->pixel_size * cam->right[k];
      c.Ou[k] = cam->pixel_size * cam->up[k];
      c.R0[k] = cam->view[k];
      c.Rt[k] = c.Ru[k] = 0.0;
    }
  }
  if (cam->projection == RC_PERSPECTIVE) {
    c.amin = 1.0;
    c.amax = cam->far_dist / n;
  } else {
    c.amin = 0.0;
    c.amax = cam->far_dist;
  }
  gl_tables(c.N, c.u, c.w, c.S);
  for (int k = 0; k < 3; ++k) {
    c.f_R0[k] = (float)c.R0[k];
    c.f_Rt[k] = (float)c.Rt[k];
    c.f_Ru[k] = (float)c.Ru[k];
    c.f_Ot[k] = (float)c.Ot[k];
    c.f_Ou[k] = (float)c.Ou[k];
  }
  c.kappa0 = f->transfer.kappa0;
  c.inv_F = f->transfer.inv_F;
  c.q0 = f->transfer.q0;

  c.surf = f->surf;
  if (f->surface) {   // bilinear patches: world and camera-space corners [m2][m1][xyz]
    f->all_affine = 0;
    for (int k = 0; k < f->K; ++k) {
      TreeConst& T = f->h_trees[k];
      T.affine = 0;
      memcpy(T.Bw, T.lagr, sizeof(double) * 12);
      for (int m = 0; m < 4; ++m)
        for (int r = 0; r < 3; ++r) {
          double acc = 0.0;
          for (int q = 0; q < 3; ++q) acc += c.cam_rot[3 * r + q] * (T.lagr[3 * m + q] - c.cam_org[q]);
          T.Bc[3 * m + r] = acc;
        }
    }
    CU(cudaMemcpyAsync(f->d_trees, f->h_trees, sizeof(TreeConst) * f->K, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(f->d_cam, &f->cc, sizeof(CamConst), cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    f->have_camera = true;
    f->have_cull = f->have_cast = false;
    return RC_OK;
  }
  // per tree: affine detection, affine ray constants, Bernstein points
  const int R = f->R, n1 = R + 1, NP = n1 * n1 * n1;
  const double eta2[3] = {0.0, 0.5, 1.0};
  f->all_affine = 1;
  for (int k = 0; k < f->K; ++k) {
    TreeConst& T = f->h_trees[k];
    const double* lagcopy = T.lagr;
    // affine test: z_m == c + M eta_m
    const double* eta = R == 1 ? nullptr : eta2;
    auto node = [&](int m) { return R == 1 ? (double)m : eta[m]; };
    double cc0[3], M[9];
    for (int q = 0; q < 3; ++q) cc0[q] = lagcopy[q];
    for (int d = 0; d < 3; ++d) {
      int m[3] = {0, 0, 0};
      m[d] = R;   // the node at t_d = 1
      int idx = (m[2] * n1 + m[1]) * n1 + m[0];
      for (int q = 0; q < 3; ++q) M[q * 3 + d] = lagcopy[idx * 3 + q] - cc0[q];
    }
    int affine = 1;
    double scale = 1.0;
    for (int q = 0; q < NP * 3; ++q) scale = std::max(scale, fabs(lagcopy[q]));
    for (int m3 = 0; m3 < n1; ++m3)
      for (int m2 = 0; m2 < n1; ++m2)
        for (int m1 = 0; m1 < n1; ++m1) {
          int idx = (m3 * n1 + m2) * n1 + m1;
          double t[3] = {node(m1), node(m2), node(m3)};
          for (int q = 0; q < 3; ++q) {
            double v = cc0[q] + M[q * 3] * t[0] + M[q * 3 + 1] * t[1] + M[q * 3 + 2] * t[2];
            if (fabs(v - lagcopy[idx * 3 + q]) > 1e-13 * scale) affine = 0;
          }
        }
    double Minv[9], det = 0.0;
    mat3_inv(M, Minv, &det);
    if (!(fabs(det) > 0) || !isfinite(det)) affine = 0;
    T.affine = affine;
    if (!affine) f->all_affine = 0;
    auto mv = [&](const double* A, const double* x, double* y) {
      for (int r = 0; r < 3; ++r) y[r] = A[3 * r] * x[0] + A[3 * r + 1] * x[1] + A[3 * r + 2] * x[2];
    };
    if (affine) {
      double tmp[3];
      for (int q = 0; q < 3; ++q) tmp[q] = c.O0[q] - cc0[q];
      mv(Minv, tmp, T.TO0);
      mv(Minv, c.Ot, T.TOt);
      mv(Minv, c.Ou, T.TOu);
      mv(Minv, c.R0, T.TR0);
      mv(Minv, c.Rt, T.TRt);
      mv(Minv, c.Ru, T.TRu);
      // camera-space affine map of the tree: X = rot (c + M t - org)
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q)
          T.Acam[3 * r + q] = c.cam_rot[3 * r] * M[q] + c.cam_rot[3 * r + 1] * M[3 + q] + c.cam_rot[3 * r + 2] * M[6 + q];
      for (int q = 0; q < 3; ++q) tmp[q] = cc0[q] - c.cam_org[q];
      mv(c.cam_rot, tmp, T.bcam);
    }
    // Bernstein control points of J_k (Lagrange -> Bernstein per axis, R=2)
    double B[81];
    memcpy(B, lagcopy, sizeof(double) * NP * 3);
    if (R == 2) {
      for (int ax = 0; ax < 3; ++ax)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            int id[3];
            for (int m = 0; m < 3; ++m) {
              int cidx[3];
              cidx[ax] = m;
              cidx[(ax + 1) % 3] = a;
              cidx[(ax + 2) % 3] = b;
              id[m] = (cidx[2] * 3 + cidx[1]) * 3 + cidx[0];
            }
            for (int q = 0; q < 3; ++q) B[id[1] * 3 + q] = 2.0 * B[id[1] * 3 + q] - 0.5 * (B[id[0] * 3 + q] + B[id[2] * 3 + q]);
          }
    }
    memcpy(T.Bw, B, sizeof(double) * NP * 3);
    for (int m = 0; m < NP; ++m) {
      double tmp[3] = {B[3 * m] - c.cam_org[0], B[3 * m + 1] - c.cam_org[1], B[3 * m + 2] - c.cam_org[2]};
      mv(c.cam_rot, tmp, &T.Bc[3 * m]);
    }
  }
  CU(cudaMemcpyAsync(f->d_trees, f->h_trees, sizeof(TreeConst) * f->K, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(f->d_cam, &f->cc, sizeof(CamConst), cudaMemcpyHostToDevice, s));
  // host buffers are pageable: make the copies complete before the host
  // structures can change again (a few KB)
  CU(cudaStreamSynchronize(s));
  f->have_camera = true;
  f->have_cull = f->have_cast = false;
  return RC_OK;
}

// ---------------------------------------------------------------------------
// cull + pair generation
// ---------------------------------------------------------------------------
static DevLeafView leaf_view(rc_forest* f) { return DevLeafView{f->d_anchor, f->d_tree, f->d_level, f->d_field}; }

static unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

extern "C" rc_status rc_cull(rc_forest* f, void* stream, int64_t* d_num_visible) {
  RC_NVTX("rc_cull");
  if (!f) return fail(RC_ERR_INVALID_ARG, "rc_cull: null forest");
  if (!f->have_camera) return fail(RC_ERR_STATE, "rc_cull before rc_camera_set");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n;
  DevLeafView L = leaf_view(f);
  if (f->surface) CU(launch_cull_surface(f->cc, f->d_trees, L, n, f->d_flag, f->d_rect_all, s));
  else CU(launch_cull(f->cc, f->d_trees, L, n, f->R, f->all_affine != 0, f->d_flag, f->d_rect_all, s));
  CU(scan_exclusive<int32_t>(f->d_flag, f->d_scan, n, f->d_scan_tmp, s));
  CU(launch_compact(f->d_flag, f->d_rect_all, f->d_scan, n, f->d_vis, f->d_vis_rect, s));
  // pair generation: chunk counts over all n slots (entries >= nvis are 0)
  CU(cudaMemsetAsync(f->d_counters, 0, sizeof(int64_t) * CNT_TOTAL, s));
  CU(cudaMemsetAsync(f->d_chunk_off, 0, sizeof(int64_t) * (n + 1), s));
  CU(launch_chunk_count(f->d_vis_rect, f->d_scan + n, n, f->d_chunk_off, f->d_counters, s));
  // in-place exclusive scan of the counts (each scan thread reads its items before writing them)
  CU(scan_exclusive<int64_t>(f->d_chunk_off, f->d_chunk_off, n, f->d_scan_tmp, s));
  if (d_num_visible) CU(cudaMemcpyAsync(d_num_visible, f->d_scan + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  f->have_cull = true;
  f->have_cast = false;
  return RC_OK;
}

extern "C" rc_status rc_leaf_weights(rc_forest* f, int64_t* d_w, int64_t capacity, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !d_w) return fail(RC_ERR_INVALID_ARG, "rc_leaf_weights: null argument");
  if (!f->have_cull) return fail(RC_ERR_STATE, "rc_leaf_weights before rc_cull");
  if (capacity < f->n) return fail(RC_ERR_CAPACITY, "rc_leaf_weights: capacity %lld < %lld leaves",
                                   (long long)capacity, (long long)f->n);
  CU(launch_leaf_weights(f->d_flag, f->d_rect_all, f->n, d_w, (cudaStream_t)stream));
  return RC_OK;
}

extern "C" rc_status rc_cull_result(rc_forest* f, int32_t* d_visible, int64_t capacity, int64_t* count, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !count) return fail(RC_ERR_INVALID_ARG, "rc_cull_result: null argument");
  if (!f->have_cull) return fail(RC_ERR_STATE, "rc_cull_result before rc_cull");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nv = 0;
  CU(cudaMemcpyAsync(&nv, f->d_scan + f->n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *count = nv;
  if (nv > capacity) return fail(RC_ERR_CAPACITY, "rc_cull_result: capacity %lld < %lld", (long long)capacity, (long long)nv);
  if (nv > 0 && d_visible) CU(cudaMemcpyAsync(d_visible, f->d_vis, sizeof(int32_t) * nv, cudaMemcpyDeviceToDevice, s));
  CU(cudaStreamSynchronize(s));
  return RC_OK;
}

// ---------------------------------------------------------------------------
// cast
// ---------------------------------------------------------------------------
static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static rc_status aggregate_to(rc_forest* f, int level, cudaStream_t s);

extern "C" rc_status rc_cast_segments(rc_forest* f, int32_t fold_levels, void* stream) {
  RC_NVTX("rc_cast_segments");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f) return fail(RC_ERR_INVALID_ARG, "rc_cast_segments: null forest");
  if (!f->have_cull) return fail(RC_ERR_STATE, "rc_cast_segments before rc_cull");
  if (!f->has_field) return fail(RC_ERR_STATE, "rc_cast_segments on a forest without a field (keys only)");
  if (fold_levels < 0 || fold_levels > RC_NODE_LEVELS)
    return fail(RC_ERR_INVALID_ARG, "fold_levels must be in [0, %d]", RC_NODE_LEVELS);
  if (!f->all_affine && !f->surface && f->R != 2) return fail(RC_ERR_INVALID_ARG, "non-affine trees require geom_degree 2");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n;
  // one small readback to size the chunk map, the units and the record buffer
  int64_t hv[3];
  CU(cudaMemcpyAsync(&hv[0], f->d_scan + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&hv[1], f->d_chunk_off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&hv[2], f->d_counters + CNT_CANDIDATES, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  f->h_num_visible = hv[0];
  f->h_chunks = hv[1];
  f->h_candidates = hv[2];
  const int64_t cand = hv[2], nvis = hv[0];
  const int64_t npix = (int64_t)f->cc.W * f->cc.H;
  CU(grow(&f->d_chunk_elem, &f->chunk_cap, std::max<int64_t>(f->h_chunks, 1), s));
  CU(grow(&f->d_hits_pp, &f->pix_cap, npix, s));
  if (nvis > 0) CU(launch_expand(f->d_chunk_off, f->d_scan + n, nvis, f->d_chunk_elem, s));
  const bool curved = !f->all_affine && !f->surface;
  const uint32_t key_base = (uint32_t)f->first_global;
  // fold units (curved path): the visible leaves of every node of the fold
  // level (64-leaf windows without folding) cut into <= 64 leaves and
  // <= RC_UNIT_CHUNKS chunks
  int64_t nunits = 0;
  if (curved && nvis > 0) {
    const int32_t* leaf_node = nullptr;
    if (fold_levels > 0) CU(build_leaf_node(f, fold_levels, s, &leaf_node));
    const int32_t* node_first = fold_levels > 0 ? f->d_node_first[fold_levels] : nullptr;
    if (!f->d_ucnt) {
      CU(dmalloc((void**)&f->d_ucnt, sizeof(int32_t) * (n + 1), s));
      CU(dmalloc((void**)&f->d_uoff, sizeof(int64_t) * (n + 1), s));
      CU(dmalloc((void**)&f->d_uend, sizeof(int32_t) * (n + 1), s));
    }
    CU(launch_units(f->d_vis, f->d_scan + n, nvis, leaf_node, node_first, f->d_chunk_off, f->d_ucnt, f->d_uoff,
                    f->d_uend, f->d_scan_tmp, key_base, nullptr, false, s));
    CU(cudaMemcpyAsync(&nunits, f->d_uoff + nvis, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    CU(grow(&f->d_units, &f->units_cap, std::max<int64_t>(nunits, 1), s));
    CU(launch_units(f->d_vis, f->d_scan + n, nvis, leaf_node, node_first, f->d_chunk_off, f->d_ucnt, f->d_uoff,
                    f->d_uend, f->d_scan_tmp, key_base, f->d_units, true, s));
  }
  f->h_units = curved ? nunits : 0;
  const int grid_curved = sm_count() * cast_curved_ctas_per_sm();
  if (curved && !f->d_scratch) {
    f->scratch_bytes = cast_curved_scratch_per_cta() * (size_t)grid_curved;
    CU(dmalloc((void**)&f->d_scratch, f->scratch_bytes, s));
  }
  // record capacity: the previous frame's count, else an estimate; a too
  // small buffer is grown to the exact count and the cast repeated
  // reuse the larger of the two record buffers (aggregation swaps them)
  if (f->seg2_cap > f->seg_cap) {
    std::swap(f->d_segs, f->d_segs2);
    std::swap(f->seg_cap, f->seg2_cap);
  }
  // first-frame estimate (C3-C5: fold-2 records are 1/7..1/4 of the candidates,
  // raw segments ~1/2), capped by the free device memory less what the
  // element slots and the aggregation / composite buffers need (the slots'
  // batch, 1/8 of the estimate and 2 GB), so that a forest near the memory
  // limit falls back to the exact regrowth instead of failing.  A short
  // buffer costs a second cast (C5's first frame: 5.1 s instead of 2.7 s with
  // a cap of half the free memory).
  int64_t est = curved ? (fold_levels > 0 ? cand / 4 : cand / 2 + cand / 8) : cand;
  if (f->h_cast_total > 0) est = 0;   // later frames: the previous count (+1/8), exact regrowth if short
  else {
    const size_t free_b = device_free_bytes();
    if (free_b > 0) {
      const int64_t slot_b = curved ? (int64_t)slot_record_bytes() *
                                          std::min<int64_t>(nvis + RC_UNIT_LEAVES, RC_SLOT_BATCH + RC_UNIT_LEAVES)
                                    : 0;
      const int64_t avail = (int64_t)free_b - slot_b - ((int64_t)2 << 30);
      const int64_t cap = std::max<int64_t>(avail / (int64_t)(sizeof(rc_seg) + sizeof(rc_seg) / 8), 0) + f->seg_cap;
      est = std::min(est, std::max<int64_t>(cap, (int64_t)(free_b / 2 / sizeof(rc_seg)) + f->seg_cap));
    }
  }
  int64_t need = std::max<int64_t>(f->h_cast_total + f->h_cast_total / 32, est) + 4096;
  CU(grow(&f->d_segs, &f->seg_cap, need, s));
  // element slots (k_prep_slots): the visible list in batches of at most
  // RC_SLOT_BATCH leaves (+ one unit window of margin), sized after the
  // records from the memory left (at least 1M leaves per batch)
  if (curved) {
    int64_t want = std::min<int64_t>(nvis + RC_UNIT_LEAVES, RC_SLOT_BATCH + RC_UNIT_LEAVES);
    if (f->slot_cap < want) {
      const size_t free_b = device_free_bytes();
      if (free_b > 0) {
        const int64_t fit = (int64_t)(free_b / 3 / slot_record_bytes());
        want = std::max<int64_t>(std::min(want, fit), std::min<int64_t>(want, ((int64_t)1 << 20) + RC_UNIT_LEAVES));
      }
    }
    if (f->slot_cap < want) {
      if (f->d_gslot) dfree(f->d_gslot, s);
      f->d_gslot = nullptr;
      f->slot_cap = 0;
      CU(dmalloc((void**)&f->d_gslot, slot_record_bytes() * (size_t)want, s));
      f->slot_cap = want;
    }
  }
  const int64_t batch = std::max<int64_t>(f->slot_cap - RC_UNIT_LEAVES, 1);
  for (int attempt = 0; attempt < 2; ++attempt) {
    CU(cudaMemsetAsync(f->d_hits_pp, 0, sizeof(int32_t) * npix, s));
    CU(cudaMemsetAsync(f->d_counters + CNT_SEGS, 0, sizeof(int64_t) * 3, s));
    CU(cudaMemsetAsync(f->d_counters + CNT_OVERFLOW, 0, sizeof(int64_t) * 3, s));
    CU(cudaMemsetAsync(f->d_counters + CNT_UNITS, 0, sizeof(int64_t) * 6, s));
    CU(cudaMemsetAsync(f->d_counters + CNT_DEPTH_CAP, 0, sizeof(int64_t), s));
    CU(cudaEventRecord(f->ev0, s));
    // per-launch events: the segment kernel alone (bench roofline) and the element preparation
    f->evk_used = 0;
    auto mark = [&](int k) -> cudaError_t {
      if (f->evk_used >= rc_forest::kEvBatches) return cudaSuccess;
      cudaEvent_t& ev = f->evk[4 * f->evk_used + k];
      if (!ev) {
        cudaError_t e = cudaEventCreate(&ev);
        if (e != cudaSuccess) return e;
      }
      return cudaEventRecord(ev, s);
    };
    if (f->h_chunks > 0) {
      if (f->surface) {
        CU(mark(0));
        CU(launch_cast_surface(f->cc, f->d_trees, leaf_view(f), f->d_vis, f->d_vis_rect, f->d_chunk_off,
                               f->d_chunk_elem, f->h_chunks, key_base, f->d_segs, f->seg_cap, f->d_hits_pp,
                               f->d_counters, sm_count() * 8, s));
        CU(mark(1));
        ++f->evk_used;
      } else if (!curved) {
        CU(mark(0));
        CU(launch_cast_affine(f->cc, f->d_trees, leaf_view(f), f->P, f->d_vis, f->d_vis_rect, f->d_chunk_off,
                              f->d_chunk_elem, f->h_chunks, key_base, f->d_segs, f->seg_cap, f->d_hits_pp,
                              f->d_counters, sm_count() * 8, s));
        CU(mark(1));
        ++f->evk_used;
      } else {
        char* gslot = reinterpret_cast<char*>(f->d_gslot);
        char* gorg = gslot + (size_t)f->slot_cap * (slot_record_bytes() - 32);
        for (int64_t v0 = 0; v0 < nvis; v0 += batch) {
          const int64_t v1 = std::min(nvis, v0 + batch);
          CU(cudaMemsetAsync(f->d_counters + CNT_UNITS, 0, sizeof(int64_t), s));
          CU(mark(2));
          CU(launch_prep_slots(f->d_trees, leaf_view(f), f->P, f->d_vis, f->d_scan + n, v0,
                               std::min(nvis, v1 + RC_UNIT_LEAVES), gslot, gorg, s));
          CU(mark(3));
          CU(mark(0));
          CU(launch_cast_curved(f->cc, f->d_trees, leaf_view(f), f->P, f->d_vis, f->d_vis_rect, f->d_chunk_off,
                                f->d_chunk_elem, f->d_units, nunits, fold_levels, key_base, f->d_scratch,
                                f->d_segs, f->seg_cap, f->d_hits_pp, f->d_counters, grid_curved, gslot, gorg, v0,
                                v1, s));
          CU(mark(1));
          if (f->evk_used < rc_forest::kEvBatches) ++f->evk_used;
          else f->evk_used = rc_forest::kEvBatches + 1;   // too many batches to time: report -1
        }
      }
    }
    CU(cudaEventRecord(f->ev1, s));
    int64_t c[2];
    CU(cudaMemcpyAsync(c, f->d_counters + CNT_SEGS, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(c + 1, f->d_counters + CNT_OVERFLOW, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    f->h_seg_total = c[0];
    f->h_cast_total = c[0];
    if (c[0] <= f->seg_cap && c[1] == 0) break;
    if (attempt == 1) return fail(RC_ERR_CAPACITY, "segment records overflow after regrowth");
    CU(grow(&f->d_segs, &f->seg_cap, c[0] + c[0] / 16 + 4096, s));
  }
  float ms = 0.0f;
  CU(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
  f->phase_ms[1] = ms;
  f->phase_ms[2] = 0.0f;
  f->rec_level = 0;
  if (!curved) f->h_raw_affine = f->h_seg_total;   // affine and surface kernels write unfolded records
  f->timed = true;
  f->have_cast = true;
  if (curved) {
    f->rec_level = fold_levels;
  } else if (fold_levels > 0) {
    // affine path: segments are written per leaf; fold them to the node level
    rc_status st = aggregate_to(f, fold_levels, s);
    if (st) return st;
  }
  return RC_OK;
}

extern "C" float rc_last_cast_ms(rc_forest* f) {
  if (!f || !f->timed) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(f->ev1) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, f->ev0, f->ev1) != cudaSuccess) return -1.0f;
  return ms;
}

extern "C" float rc_last_phase_ms(rc_forest* f, int32_t phase) {
  if (!f) return -1.0f;
  if (phase == 6 || phase == 7) {   // segment kernel launches alone / element preparation launches
    if (!f->timed || f->evk_used <= 0 || f->evk_used > rc_forest::kEvBatches) return -1.0f;
    if (cudaEventSynchronize(f->ev1) != cudaSuccess) return -1.0f;
    float tot = 0.0f;
    for (int b = 0; b < f->evk_used; ++b) {
      const int k = phase == 6 ? 0 : 2;
      if (!f->evk[4 * b + k] || !f->evk[4 * b + k + 1]) continue;
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, f->evk[4 * b + k], f->evk[4 * b + k + 1]) != cudaSuccess) return -1.0f;
      tot += ms;
    }
    return tot;
  }
  if (phase == 3) return (float)f->last_composite_copy;
  if (phase == 4 || phase == 5) {   // composite: bucketing (hist, scan, scatter) / fold kernels
    if (!f->composite_timed || cudaEventSynchronize(f->evc[2]) != cudaSuccess) return -1.0f;
    float ms = -1.0f;
    if (cudaEventElapsedTime(&ms, f->evc[phase - 4], f->evc[phase - 3]) != cudaSuccess) return -1.0f;
    return ms;
  }
  if (!f->timed) return -1.0f;
  if (phase == 0 || phase == 1) return rc_last_cast_ms(f);
  if (phase == 2) return 0.0f;
  return -1.0f;
}

extern "C" rc_status rc_segments_get(rc_forest* f, rc_segments* out, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !out) return fail(RC_ERR_INVALID_ARG, "rc_segments_get: null argument");
  if (!f->have_cast) return fail(RC_ERR_STATE, "rc_segments_get before rc_cast_segments");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t c[CNT_TOTAL];
  CU(cudaMemcpyAsync(c, f->d_counters, sizeof(int64_t) * CNT_TOTAL, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  out->count = std::min<int64_t>(c[CNT_SEGS], f->seg_cap);
  out->candidates = c[CNT_CANDIDATES];
  out->hit_pairs = c[CNT_HITPAIRS];
  out->newton_failures = c[CNT_NEWTON_FAIL];
  out->face_failures = c[CNT_FACE_FAIL];
  out->num_visible = f->h_num_visible;
  out->raw_segments = (f->all_affine || f->surface) ? f->h_raw_affine : c[CNT_RAW];
  out->level = f->rec_level;
  out->units = f->h_units;
  out->unfolded_units = c[CNT_UNFOLDED];
  out->face_tasks = c[CNT_TASKS];
  out->fallback_tasks = c[CNT_FALLBACK];
  out->segs = f->d_segs;
  out->hits_per_pixel = f->d_hits_pp;
  out->depth_capped = c[CNT_DEPTH_CAP];
  if (c[CNT_OVERFLOW] > 0)
    return fail(RC_ERR_CAPACITY, "segment buffer overflow: %lld records dropped", (long long)c[CNT_OVERFLOW]);
  return RC_OK;
}

// ---------------------------------------------------------------------------
// pack + composite
// ---------------------------------------------------------------------------
static rc_status check_tiling(rc_forest* f, const rc_tiling* t) {
  if (!t) return fail(RC_ERR_INVALID_ARG, "null tiling");
  if (t->tiles_x < 1 || t->tiles_y < 1 || f->cc.W % t->tiles_x || f->cc.H % t->tiles_y)
    return fail(RC_ERR_INVALID_ARG, "tiles must divide the image");
  if (t->nranks < 1 || t->nranks > RC_MAX_RANKS || t->rank < 0 || t->rank >= t->nranks)
    return fail(RC_ERR_INVALID_ARG, "bad nranks/rank");
  return RC_OK;
}

// K5: the current records permuted by owner rank into f->d_send on the
// device (counts in d_counters[CNT_SEND..], exclusive offsets in
// d_scan_tmp[0..nranks]); no host synchronisation.
static rc_status pack_device(rc_forest* f, const rc_tiling* t, cudaStream_t s) {
  const int tw = f->cc.W / t->tiles_x, th = f->cc.H / t->tiles_y;
  CU(grow(&f->d_send, &f->send_cap, std::max<int64_t>(f->seg_cap, 1), s));
  int64_t* d_cnt = f->d_counters + CNT_SEND;
  static_assert(CNT_TOTAL >= CNT_SEND + RC_MAX_RANKS, "counter space");
  int64_t* d_off = f->d_scan_tmp;
  int64_t* d_cursor = f->d_scan_tmp + 80;
  CU(cudaMemsetAsync(d_cnt, 0, sizeof(int64_t) * t->nranks, s));
  CU(cudaMemsetAsync(d_cursor, 0, sizeof(int64_t) * t->nranks, s));
  int64_t* d_nseg = f->d_counters + CNT_SEGS;
  const int grid = sm_count() * 4;
  CU(launch_pack(f->d_segs, d_nseg, f->cc.W, tw, th, t->tiles_x, t->nranks, d_cnt, nullptr, nullptr, nullptr, grid,
                 true, s));
  CU(launch_pack_offsets(d_cnt, t->nranks, d_off, s));
  CU(launch_pack(f->d_segs, d_nseg, f->cc.W, tw, th, t->tiles_x, t->nranks, nullptr, d_off, d_cursor, f->d_send,
                 grid, false, s));
  return RC_OK;
}

extern "C" rc_status rc_pack_tiles(rc_forest* f, const rc_tiling* t, int64_t* h_send_counts, const rc_seg** d_send,
                                   void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !h_send_counts || !d_send) return fail(RC_ERR_INVALID_ARG, "rc_pack_tiles: null argument");
  if (!f->have_cast) return fail(RC_ERR_STATE, "rc_pack_tiles before rc_cast_segments");
  rc_status st = check_tiling(f, t);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = pack_device(f, t, s))) return st;
  CU(cudaMemcpyAsync(h_send_counts, f->d_counters + CNT_SEND, sizeof(int64_t) * t->nranks, cudaMemcpyDeviceToHost,
                     s));
  CU(cudaStreamSynchronize(s));
  *d_send = f->d_send;
  return RC_OK;
}

extern "C" rc_status rc_composite_records(rc_forest* f, const rc_tiling* t, const rc_seg* d_recv, int64_t nrecv,
                                          const float background[3], float* d_rgba, int64_t capacity_floats,
                                          void* stream) {
  RC_NVTX("rc_composite_records");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !d_rgba) return fail(RC_ERR_INVALID_ARG, "rc_composite_records: null argument");
  if (!f->have_camera) return fail(RC_ERR_STATE, "rc_composite_records before rc_camera_set");
  if (nrecv < 0 || (nrecv > 0 && !d_recv)) return fail(RC_ERR_INVALID_ARG, "rc_composite_records: bad records");
  rc_status st = check_tiling(f, t);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int W = f->cc.W, H = f->cc.H;
  const int tw = W / t->tiles_x, th = H / t->tiles_y;
  std::vector<int32_t> mine;
  for (int ty = 0; ty < t->tiles_y; ++ty)
    for (int tx = 0; tx < t->tiles_x; ++tx)
      if ((tx + ty) % t->nranks == t->rank) mine.push_back(ty * t->tiles_x + tx);
  const int64_t npix_out = (int64_t)mine.size() * tw * th;
  if (capacity_floats < 4 * npix_out)
    return fail(RC_ERR_CAPACITY, "rc_composite: need %lld floats", (long long)(4 * npix_out));
  const rc_seg* src = d_recv;
  int64_t nsrc = nrecv;
  if (!src) {
    if (!f->have_cast) return fail(RC_ERR_STATE, "rc_composite: no segments");
    int64_t c = 0;
    CU(cudaMemcpyAsync(&c, f->d_counters + CNT_SEGS, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    src = f->d_segs;
    nsrc = std::min(c, f->seg_cap);
  }
  const int64_t npix = (int64_t)W * H;
  // (re)allocate per-pixel arrays sized to the image
  if (!f->d_pix_cnt || f->pix_cnt_cap < npix) {
    if (f->d_pix_cnt) dfree(f->d_pix_cnt, s);
    if (f->d_pix_off) dfree(f->d_pix_off, s);
    f->d_pix_cnt = nullptr;
    f->d_pix_off = nullptr;
    CU(dmalloc((void**)&f->d_pix_cnt, sizeof(int32_t) * (npix + 2), s));   // also the band counts (<= npix/32 + 1)
    CU(dmalloc((void**)&f->d_pix_off, sizeof(int64_t) * (npix + 1), s));
    f->pix_cnt_cap = npix;
  }
  int64_t need_tmp = (int64_t)scan_tmp_size(npix + 1) + 128;
  if (need_tmp > f->scan_tmp_cap) CU(grow(&f->d_scan_tmp, &f->scan_tmp_cap, need_tmp, s));
  if (nsrc >= (int64_t)UINT32_MAX) return fail(RC_ERR_CAPACITY, "more than 2^32 records in one composite");
  // pixel-sorted copy of the records when memory allows (contiguous reads in
  // the fold), else a permutation of record indices
  bool copy = false;
  {
    const size_t have = f->sorted_cap >= nsrc ? (size_t)-1 : 0;
    if (have || device_free_bytes() > (size_t)nsrc * sizeof(rc_seg) + ((size_t)2 << 30))
      copy = grow(&f->d_sorted, &f->sorted_cap, std::max<int64_t>(nsrc, 1), s) == cudaSuccess;
  }
  f->last_composite_copy = copy ? 1 : 0;
  if (!copy) CU(grow(&f->d_perm, &f->perm_cap, std::max<int64_t>(nsrc, 1), s));
  // the tile list lives on the device across frames: no per-frame allocation
  // or pageable copy (both stalled the host for tens of ms at times)
  const int32_t tkey[4] = {t->tiles_x, t->tiles_y, t->nranks, t->rank};
  if (memcmp(tkey, f->tiling_key, sizeof tkey) != 0) {
    const int64_t nt = std::max<int64_t>((int64_t)mine.size(), 1);
    CU(grow(&f->d_tiles, &f->tiles_cap, nt, s));
    if (f->h_tiles_cap < nt) {
      if (f->h_tiles) cudaFreeHost(f->h_tiles);
      f->h_tiles = nullptr;
      f->h_tiles_cap = 0;
      CU(cudaMallocHost((void**)&f->h_tiles, sizeof(int32_t) * nt));
      f->h_tiles_cap = nt;
    }
    if (!mine.empty()) {
      memcpy(f->h_tiles, mine.data(), sizeof(int32_t) * mine.size());
      CU(cudaMemcpyAsync(f->d_tiles, f->h_tiles, sizeof(int32_t) * mine.size(), cudaMemcpyHostToDevice, s));
      CU(cudaStreamSynchronize(s));   // h_tiles may be rewritten by the next call
    }
    memcpy(f->tiling_key, tkey, sizeof tkey);
  }
  const int32_t* d_my_tiles = f->d_tiles;
  CU(cudaEventRecord(f->evc[0], s));
  CU(cudaMemsetAsync(f->d_pix_cnt, 0, sizeof(int32_t) * npix, s));
  int grid = sm_count() * 8;
  if (nsrc > 0) {
    CU(launch_hist(src, nsrc, f->d_pix_cnt, grid, s));
  }
  CU(scan_exclusive<int32_t>(f->d_pix_cnt, f->d_pix_off, npix, f->d_scan_tmp, s));
  CU(cudaMemsetAsync(f->d_pix_cnt, 0, sizeof(int32_t) * npix, s));
  if (nsrc > 0) {
    if (copy) CU(launch_scatter_rec(src, nsrc, f->d_pix_off, f->d_pix_cnt, f->d_sorted, grid, s));
    else CU(launch_scatter(src, nsrc, f->d_pix_off, f->d_pix_cnt, f->d_perm, grid, s));
  }
  CU(cudaEventRecord(f->evc[1], s));
  if (npix_out > 0) {
    float bg[3] = {0, 0, 0};
    if (background) memcpy(bg, background, sizeof bg);
    CU(grow(&f->d_defer, &f->defer_cap, npix_out, s));
    CU(launch_fold(copy ? f->d_sorted : src, copy ? nullptr : f->d_perm, f->d_pix_off, W, H, tw, th, d_my_tiles,
                   t->tiles_x, npix_out, bg, 1e-6f, d_rgba, f->d_defer, f->d_counters, sm_count() * 16, s));
  }
  CU(cudaEventRecord(f->evc[2], s));
  f->composite_timed = true;
  return RC_OK;
}

extern "C" rc_status rc_composite_tiles(rc_forest* f, const rc_tiling* t, rc_comm* comm, const float background[3],
                                        float* d_rgba, int64_t capacity_floats, void* stream) {
  RC_NVTX("rc_composite_tiles");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !t) return fail(RC_ERR_INVALID_ARG, "rc_composite_tiles: null argument");
  if (!comm) return rc_composite_records(f, t, nullptr, 0, background, d_rgba, capacity_floats, stream);
  if (!f->have_cast) return fail(RC_ERR_STATE, "rc_composite_tiles before rc_cast_segments");
  if (comm->nranks != t->nranks || comm->rank != t->rank)
    return fail(RC_ERR_INVALID_ARG, "rc_composite_tiles: tiling ranks %d/%d != communicator %d/%d", t->rank,
                t->nranks, comm->rank, comm->nranks);
  rc_status st = check_tiling(f, t);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int P = t->nranks;
  // K5: pack by owner on the device
  if ((st = pack_device(f, t, s))) return st;
  // count all-to-all (NCCL), then one read of both count vectors
  if (!f->d_xcnt) CU(dmalloc((void**)&f->d_xcnt, sizeof(int64_t) * 2 * RC_MAX_RANKS, s));
  if (!f->h_xcnt) CU(cudaMallocHost((void**)&f->h_xcnt, sizeof(int64_t) * 2 * RC_MAX_RANKS));
  CU(cudaMemcpyAsync(f->d_xcnt, f->d_counters + CNT_SEND, sizeof(int64_t) * P, cudaMemcpyDeviceToDevice, s));
  int r = 0;
  if (comm->partners) {   // counts only between the discovered pairs (rc_exchange_partners)
    CU(cudaMemsetAsync(f->d_xcnt + RC_MAX_RANKS, 0, sizeof(int64_t) * RC_MAX_RANKS, s));
    r = nccl_partner_i64(comm, f->d_xcnt, f->d_xcnt + RC_MAX_RANKS, s);
  } else {
    r = nccl_alltoall_i64(comm, f->d_xcnt, f->d_xcnt + RC_MAX_RANKS, s);
  }
  if (r) return fail(RC_ERR_NCCL, "count exchange: %s", nccl_error_string(r));
  CU(cudaMemcpyAsync(f->h_xcnt, f->d_xcnt, sizeof(int64_t) * 2 * RC_MAX_RANKS, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));   // the receive sizes (NCCL p2p takes host counts)
  int64_t scnt[RC_MAX_RANKS], rcnt[RC_MAX_RANKS], soff[RC_MAX_RANKS], roff[RC_MAX_RANKS];
  int64_t ts = 0, tr = 0;
  int missed = -1;   // a destination with records that the partner discovery did not list
  for (int p = 0; p < P; ++p) {
    scnt[p] = f->h_xcnt[p] * (int64_t)sizeof(rc_seg);
    rcnt[p] = f->h_xcnt[RC_MAX_RANKS + p] * (int64_t)sizeof(rc_seg);
    soff[p] = ts;
    roff[p] = tr;
    ts += scnt[p];
    tr += rcnt[p];
    if (comm->partners && p != t->rank && !comm->send_to[p] && scnt[p] > 0) {
      missed = p;
      scnt[p] = 0;   // its receiver posts no receive: drop, report after the collective
    }
  }
  const int64_t nrecv = tr / (int64_t)sizeof(rc_seg);
  CU(grow(&f->d_recv, &f->recv_cap, std::max<int64_t>(nrecv, 1), s));
  r = nccl_exchange(comm, reinterpret_cast<const char*>(f->d_send), soff, scnt, reinterpret_cast<char*>(f->d_recv),
                    roff, rcnt, s);
  if (r) return fail(RC_ERR_NCCL, "record exchange: %s", nccl_error_string(r));
  f->h_last_recv = nrecv;
  st = rc_composite_records(f, t, f->d_recv, nrecv, background, d_rgba, capacity_floats, stream);
  if (st == RC_OK && missed >= 0)
    return fail(RC_ERR_STATE, "rc_composite_tiles: records for rank %d, which the partner discovery did not list",
                missed);
  return st;
}

extern "C" rc_status rc_composite(rc_forest* f, const float background[3], float* d_rgba, int64_t capacity_floats,
                                  void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f) return fail(RC_ERR_INVALID_ARG, "rc_composite: null forest");
  rc_tiling t{1, 1, 1, 0};
  return rc_composite_records(f, &t, nullptr, 0, background, d_rgba, capacity_floats, stream);
}

// One aggregation pass: the current records (node level f->rec_level) are
// combined per (node of `level`, pixel) where they touch (k_coarsen).
static rc_status aggregate_to(rc_forest* f, int level, cudaStream_t s) {
  if (level <= f->rec_level) return RC_OK;
  int64_t nrec = 0;
  CU(cudaMemcpyAsync(&nrec, f->d_counters + CNT_SEGS, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  nrec = std::min(nrec, f->seg_cap);
  const int64_t npix = (int64_t)f->cc.W * f->cc.H;
  if (nrec >= (int64_t)UINT32_MAX) return fail(RC_ERR_CAPACITY, "more than 2^32 records in one aggregation");
  if (!f->d_pix_cnt || f->pix_cnt_cap < npix) {
    if (f->d_pix_cnt) dfree(f->d_pix_cnt, s);
    if (f->d_pix_off) dfree(f->d_pix_off, s);
    f->d_pix_cnt = nullptr;
    f->d_pix_off = nullptr;
    CU(dmalloc((void**)&f->d_pix_cnt, sizeof(int32_t) * (npix + 2), s));   // also the band counts (<= npix/32 + 1)
    CU(dmalloc((void**)&f->d_pix_off, sizeof(int64_t) * (npix + 1), s));
    f->pix_cnt_cap = npix;
  }
  int64_t need_tmp = (int64_t)scan_tmp_size(npix + 1) + 128;
  if (need_tmp > f->scan_tmp_cap) CU(grow(&f->d_scan_tmp, &f->scan_tmp_cap, need_tmp, s));
  CU(grow(&f->d_perm, &f->perm_cap, std::max<int64_t>(nrec, 1), s));
  const int grid = sm_count() * 8;
  // output buffer: half the input first for one cycle, a quarter for several
  // (a cycle roughly halves the count), grown to the exact
  // count and the pass repeated if short; before the pass it holds the
  // bucketing's scratch (index + band-local pixel: 8 bytes per input record,
  // the buffer has >= 8)
  int64_t want = std::max<int64_t>(nrec / (level - f->rec_level >= 2 ? 4 : 2) + 4096, 1);
  CU(grow(&f->d_segs2, &f->seg2_cap, want, s));
  const int64_t nbands = (npix + 31) / 32;
  if (f->boff_cap < nbands + 1) CU(grow(&f->d_boff, &f->boff_cap, nbands + 1, s));
  CU(launch_band_bucket(f->d_segs, nrec, npix, f->d_pix_cnt, f->d_boff, f->d_scan_tmp, f->d_segs2, f->d_perm,
                        f->d_pix_off, grid, s));
  // pixels deferred to the list pass [0, npix) and pixels of the mid pass (256 < n <= 512) [npix, 2 npix)
  CU(grow(&f->d_defer, &f->defer_cap, std::max<int64_t>(2 * npix, 1), s));
  const int32_t* leaf_node = nullptr;   // node of every leaf at the target level
  CU(build_leaf_node(f, level, s, &leaf_node));
  int64_t nout = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    CU(grow(&f->d_segs2, &f->seg2_cap, want, s));
    CU(cudaMemsetAsync(f->d_counters + CNT_AGG_OUT, 0, sizeof(int64_t), s));
    CU(cudaMemsetAsync(f->d_counters + CNT_OVERFLOW, 0, sizeof(int64_t), s));
    CU(launch_coarsen(f->d_segs, nrec, f->n, f->d_perm, f->d_pix_off, npix, f->d_node_first[level], leaf_node,
                      (uint32_t)f->first_global, 1e-6f, f->d_segs2, f->seg2_cap, f->d_defer, f->d_defer + npix,
                      f->d_counters,
                      sm_count() * 16, s));
    CU(cudaMemcpyAsync(&nout, f->d_counters + CNT_AGG_OUT, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (nout <= f->seg2_cap) break;
    want = nout;
  }
  if (nout > f->seg2_cap) return fail(RC_ERR_CAPACITY, "aggregation output overflow");
  CU(cudaMemsetAsync(f->d_counters + CNT_OVERFLOW, 0, sizeof(int64_t), s));
  CU(cudaMemcpyAsync(f->d_counters + CNT_SEGS, f->d_counters + CNT_AGG_OUT, sizeof(int64_t),
                     cudaMemcpyDeviceToDevice, s));
  std::swap(f->d_segs, f->d_segs2);
  std::swap(f->seg_cap, f->seg2_cap);
  f->rec_level = level;
  f->h_seg_total = nout;
  return RC_OK;
}

extern "C" rc_status rc_aggregate(rc_forest* f, int32_t cycles, void* stream) {
  RC_NVTX("rc_aggregate");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f) return fail(RC_ERR_INVALID_ARG, "rc_aggregate: null forest");
  if (cycles < 0) return fail(RC_ERR_INVALID_ARG, "cycles must be >= 0");
  if (cycles == 0) return RC_OK;
  if (!f->have_cast) return fail(RC_ERR_STATE, "rc_aggregate before rc_cast_segments");
  if (f->rec_level + cycles > RC_NODE_LEVELS)
    return fail(RC_ERR_INVALID_ARG, "records at level %d: at most %d more cycles", f->rec_level,
                RC_NODE_LEVELS - f->rec_level);
  return aggregate_to(f, f->rec_level + cycles, (cudaStream_t)stream);
}

extern "C" rc_status rc_segments_set(rc_forest* f, const rc_seg* d_recs, int64_t n, int32_t level, void* stream) {
  RC_NVTX("rc_segments_set");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || (n > 0 && !d_recs) || n < 0) return fail(RC_ERR_INVALID_ARG, "rc_segments_set: bad arguments");
  if (!f->have_camera) return fail(RC_ERR_STATE, "rc_segments_set before rc_camera_set");
  if (level < 0 || level > RC_NODE_LEVELS) return fail(RC_ERR_INVALID_ARG, "level must be in [0, %d]", RC_NODE_LEVELS);
  cudaStream_t s = (cudaStream_t)stream;
  CU(grow(&f->d_segs, &f->seg_cap, std::max<int64_t>(n + 4096, 1), s));
  if (n > 0) CU(cudaMemcpyAsync(f->d_segs, d_recs, sizeof(rc_seg) * n, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(f->d_counters + CNT_SEGS, &n, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  CU(cudaMemsetAsync(f->d_counters + CNT_OVERFLOW, 0, sizeof(int64_t), s));
  CU(cudaStreamSynchronize(s));   // &n is a host stack value
  f->rec_level = level;
  f->h_seg_total = n;
  f->have_cast = true;
  return RC_OK;
}

extern "C" rc_status rc_debug_pair(rc_forest* f, int64_t local_leaf, int32_t i, int32_t j, rc_pair_result* out,
                                   void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !out) return fail(RC_ERR_INVALID_ARG, "rc_debug_pair: null argument");
  if (!f->have_camera) return fail(RC_ERR_STATE, "rc_debug_pair before rc_camera_set");
  if (local_leaf < 0 || local_leaf >= f->n || i < 0 || j < 0 || i >= f->cc.W || j >= f->cc.H)
    return fail(RC_ERR_INVALID_ARG, "rc_debug_pair: leaf or pixel out of range");
  if (!f->all_affine && f->R != 2) return fail(RC_ERR_INVALID_ARG, "non-affine trees require geom_degree 2");
  if (!f->has_field) return fail(RC_ERR_STATE, "rc_debug_pair on a forest without a field (keys only)");
  if (f->surface) return fail(RC_ERR_INVALID_ARG, "rc_debug_pair: surface forests are not supported");
  cudaStream_t s = (cudaStream_t)stream;
  const bool curved = !f->all_affine;
  // a one-leaf, one-pixel work list through the frame's own segment kernel (fold level 0)
  struct Dbg {
    int32_t vis[4];
    Rect16 rect[2];
    int64_t chunk_off[2];
    int32_t chunk_elem[4];
    Unit unit;
  } h;
  memset(&h, 0, sizeof h);
  h.vis[0] = (int32_t)local_leaf;
  h.rect[0] = Rect16{(int16_t)i, (int16_t)i, (int16_t)j, (int16_t)j};
  h.chunk_off[0] = 0;
  h.chunk_off[1] = 1;
  h.unit = Unit{0, 1, 0u, 0, 1, 0};
  static const int64_t one = 1;
  const int64_t npix = (int64_t)f->cc.W * f->cc.H;
  const size_t scratch = curved ? cast_curved_scratch_per_cta() : 0;
  const size_t off_cnt = 256, off_segs = off_cnt + sizeof(int64_t) * CNT_TOTAL, off_hits = off_segs + 8 * sizeof(rc_seg);
  const size_t off_scr = (off_hits + sizeof(int32_t) * npix + 255) & ~(size_t)255;
  const size_t off_slot = (off_scr + scratch + 255) & ~(size_t)255;
  const size_t off_org = off_slot + slot_record_bytes();
  char* d = nullptr;
  CU(dmalloc((void**)&d, off_org + 64, s));
  Dbg* dd = reinterpret_cast<Dbg*>(d);
  int64_t* cnt = reinterpret_cast<int64_t*>(d + off_cnt);
  rc_seg* segs = reinterpret_cast<rc_seg*>(d + off_segs);
  int32_t* hits = reinterpret_cast<int32_t*>(d + off_hits);
  cudaError_t e = cudaMemcpyAsync(dd, &h, sizeof h, cudaMemcpyHostToDevice, s);
  if (!e) e = cudaMemsetAsync(cnt, 0, sizeof(int64_t) * CNT_TOTAL, s);
  if (!e) e = cudaMemsetAsync(hits, 0, sizeof(int32_t) * npix, s);
  if (!e) {
    const uint32_t key_base = (uint32_t)f->first_global;
    if (curved) {
      e = cudaMemcpyAsync(cnt + CNT_SEGS, &one, sizeof(int64_t), cudaMemcpyHostToDevice, s);   // visible count 1
      if (!e) e = launch_prep_slots(f->d_trees, leaf_view(f), f->P, dd->vis, cnt + CNT_SEGS, 0, 1, d + off_slot,
                                    d + off_org, s);
      if (!e) e = cudaMemsetAsync(cnt, 0, sizeof(int64_t) * CNT_TOTAL, s);
      if (!e)
        e = launch_cast_curved(f->cc, f->d_trees, leaf_view(f), f->P, dd->vis, dd->rect, dd->chunk_off,
                               dd->chunk_elem, &dd->unit, 1, 0, key_base, d + off_scr, segs, 8, hits, cnt, 1,
                               d + off_slot, d + off_org, 0, 1, s);
    } else {
      e = launch_cast_affine(f->cc, f->d_trees, leaf_view(f), f->P, dd->vis, dd->rect, dd->chunk_off,
                             dd->chunk_elem, 1, key_base, segs, 8, hits, cnt, 1, s);
    }
  }
  int64_t hc[CNT_TOTAL];
  rc_seg hs[8];
  (void)one;
  if (!e) e = cudaMemcpyAsync(hc, cnt, sizeof hc, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaMemcpyAsync(hs, segs, sizeof hs, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  dfree(d, s);
  if (e) return fail(RC_ERR_CUDA, "rc_debug_pair: %s", cudaGetErrorString(e));
  const int ns = (int)std::min<int64_t>(hc[CNT_SEGS], 4);
  std::sort(hs, hs + ns, [](const rc_seg& x, const rc_seg& y) { return x.alpha_near < y.alpha_near; });
  memset(out, 0, sizeof *out);
  out->nseg = ns;
  for (int k = 0; k < ns; ++k) {
    out->alpha_near[k] = hs[k].alpha_near;
    out->alpha_far[k] = hs[k].alpha_far;
    out->a[k] = hs[k].a;
    for (int c = 0; c < 3; ++c) out->b[k][c] = hs[k].b[c];
  }
  if (hc[CNT_NEWTON_FAIL] > 0) return fail(RC_ERR_NUMERIC, "rc_debug_pair: Newton did not converge");
  return RC_OK;
}

extern "C" rc_status rc_node_table(rc_forest* f, int32_t level, int32_t* d_first, int64_t capacity, int64_t* count,
                                   void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !count) return fail(RC_ERR_INVALID_ARG, "rc_node_table: null argument");
  if (level < 1 || level > RC_NODE_LEVELS) return fail(RC_ERR_INVALID_ARG, "level must be in [1, %d]", RC_NODE_LEVELS);
  *count = f->n_nodes[level];
  if (f->n_nodes[level] > capacity) return fail(RC_ERR_CAPACITY, "rc_node_table: capacity too small");
  cudaStream_t s = (cudaStream_t)stream;
  if (d_first && f->n_nodes[level] > 0)
    CU(cudaMemcpyAsync(d_first, f->d_node_first[level], sizeof(int32_t) * f->n_nodes[level],
                       cudaMemcpyDeviceToDevice, s));
  CU(cudaStreamSynchronize(s));
  return RC_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph frames (C1 / C2 frames are launch bound).  Affine
// forests, fold level 0, one image: after an ordinary frame has sized every
// buffer for the camera, the frame is enqueued without host synchronisation
// -- counts are read on the device (chunk total, record total), the grids
// cover the forest's capacity -- captured once and replayed.
// ---------------------------------------------------------------------------
static rc_status enqueue_affine_frame(rc_forest* f, const float bg[3], float* d_rgba, cudaStream_t s) {
  const int64_t n = f->n;
  const int W = f->cc.W, H = f->cc.H;
  const int64_t npix = (int64_t)W * H;
  // camera constants (rc_camera_set's upload, from pinned copies)
  CU(cudaMemcpyAsync(f->d_trees, f->h_trees_pin, sizeof(TreeConst) * f->K, cudaMemcpyHostToDevice, s));
  // cull + pair generation (rc_cull)
  DevLeafView L = leaf_view(f);
  CU(launch_cull(f->cc, f->d_trees, L, n, f->R, true, f->d_flag, f->d_rect_all, s));
  CU(scan_exclusive<int32_t>(f->d_flag, f->d_scan, n, f->d_scan_tmp, s));
  CU(launch_compact(f->d_flag, f->d_rect_all, f->d_scan, n, f->d_vis, f->d_vis_rect, s));
  CU(cudaMemsetAsync(f->d_counters, 0, sizeof(int64_t) * CNT_TOTAL, s));
  CU(cudaMemsetAsync(f->d_chunk_off, 0, sizeof(int64_t) * (n + 1), s));
  CU(launch_chunk_count(f->d_vis_rect, f->d_scan + n, n, f->d_chunk_off, f->d_counters, s));
  CU(scan_exclusive<int64_t>(f->d_chunk_off, f->d_chunk_off, n, f->d_scan_tmp, s));
  // segments (rc_cast_segments): counts on the device
  CU(launch_expand(f->d_chunk_off, f->d_scan + n, n, f->d_chunk_elem, s));
  CU(cudaMemsetAsync(f->d_hits_pp, 0, sizeof(int32_t) * npix, s));
  CU(launch_cast_affine(f->cc, f->d_trees, L, f->P, f->d_vis, f->d_vis_rect, f->d_chunk_off, f->d_chunk_elem,
                        f->chunk_cap, (uint32_t)f->first_global, f->d_segs, f->seg_cap, f->d_hits_pp, f->d_counters,
                        sm_count() * 8, s, f->d_chunk_off + n));
  // composite of the whole image (rc_composite), record count on the device
  const int64_t* d_nrec = f->d_counters + CNT_SEGS;
  const int grid = sm_count() * 8;
  CU(cudaMemsetAsync(f->d_pix_cnt, 0, sizeof(int32_t) * npix, s));
  CU(launch_hist(f->d_segs, f->seg_cap, f->d_pix_cnt, grid, s, d_nrec));
  CU(scan_exclusive<int32_t>(f->d_pix_cnt, f->d_pix_off, npix, f->d_scan_tmp, s));
  CU(cudaMemsetAsync(f->d_pix_cnt, 0, sizeof(int32_t) * npix, s));
  CU(launch_scatter_rec(f->d_segs, f->seg_cap, f->d_pix_off, f->d_pix_cnt, f->d_sorted, grid, s, d_nrec));
  CU(launch_fold(f->d_sorted, nullptr, f->d_pix_off, W, H, W, H, f->d_tiles, 1, npix, bg, 1e-6f, d_rgba, f->d_defer,
                 f->d_counters, sm_count() * 16, s));
  return RC_OK;
}

extern "C" rc_status rc_frame_capture(rc_forest* f, const rc_camera* cam, const float background[3], float* d_rgba,
                                      int64_t capacity_floats, void* stream) {
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f || !cam || !d_rgba) return fail(RC_ERR_INVALID_ARG, "rc_frame_capture: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  rc_status st = rc_render_frame(f, cam, 0, 0, background, d_rgba, capacity_floats, nullptr, stream);
  if (st) return st;
  if (!f->all_affine) return fail(RC_ERR_STATE, "rc_frame_capture: graph frames are for affine forests");
  if (f->last_composite_copy != 1) return fail(RC_ERR_STATE, "rc_frame_capture: no memory for the record copy");
  if (!f->h_trees_pin) CU(cudaMallocHost((void**)&f->h_trees_pin, sizeof(TreeConst) * f->K));
  memcpy(f->h_trees_pin, f->h_trees, sizeof(TreeConst) * f->K);
  float bg[3] = {0, 0, 0};
  if (background) memcpy(bg, background, sizeof bg);
  if (f->graph_exec) {
    cudaGraphExecDestroy(f->graph_exec);
    f->graph_exec = nullptr;
  }
  CU(cudaStreamSynchronize(s));
  // capture on a library stream (the caller's may be the legacy default stream, which cannot
  // capture); the graph is launched on the caller's stream
  if (!f->cap_stream) CU(cudaStreamCreateWithFlags(&f->cap_stream, cudaStreamNonBlocking));
  cudaStream_t cs = f->cap_stream;
  CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const int64_t k0 = g_launches.load();
  st = enqueue_affine_frame(f, bg, d_rgba, cs);
  f->graph_kernels = g_launches.load() - k0;   // kernel nodes of the graph (counted again per replay)
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &g);
  if (st) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return fail(RC_ERR_CUDA, "rc_frame_capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&f->graph_exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(RC_ERR_CUDA, "rc_frame_capture: instantiate: %s", cudaGetErrorString(e));
  return RC_OK;
}

extern "C" rc_status rc_frame_replay(rc_forest* f, void* stream) {
  RC_NVTX("rc_frame_replay");
  if (f) f->last_stream = (cudaStream_t)stream;
  if (!f) return fail(RC_ERR_INVALID_ARG, "rc_frame_replay: null forest");
  if (!f->graph_exec) return fail(RC_ERR_STATE, "rc_frame_replay before rc_frame_capture");
  CU(cudaGraphLaunch(f->graph_exec, (cudaStream_t)stream));
  g_launches += f->graph_kernels;
  return RC_OK;
}

extern "C" rc_status rc_render_frame(rc_forest* f, const rc_camera* cam, int32_t fold_levels, int32_t cycles,
                                     const float background[3], float* d_rgba, int64_t capacity_floats,
                                     int64_t* hit_pairs, void* stream) {
  RC_NVTX("rc_render_frame");
  if (f) f->last_stream = (cudaStream_t)stream;
  rc_status st;
  if ((st = rc_camera_set(f, cam, stream))) return st;
  if ((st = rc_cull(f, stream, nullptr))) return st;
  if ((st = rc_cast_segments(f, fold_levels, stream))) return st;
  if (cycles > 0 && (st = rc_aggregate(f, cycles, stream))) return st;
  if ((st = rc_composite(f, background, d_rgba, capacity_floats, stream))) return st;
  if (hit_pairs) {
    cudaStream_t s = (cudaStream_t)stream;
    CU(cudaMemcpyAsync(hit_pairs, f->d_counters + CNT_HITPAIRS, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  return RC_OK;
}
