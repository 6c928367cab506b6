// rc_internal.cuh -- internal definitions of librc (B200 / sm_100a).
// Shares nothing with oracle/ (independent implementation of the method).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/rc.h"

// Device-side bounds checks of the checked build (tag "checks": -DRC_CHECKS,
// tools/gpu_checks.sh).  compute-sanitizer is not available on the GPU pool
// this project runs on, so index bounds of the gathers and scatters are
// asserted in place instead; a violation prints the condition and traps.
#ifdef RC_CHECKS
#include <cstdio>
#define RC_DCHECK(c)                                                                   \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("RC_CHECKS %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,     \
             (int)blockIdx.x, (int)threadIdx.x);                                      \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define RC_DCHECK(c) \
  do {               \
  } while (0)
#endif

// NVTX ranges around the C ABI's phases (SURVEY §5 tracing): header-only
// NVTX3, a no-op unless a tool (nsys / ncu --nvtx) injects itself.
#include <nvtx3/nvToolsExt.h>
namespace rc {
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
}  // namespace rc
#define RC_NVTX(name) ::rc::NvtxScope rc_nvtx_scope_(name)

#define RC_MAX_N 8          // GL points per segment
#define RC_MAX_RANKS 64     // tile owners / communicator size
#define RC_MAX_TREES 4096
#define RC_MAXLEVEL 18
#define RC_CHUNK 32         // candidate pairs per warp work item (one element)
#define RC_NODE_LEVELS 8    // coarsening levels of the node tables (fold + aggregation cycles)
#define RC_UNIT_CHUNKS 128  // chunks per fold unit of the curved segment kernel (<= 4096 pairs)
#define RC_UNIT_LEAVES 64   // visible leaves per fold unit (their geometry is staged in shared memory)
#define RC_SLOT_BATCH (1 << 23)   // visible leaves per element-slot batch of the curved path (672 B each)

// Fold unit of the curved segment kernel (row a6): a contiguous chunk range
// of at most RC_UNIT_LEAVES visible leaves [vfirst, vfirst+nvis) inside one
// node of the fold level (64 consecutive visible leaves when not folding).
struct __align__(16) Unit {
  int64_t chunk_begin;
  int32_t nchunks;
  uint32_t key;                 // global SFC index of the node's first leaf (0 when not folding)
  int32_t vfirst, nvis;         // visible-leaf window holding the unit's chunks
  int64_t pad;
};

// node k of a level owns leaves [first[k], first[k+1]); returns k for leaf e
__device__ __forceinline__ int64_t node_of(const int32_t* __restrict__ first, int64_t nnodes, int32_t e) {
  int64_t lo = 0, hi = nnodes;   // invariant first[lo] <= e < first[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (first[mid] <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Camera constants (host fp64 preprocessing, rc_camera_set).
struct CamConst {
  int proj, W, H, N;
  int newton_max;
  float newton_tol;
  double O0[3], Ot[3], Ou[3];   // world ray origin  O(i,j) = O0 + di Ot + dj Ou
  double R0[3], Rt[3], Ru[3];   // world ray dir     R(i,j) = R0 + di Rt + dj Ru
  double amin, amax;            // visible alpha range
  double cam_rot[9];            // rows t, u, v/n
  double cam_org[3];            // o (perspective) / P0 (ortho)
  double n, ell, far_dist;
  float u[RC_MAX_N], w[RC_MAX_N], S[RC_MAX_N * RC_MAX_N];
  float kappa0, inv_F, q0;
  float f_R0[3], f_Rt[3], f_Ru[3], f_Ot[3], f_Ou[3];   // fp32 copies for the conservative prefilter
  int scheme;                   // RC_SCHEME_* (segment integrator)
  int max_depth;                // Alg. 1 recursion cap
  float c_rk;                   // Alg. 1 threshold (0: no recursion)
  rc_surface surf;              // surface forests: transfer of the corner-interpolated value
};

// Per-tree constants (device buffer, warp-uniform reads).
struct TreeConst {
  int affine;                   // 1: J_k affine -> slab path
  int pad;
  // affine: tree-reference ray t(i,j,alpha) = TO0 + di TOt + dj TOu + alpha (TR0 + di TRt + dj TRu)
  double TO0[3], TOt[3], TOu[3], TR0[3], TRt[3], TRu[3];
  // affine culling: camera-space X = Acam t + bcam
  double Acam[9], bcam[3];
  // Bernstein control points of J_k: world [27][3] and camera space [27][3]
  double Bw[81];
  double Bc[81];
  double lagr[81];              // Lagrange control points as given (host copy)
};

struct DevLeafView {
  const int32_t* anchor;  // [n][3]
  const int32_t* tree;    // [n]
  const int8_t* level;    // [n]
  const float* field;     // [n][(P+1)^3]
};

// short rect (i0,i1,j0,j1), inclusive
struct __align__(8) Rect16 {
  int16_t i0, i1, j0, j1;
};

struct rc_forest {
  int K, R, P;
  int64_t n, first_global;
  bool has_field = true;           // false: keys-only forest (aggregation / partition bookkeeping)
  bool borrowed = false;           // RC_DEVICE_BORROW: d_anchor / d_tree / d_field are the caller's
  cudaStream_t last_stream = nullptr;   // stream of the last call (one forest per stream at a time)
  bool surface = false;            // dim = 2: quadtree leaves on bilinear patches (surface.cu)
  rc_surface surf{};
  rc_transfer transfer;
  // device leaves
  int32_t* d_anchor = nullptr;
  int32_t* d_tree = nullptr;
  int8_t* d_level = nullptr;
  float* d_field = nullptr;
  // camera
  bool have_camera = false, have_cull = false, have_cast = false;
  rc_camera cam{};
  CamConst cc{};
  TreeConst* d_trees = nullptr;
  TreeConst* h_trees = nullptr;
  CamConst* d_cam = nullptr;
  int all_affine = 1;
  // cull
  int32_t* d_flag = nullptr;      // [n] visible flag
  Rect16* d_rect_all = nullptr;   // [n]
  int64_t* d_scan = nullptr;      // [n+1]
  int32_t* d_vis = nullptr;       // [n] compacted visible leaf index
  Rect16* d_vis_rect = nullptr;   // [n]
  int64_t* d_chunk_off = nullptr; // [n+1]
  int64_t* d_counters = nullptr;  // misc device counters (see enum in rc.cu)
  int64_t h_num_visible = 0;
  // chunks / segments
  int32_t* d_chunk_elem = nullptr;
  int64_t chunk_cap = 0;
  rc_seg* d_segs = nullptr;
  int64_t seg_cap = 0;
  int32_t* d_hits_pp = nullptr;   // [W*H]
  int64_t pix_cap = 0;
  int64_t h_candidates = 0, h_chunks = 0;
  // composite scratch
  int32_t* d_pix_cnt = nullptr;   // [W*H]
  int64_t pix_cnt_cap = 0;
  int64_t* d_pix_off = nullptr;   // [W*H+1]
  uint32_t* d_perm = nullptr;     // pixel-bucketed permutation of the records
  int64_t perm_cap = 0;
  rc_seg* d_send = nullptr;
  int64_t send_cap = 0;
  rc_seg* d_recv = nullptr;        // records received by the tile exchange
  int64_t recv_cap = 0, h_last_recv = 0;
  int64_t* d_xcnt = nullptr;       // [2][RC_MAX_RANKS] send / receive counts of the exchange
  int64_t* h_xcnt = nullptr;       // pinned copy
  TreeConst* h_trees_pin = nullptr; // graph frames: pinned camera constants of the captured frame
  cudaGraphExec_t graph_exec = nullptr;
  int64_t graph_kernels = 0;       // kernel launches one replay of graph_exec makes
  cudaStream_t cap_stream = nullptr;
  // scan scratch
  int64_t* d_scan_tmp = nullptr;
  int64_t scan_tmp_cap = 0;
  // curved path: intersection items of one chunk batch (64 B each)
  void* d_items = nullptr;
  int64_t items_cap = 0;
  int64_t h_seg_total = 0;
  int64_t h_cast_total = 0;   // records written by the last rc_cast_segments (before aggregation)
  int64_t h_raw_affine = 0;        // affine path: segments before folding
  // coarsening hierarchy (nodes.cu): node tables of levels 1..RC_NODE_LEVELS
  int32_t* d_node_first[RC_NODE_LEVELS + 1] = {};
  int64_t n_nodes[RC_NODE_LEVELS + 1] = {};
  int32_t* d_leaf_nodes[2] = {nullptr, nullptr};   // per-leaf node index at levels leaf_node_lv[]
  int leaf_node_lv[2] = {-1, -1};
  int leaf_node_next = 0;
  int rec_level = 0;               // node level of the current records (0 = leaves)
  // fold units of the curved kernel
  int32_t* d_ucnt = nullptr;       // [n+1] units per visible leaf (node starts only)
  int64_t* d_uoff = nullptr;       // [n+1] exclusive scan of d_ucnt
  int32_t* d_uend = nullptr;       // [n]
  Unit* d_units = nullptr;
  int64_t units_cap = 0;
  int64_t h_units = 0;
  void* d_scratch = nullptr;       // per-CTA item / segment / key scratch of the fused kernel
  void* d_gslot = nullptr;         // element slots of one batch of visible leaves (k_prep_slots)
  int64_t slot_cap = 0;
  size_t scratch_bytes = 0;
  // aggregation output (ping-pong with d_segs)
  int32_t* d_defer = nullptr;      // composite: deferred pixels [w*h]
  int64_t* d_boff = nullptr;       // aggregation: band offsets of the banded pixel bucketing
  int64_t boff_cap = 0;
  int32_t* d_tiles = nullptr;      // composite: this rank's tile ids (uploaded when the tiling changes)
  int32_t* h_tiles = nullptr;      // pinned staging of d_tiles
  int64_t tiles_cap = 0, h_tiles_cap = 0;
  int32_t tiling_key[4] = {-1, -1, -1, -1};   // tiles_x, tiles_y, nranks, rank of d_tiles
  rc_seg* d_sorted = nullptr;      // composite: pixel-bucketed copy of the records
  int last_composite_copy = -1;    // diagnostic: 1 copy path, 0 permutation path
  int64_t sorted_cap = 0;
  int64_t defer_cap = 0;
  rc_seg* d_segs2 = nullptr;
  int64_t seg2_cap = 0;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evc[3] = {nullptr, nullptr, nullptr};   // composite: start, after scatter, after fold
  bool composite_timed = false;
  cudaEvent_t evb[4] = {nullptr, nullptr, nullptr, nullptr};
  // per batch of the last rc_cast_segments: segment kernel start/end, prep start/end
  static constexpr int kEvBatches = 64;
  cudaEvent_t evk[4 * kEvBatches] = {};
  int evk_used = 0;   // batches timed (0: none)
  float phase_ms[3] = {0, 0, 0};
  bool timed = false;
};

// Device counters layout
enum {
  CNT_SEGS = 0,        // segment records written
  CNT_HITPAIRS = 1,    // pairs with >= 1 segment
  CNT_NEWTON_FAIL = 2,
  CNT_CANDIDATES = 3,
  CNT_OVERFLOW = 4,
  CNT_WORK = 5,        // dynamic work counter of the segment kernel
  CNT_FACE_FAIL = 6,   // face-root Newton non-convergence (diagnostic)
  CNT_ITEMS = 7,       // curved path: (pair, segment) items of the current batch
  CNT_SEND = 8,        // [8..8+64) per-rank cursors for pack
  CNT_UNITS = 72,      // dynamic unit counter of the fused curved kernel
  CNT_RAW = 73,        // segments before folding
  CNT_UNFOLDED = 74,   // units whose segments exceeded the on-chip sort (emitted unfolded)
  CNT_AGG_OUT = 75,    // records written by an aggregation pass
  CNT_TASKS = 76,      // curved path: (pixel, face) root-finding tasks
  CNT_FALLBACK = 77,   // ... of which needed the projected-patch (2D) method
  CNT_DEFER = 78,      // composite: pixels deferred to the large-pixel pass
  CNT_BIGPIX = 79,     // composite: pixels with more records than FOLD_CAP_LIST (written as NaN)
  CNT_DEPTH_CAP = 80,  // Alg. 1 steps taken at the recursion cap (must be 0)
  CNT_MID = 81,        // aggregation: pixels with 256 < n <= 512 records (second fast pass)
  CNT_TOTAL = 96
};

// NCCL communicator (comm.cu)
struct rc_comm {
  void* nccl = nullptr;   // ncclComm_t
  int nranks = 1, rank = 0, device = 0;
  // exchange partners (rc_comm_set_partners, NEXT(4)): counts and records move
  // only between discovered pairs instead of an all-to-all
  bool partners = false;
  uint8_t send_to[RC_MAX_RANKS] = {}, recv_from[RC_MAX_RANKS] = {};
};

// ---- kernels / launchers (defined in the .cu files) ----
namespace rc {
rc_status rc_fail(rc_status st, const char* fmt, ...);   // sets rc_last_error (rc_api.cu)
const char* nccl_error_string(int r);
int nccl_exchange(rc_comm* c, const char* sbuf, const int64_t* soff, const int64_t* scnt, char* rbuf,
                  const int64_t* roff, const int64_t* rcnt, cudaStream_t s);
int nccl_alltoall_i64(rc_comm* c, const int64_t* d_send, int64_t* d_recv, cudaStream_t s);
int nccl_partner_i64(rc_comm* c, const int64_t* d_send, int64_t* d_recv, cudaStream_t s);
extern std::atomic<int64_t> g_launches;   // several host threads may drive forests at once
cudaError_t scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t s);
size_t scan_tmp_size(int64_t n);
}  // namespace rc

namespace rc {
cudaError_t build_node_levels(rc_forest* f, cudaStream_t s);
// caching pool (pool.cu): stream-ordered reuse; idle = no pending work reads p
cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s, bool idle = false);
void dtrim();
size_t device_free_bytes();   // cudaMemGetInfo's free bytes + the pool's cached blocks on this device
cudaError_t build_leaf_node(rc_forest* f, int c, cudaStream_t s, const int32_t** out);
template <typename Tin>
cudaError_t scan_exclusive(const Tin* in, int64_t* out, int64_t n, int64_t* tmp, cudaStream_t s);
}  // namespace rc
