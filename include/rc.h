/* rc.h -- C ABI of the B200-native forest-of-octrees raycasting hot path.
 *
 * Method: C. Burstedde, "Distributed-Memory Forest-of-Octrees Raycasting",
 * arXiv 1809.01334.  PAPER.md line numbers refer to the paper text
 * (/root/reference/PAPER.md); SURVEY.md §8 fixes the readings used here.
 *
 * Conventions for every entry point:
 *  - returns rc_status; nothing throws, exits or prints.  On failure
 *    rc_last_error() describes the failing call (thread-local, valid until the
 *    next rc_* call on the same thread).
 *  - all device work is enqueued on the caller's stream (a cudaStream_t passed
 *    as void*, e.g. torch.cuda.current_stream().cuda_stream); entries marked
 *    [sync] synchronise that stream before returning.
 *  - pointers named d_* are device pointers, h_* host pointers.  The caller
 *    owns every buffer it passes; the library owns its device scratch and the
 *    views it hands out (valid until the next call that recomputes them or
 *    rc_forest_destroy).
 *  - one rc_forest per host thread / stream at a time.
 */
#ifndef RC_H
#define RC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RC_OK = 0,
  RC_ERR_INVALID_ARG = -1,   /* null pointer, R or P not in {1,2}, n <= 0, bad camera   */
  RC_ERR_NOT_SFC_SORTED = -2,/* leaves not strictly increasing in (tree, Morton key)    */
  RC_ERR_OUT_OF_MEMORY = -3,
  RC_ERR_CUDA = -4,          /* CUDA runtime error; rc_last_error() has the call site   */
  RC_ERR_NCCL = -5,          /* NCCL missing or a collective failed (rc_comm_*)          */
  RC_ERR_CAPACITY = -6,      /* caller buffer too small; *required is written           */
  RC_ERR_STATE = -7,         /* call order violated (cast before camera_set, ...)       */
  RC_ERR_NUMERIC = -8        /* non-finite input                                        */
} rc_status;

const char* rc_last_error(void);
int32_t rc_version(void);    /* ABI version, currently 4 */

/* ------------------------------------------------------------------------
 * Forest: SFC-ordered leaves of a forest of octrees with per-tree degree-R
 * tensor-product Lagrange geometry on Gauss-Lobatto nodes (PAPER.md:82-158,
 * Eq. geometrytrafo / tensorgeom) and a per-element nodal scalar field
 * (SURVEY §8(c) R11).  Element map X_E(xi) = J_k(a 2^-18 + 2^-level xi)
 * (PAPER.md:104-107).
 * ---------------------------------------------------------------------- */
typedef struct {
  float kappa0;   /* kappa = kappa0 (f inv_F)^2 */
  float inv_F;    /* 1/F, F = max |nodal f|                                       */
  float q0;       /* q = q0 ((1+f~)/2, (1-f~)/2, 1/2)  RGB emission density      */
} rc_transfer;

typedef struct {      /* surface transfer of the corner-interpolated value v (surface forests) */
  float a[2];         /* A_s = clamp(a[0] + a[1] v, 0, 1)                                  */
  float i[3][3];      /* I_s,c = i[c][0] + i[c][1] v + i[c][2] exp(-((1 - v) k)^2 / 2)      */
  float k;
} rc_surface;

enum { RC_HOST_COPY = 0, RC_DEVICE_COPY = 1, RC_HOST_COPY_TRUSTED = 2, RC_DEVICE_BORROW = 3 };

typedef struct {
  int32_t num_trees;          /* K >= 1                                                  */
  int32_t geom_degree;        /* R in {1,2}: GLL nodes {0,1} / {0,1/2,1}                  */
  const double* tree_ctrl;    /* HOST [K][R+1][R+1][R+1][3], index [k][m3][m2][m1][xyz]   */
  int32_t field_degree;       /* P in {1,2}: (P+1)^3 nodal values per element            */
  int64_t num_leaves;         /* n >= 1 (this GPU's contiguous SFC range)                */
  int64_t first_global_leaf;  /* global SFC index of leaf 0 (tie-break key, R16)         */
  const int32_t* leaf_anchor; /* [n][3] in units of 2^-18 of the tree cube               */
  const int32_t* leaf_tree;   /* [n]                                                     */
  const int8_t* leaf_level;   /* [n], 0..18                                              */
  const float* leaf_field;    /* [n][(P+1)^3], node order [k3][k2][k1]; NULL: keys-only
                                 forest (node tables, rc_segments_set, rc_aggregate and the
                                 composite; rc_cast_segments / rc_debug_pair refuse)    */
  int32_t memory;             /* RC_HOST_COPY: leaf arrays are host pointers (checked);
                                 RC_HOST_COPY_TRUSTED: host pointers, the caller
                                 guarantees SFC order (no host-side check; pinned
                                 memory gives asynchronous DMA);
                                 RC_DEVICE_COPY: leaf arrays are device pointers;
                                 RC_DEVICE_BORROW: device pointers used in place (anchor,
                                 tree, field; the 1-byte levels are copied), owned by the
                                 caller and alive until rc_forest_destroy returns        */
  rc_transfer transfer;
  /* surface forests (§2.8, App. A.1):
   * dim = 2 makes the leaves quadtree leaves (leaf_anchor[3e+2] == 0) of
   * bilinear tree patches: geom_degree = field_degree = 1, tree_ctrl is
   * [K][2][2][3] ([k][m2][m1][xyz]) and leaf_field [n][4] the corner values
   * ([k2][k1]).  A ray meets a leaf patch X_E(s), s in [0,1)^2, in at most two
   * points; each is a zero-length record (alpha_near == alpha_far) with
   * Eq. ABphi: A = A_s^(1/cos phi), b = I_s (1 - A) (Eq. BIrelation), phi the
   * angle between the ray and the patch normal; A_s = 0 is opaque.  dim = 0
   * or 3: volume forest (the rest of this header), surface ignored. */
  int32_t dim;
  rc_surface surface;
} rc_forest_desc;

typedef struct rc_forest rc_forest;

/* Copies the leaves to device memory (device layout in DESIGN.md §4).  Checks
 * strict SFC order on the host for RC_HOST_COPY (RC_ERR_NOT_SFC_SORTED).
 * [sync] */
rc_status rc_forest_create(const rc_forest_desc* desc, void* stream, rc_forest** out);
rc_status rc_forest_destroy(rc_forest* f);

/* ------------------------------------------------------------------------
 * Camera (Fig. camera, Eq. ray; orthographic per SURVEY R4).
 * Perspective: ray o + alpha r, r = v + l((i-(w-1)/2) t + (j-(h-1)/2) u),
 * visible alpha in [1, f/|v|].  Orthographic: origin o + l(...), direction v
 * (unit), alpha in [0, f].  t, u unit, (t,u,v/|v|) orthonormal.
 * ---------------------------------------------------------------------- */
enum { RC_PERSPECTIVE = 0, RC_ORTHOGRAPHIC = 1 };

typedef struct {
  int32_t projection;
  double origin[3], view[3], right[3], up[3];
  double pixel_size;      /* l  */
  double far_dist;        /* f  */
  int32_t width, height;  /* w, h; pixel id = j*w + i                       */
  int32_t gl_points;      /* N in [1,8] Gauss-Legendre points per segment  */
  double newton_tol;      /* R=2: stop when ||dxi||_inf < tol                */
  int32_t newton_max_iter;/* R=2: iteration cap; failures are counted, never silent     */
  /* segment integrator (§2.7).  RC_SCHEME_GL with c_rk = 0 is the
   * N-point rule of SURVEY R13 (the default); every scheme with c_rk > 0 runs
   * Alg. 1: a step evaluating dx*kappa > c_rk at one of its nodes is replaced by
   * its two halves (downstream half (+) upstream half), at most max_depth levels
   * (steps at the cap are taken and counted in rc_segments.depth_capped). */
  int32_t scheme;         /* RC_SCHEME_*                                                */
  double c_rk;            /* Alg. 1 threshold (0: no recursion)                         */
  int32_t max_depth;      /* Alg. 1 recursion cap in [0, 24] (0 = 24)                   */
} rc_camera;
enum { RC_SCHEME_GL = 0, RC_SCHEME_EULER = 1, RC_SCHEME_HEUN2 = 2, RC_SCHEME_HEUN3 = 3, RC_SCHEME_RK4 = 4,
       RC_SCHEME_GAUSS2 = 5, RC_SCHEME_SIMPSON = 6 };

/* Host fp64 preprocessing: per-tree camera constants and GL tables
 * (Eq. camerapoints).  Validates the camera (orthonormal
 * frame to 1e-9, f > n, w,h in [1,32767], N in [1,8]).  Async. */
rc_status rc_camera_set(rc_forest* f, const rc_camera* cam, void* stream);

/* ------------------------------------------------------------------------
 * Cull: leaf visible iff the pixel-
 * centre rectangle of the camera-space AABB of its Bernstein-Bezier points
 * is non-empty.  Produces the compacted visible list (SFC order) and the
 * per-visible-leaf pixel rectangles on the device.  Async.
 * d_num_visible (optional, device int64 scalar): receives the number of
 * visible leaves (stream-ordered, no host sync).
 * ---------------------------------------------------------------------- */
rc_status rc_cull(rc_forest* f, void* stream, int64_t* d_num_visible);

/* [sync] Copies the visible leaf indices (local, SFC order) to the caller's
 * device buffer d_visible[capacity]; *count = number of visible leaves.
 * RC_ERR_CAPACITY (with *count set) if capacity is too small. */
rc_status rc_cull_result(rc_forest* f, int32_t* d_visible, int64_t capacity, int64_t* count, void* stream);

/* Partition weights of the last cull ("weight proportional
 * to its visible pixel count"): d_w[e] = (pixel-centre
 * rectangle area of leaf e, 0 when culled) + 1 for every local leaf, device
 * int64 [num_leaves].  Async.  Must follow rc_cull. */
rc_status rc_leaf_weights(rc_forest* f, int64_t* d_w, int64_t capacity, void* stream);

/* ------------------------------------------------------------------------
 * Cast segments (PAPER.md:921-953 leaf-level rendering): for every candidate
 * (visible leaf, pixel in its rectangle) pair, intersect the ray with the
 * element (slab test in reference coordinates for affine trees; face roots
 * + Newton for curved R=2 trees, App. A.1) and integrate dI/ds = -kappa I + q
 * over each inside interval with the N-point nested Gauss-Legendre rule
 * (SURVEY R13), giving the segment (alpha_near, alpha_far, a, b[3]) of
 * Eq. ABgeneral, near end = camera side.
 *
 * fold_levels = c in [0, 8] (row a6): the segments are combined per
 * (node of coarsening level c, pixel) where they touch, nearest first with
 * Eq. aggregate -- the first c coarsening cycles of
 * PAPER.md:956-977, done on chip for curved trees.  Level 0
 * gives one record per (leaf, pixel, segment).  Records are keyed by the
 * global SFC index of the node's first leaf (the leaf itself at level 0).
 * Node levels: level c+1 replaces every complete local family of 8 siblings
 * of level c by its parent (rc_node_table).
 * Must follow rc_cull.  [sync] (small D2H reads to size the outputs; a too
 * small record buffer is grown and the kernel repeated).
 * ---------------------------------------------------------------------- */
typedef struct {              /* 32-byte segment record, also the wire format          */
  uint32_t pixel;             /* j*w + i                                                */
  float alpha_near, alpha_far;/* ray parameter interval, alpha_near < alpha_far         */
  float a;                    /* transmission, shared by the channels (scalar kappa)     */
  float b[3];                 /* emission per channel                                   */
  uint32_t key;               /* global SFC index of the record's node's first leaf
                                 (tie-break R16; the leaf itself at level 0)            */
} rc_seg;

typedef struct {
  int64_t count;               /* number of records in segs                            */
  int64_t candidates;          /* candidate (leaf, pixel) pairs evaluated              */
  int64_t hit_pairs;           /* pairs with >= 1 segment (the metric's unit)          */
  int64_t newton_failures;     /* R=2 Newton non-convergence count, all solves (must be 0) */
  int64_t face_failures;       /* ... of which face-root solves (diagnostic)               */
  int64_t num_visible;
  int64_t raw_segments;        /* segments before any folding                          */
  int64_t level;               /* node level of the records (fold + aggregation cycles) */
  int64_t units;               /* fold units of the curved kernel                      */
  int64_t unfolded_units;      /* units too large for the bucket fold (bitonic batches instead) */
  int64_t face_tasks;          /* curved path: (pixel, face) root-finding tasks (diagnostic) */
  int64_t fallback_tasks;      /* ... of which needed the projected-patch method (diagnostic) */
  const rc_seg* segs;          /* device view, library-owned                           */
  const int32_t* hits_per_pixel; /* device [w*h]: pairs with >= 1 segment per pixel     */
  int64_t depth_capped;        /* Alg. 1 steps taken at max_depth (must be 0)          */
} rc_segments;

rc_status rc_cast_segments(rc_forest* f, int32_t fold_levels, void* stream);
/* [sync] fills *out with counts and device views of the current segments. */
rc_status rc_segments_get(rc_forest* f, rc_segments* out, void* stream);

/* Replaces the forest's current records by n caller records (device rc_seg,
 * copied) at node level `level` (the keys are global SFC indices of the
 * first leaves of level-`level` nodes of THIS forest): the import side of a
 * repartition between coarsening cycles, after which
 * rc_aggregate continues on them.  [sync] (sizes the buffer). */
rc_status rc_segments_set(rc_forest* f, const rc_seg* d_recs, int64_t n, int32_t level, void* stream);

/* Parity / debug export (not timed): evaluates one (visible leaf, pixel)
 * pair exactly as the segment kernel does (same device
 * code: intersection, GL rule), without folding.  local_leaf: index into
 * this forest's leaves (any leaf, culled or not); (i, j): pixel.  Up to 4
 * segments in alpha order; nseg = 0 for a miss.  Must follow rc_camera_set.
 * [sync] */
typedef struct {
  int32_t nseg;
  float alpha_near[4], alpha_far[4], a[4], b[4][3];
} rc_pair_result;
rc_status rc_debug_pair(rc_forest* f, int64_t local_leaf, int32_t i, int32_t j, rc_pair_result* out,
                        void* stream);

/* [sync] Copies the node table of coarsening level `level` in [1, 8] (local
 * index of each node's first leaf, SFC order) to d_first[capacity] (device);
 * *count = number of nodes.  RC_ERR_CAPACITY if capacity is too small. */
rc_status rc_node_table(rc_forest* f, int32_t level, int32_t* d_first, int64_t capacity, int64_t* count,
                        void* stream);

/* ------------------------------------------------------------------------
 * Aggregate (PAPER.md:956-994 coarsening cycles, row a7): `cycles` more
 * levels: every complete local family of siblings is replaced by its parent
 * and, per (parent, pixel), the children's records are merged in alpha order,
 * touching ones combined with Eq. aggregate.  Lossless up to
 * roundoff.  The record level rises by `cycles` (at most 8 in total).  [sync]
 * ---------------------------------------------------------------------- */
rc_status rc_aggregate(rc_forest* f, int32_t cycles, void* stream);

/* ------------------------------------------------------------------------
 * Multi-GPU communicator: NCCL, loaded at run time
 * (libnccl.so.2; RC_ERR_NCCL when missing).  Rank 0 draws the id with
 * rc_comm_unique_id, the caller broadcasts its 128 bytes (e.g. with
 * torch.distributed), every rank calls rc_comm_create collectively on its
 * own device (the current CUDA device).  One rank per GPU.
 * ---------------------------------------------------------------------- */
typedef struct rc_comm rc_comm;
rc_status rc_comm_unique_id(uint8_t id[128]);
rc_status rc_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, void* stream, rc_comm** out);
rc_status rc_comm_destroy(rc_comm* c);

/* ------------------------------------------------------------------------
 * Composite.  Image tiles of
 * tw x th = (w/tiles_x) x (h/tiles_y) pixels; tile (tx,ty) is owned by rank
 * (tx + ty) mod nranks.
 *
 * rc_composite_tiles: the whole exchange + composite of this rank's tiles.
 *   comm == NULL: composites this forest's own records for the tiles of
 *   t->rank (one GPU: t = {tx, ty, 1, 0}).  comm != NULL (t->nranks and
 *   t->rank must match it): the records are packed by owner on the device
 *   (K5), the per-destination counts go through an NCCL all-to-all, and the
 *   records through grouped ncclSend / ncclRecv on the caller's stream
 *   (PAPER.md:1053-1056); the owner composites what it receives.  One host
 *   synchronisation (the receive sizes).  Collective: every rank calls it.
 *   Composite per owned pixel: order the records by (alpha_near, key) (total
 *   order: then alpha_far, a, b), cut and average clusters of overlaps beyond
 *   1e-6 max(1,alpha) (Eq. segsplit, Eq. segaverage, D14), fold
 *   nearest-first with Eq. aggregate in fp64 and apply the background
 *   I_v = A I_b + B.  Output d_rgba: float [my tiles in
 *   row-major tile order][th][tw][4] = (R,G,B, 1-A).  At most 16384 records
 *   per pixel (more: the pixel is NaN).
 * rc_pack_tiles: permutes the current segments by owner rank into the
 *   library-owned send buffer *d_send and writes h_send_counts[nranks]
 *   (records per destination, in rank order); for callers that move the
 *   records themselves.  [sync]
 * rc_composite_records: the composite of caller-provided records d_recv
 *   (device rc_seg [nrecv]; NULL = the forest's own records).  Async.
 * rc_composite: single-GPU shortcut: the whole image, d_rgba [h][w][4].
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t tiles_x, tiles_y;   /* w % tiles_x == 0 and h % tiles_y == 0                 */
  int32_t nranks, rank;       /* nranks <= 64                                           */
} rc_tiling;

rc_status rc_composite_tiles(rc_forest* f, const rc_tiling* t, rc_comm* comm, const float background[3],
                             float* d_rgba, int64_t capacity_floats, void* stream);
rc_status rc_pack_tiles(rc_forest* f, const rc_tiling* t, int64_t* h_send_counts, const rc_seg** d_send,
                        void* stream);
rc_status rc_composite_records(rc_forest* f, const rc_tiling* t, const rc_seg* d_recv, int64_t nrecv,
                               const float background[3], float* d_rgba, int64_t capacity_floats, void* stream);
rc_status rc_composite(rc_forest* f, const float background[3], float* d_rgba, int64_t capacity_floats,
                       void* stream);

/* ------------------------------------------------------------------------
 * Exchange partners without communication (
 * PAPER.md:1030-1114).  Partition markers: the tree and anchor of every rank's
 * first leaf, known to every rank.  h_markers[nranks+1]:
 * marker p = first leaf of rank p in SFC order (an empty rank repeats the next
 * rank's marker), marker 0 = (0, {0,0,0}), marker nranks = (num_trees,
 * {0,0,0}); rank p owns the SFC positions [marker p, marker p+1).
 *
 * rc_exchange_partners: the paper's receiver-side traversal -- top down from
 * every tree root over virtual nodes, the marker range split by nested binary
 * searches, stopping where the node's pixel-centre rectangle (SURVEY R6 on the
 * node's camera-space Bernstein box, padded by 1e-9) misses the writer's
 * tiles and recording the owner once the range holds one non-empty rank
 * (PAPER.md:1093-1103).  h_recv_from[p] = 1: rank p sends records to this
 * rank (t->rank); h_send_to[q] = 1: this rank sends to writer q (the same
 * relation evaluated for every writer, DESIGN D19), so the lists of all ranks
 * agree by construction.  Tile owners as in rc_composite_tiles.  Either
 * output may be NULL.  Host only (O(nranks x depth x 8) node boxes per
 * writer); must follow rc_camera_set.  Every pair that carries a record is
 * listed (node boxes contain their leaves' boxes).
 * rc_comm_set_partners: the lists for the exchanges of rc_composite_tiles on
 * this communicator: the counts move by grouped ncclSend / ncclRecv between
 * listed pairs only (instead of the count all-to-all), the records likewise.
 * Records for an unlisted writer are not sent and the call returns
 * RC_ERR_STATE after the collective.  NULL, NULL: back to the all-to-all.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t tree;
  int32_t anchor[3];          /* units of 2^-18 of the tree cube */
} rc_marker;
rc_status rc_exchange_partners(rc_forest* f, const rc_tiling* t, const rc_marker* h_markers, uint8_t* h_send_to,
                               uint8_t* h_recv_from);
rc_status rc_comm_set_partners(rc_comm* c, const uint8_t* h_send_to, const uint8_t* h_recv_from);

/* ------------------------------------------------------------------------
 * Multiple image instances and the vforest (
 * PAPER.md:835-841, 861-919).  Per instance: rc_camera_set(instance camera) +
 * rc_cull, then rc_visible_area_add(f, d_w) adds the pixel-centre rectangle
 * area of every leaf (0 when culled) to d_w (device int64 [num_leaves],
 * caller-owned and zeroed by the caller; async): a leaf is visible while one
 * instance sees it and its weight is its visible pixel count summed over the
 * instances.
 * rc_vforest_create: a new forest (the vforest, "copying only the data of
 * the visible elements") of the leaves with d_w[e] > 0 in
 * SFC order -- keys and field gathered on the device, same trees, transfer
 * and kind; first_global_leaf = its SFC index offset (the vforest's own
 * numbering).  *h_count = its leaves; 0 leaves: *out = NULL.  d_w_out
 * (optional, device int64 [num_leaves]): the kept leaves' weights, for the
 * repartition.  The input forest is unchanged.  [sync]
 * ---------------------------------------------------------------------- */
rc_status rc_visible_area_add(rc_forest* f, int64_t* d_w, int64_t capacity, void* stream);
/* Copies the forest's leaves out (device buffers of capacity >= num_leaves
 * rows, layouts as rc_forest_desc; any pointer may be NULL): the rows a
 * repartition moves to their new owners.  Async. */
rc_status rc_forest_leaves(rc_forest* f, int32_t* d_anchor, int32_t* d_tree, int8_t* d_level, float* d_field,
                           int64_t capacity, void* stream);
rc_status rc_vforest_create(rc_forest* f, const int64_t* d_w, int64_t first_global_leaf, void* stream,
                            rc_forest** out, int64_t* h_count, int64_t* d_w_out);

/* ------------------------------------------------------------------------
 * One whole frame on one GPU from device-resident inputs:
 * rc_camera_set + rc_cull + rc_cast_segments(fold_levels) +
 * rc_aggregate(cycles) + rc_composite.  *hit_pairs (optional) receives the metric's unit count.
 * ---------------------------------------------------------------------- */
rc_status rc_render_frame(rc_forest* f, const rc_camera* cam, int32_t fold_levels, int32_t cycles,
                          const float background[3], float* d_rgba, int64_t capacity_floats, int64_t* hit_pairs,
                          void* stream);

/* CUDA-graph frames for launch-bound affine forests (C1, C2).
 * rc_frame_capture runs one rc_render_frame (fold level 0, no cycles) that
 * sizes every buffer for the camera, then captures the same frame without host
 * synchronisation (counts read on the device) into a graph owned by the
 * forest; rc_frame_replay launches it on the caller's stream (async).  The
 * graph renders this camera into this d_rgba; capture again after a camera
 * change.  RC_ERR_STATE for curved forests. */
rc_status rc_frame_capture(rc_forest* f, const rc_camera* cam, const float background[3], float* d_rgba,
                           int64_t capacity_floats, void* stream);
rc_status rc_frame_replay(rc_forest* f, void* stream);

/* Device memory: librc keeps the blocks of destroyed forests and regrown
 * buffers in a caching pool (reused by later allocations of similar size;
 * released automatically when an allocation would otherwise fail).
 * rc_pool_trim returns every cached block to the driver. */
rc_status rc_pool_trim(void);

/* Instrumentation: kernel launches issued by the library since the last
 * reset, and the device time of the segment kernel(s) of the last
 * rc_cast_segments measured with CUDA events on the caller's stream. */
int64_t rc_launch_count(int32_t reset);
float rc_last_cast_ms(rc_forest* f);
/* [sync] device time of the last rc_cast_segments' segment kernel (CUDA
 * events on the caller's stream): phase 0 or 1 = the kernel (intersection,
 * integration and fold are fused), 2 = 0 (kept for ABI stability);
 * phase 3 = diagnostic of the last composite: 1 if it sorted a pixel-bucketed
 * copy of the records, 0 if it gathered them through a permutation;
 * phase 4 / 5 = device time of the last composite's pixel bucketing (k_hist,
 * scan, scatter) / per-pixel fold kernels (k_fold), -1 before any composite;
 * phase 6 / 7 = summed device time of the last rc_cast_segments' segment
 * kernel launches alone / of its element-preparation launches (curved forests:
 * k_prep_slots per batch; 0 otherwise), events around each launch, -1 when
 * not measured. */
float rc_last_phase_ms(rc_forest* f, int32_t phase);

#ifdef __cplusplus
}
#endif
#endif
