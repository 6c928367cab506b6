/* oracle.h -- plain fp64 CPU oracle for Burstedde, "Distributed-Memory
 * Forest-of-Octrees Raycasting" (arXiv 1809.01334).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * Shares no code, header, table or constant generator with the CUDA path
 * (paper_1809_01334_b200/).  Every function cites the passage it follows;
 * PAPER.md line numbers refer to /root/reference/PAPER.md.
 *
 * Parity unpinned: per-pair (a,b) on curved (R=2) elements with non-constant
 * fields is pinned only by self-convergence; see DESIGN.md.
 */
#ifndef RC_ORACLE_H
#define RC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t R;               /* geometry degree, GLL nodes {0,1} or {0,1/2,1} */
  int32_t P;               /* field degree */
  int32_t K;               /* number of trees */
  const double* tree_ctrl; /* [K][R+1][R+1][R+1][3] */
  int64_t n;               /* leaves */
  const int32_t* anchor;   /* [n][3], units 2^-18 */
  const int32_t* tree;     /* [n] */
  const int8_t* level;     /* [n] */
  const float* field;      /* [n][(P+1)^3], node order [k3][k2][k1]; surfaces: [n][4] corners [k2][k1] */
  double kappa0, inv_F, q0;
  /* surface forests (§2.8): dim = 2 means
   * quadtree leaves (anchor[3*e+2] = 0) on bilinear tree patches tree_ctrl
   * [K][2][2][3] ([k][m2][m1][xyz]); the corner values v of an element give
   * A_s = clamp(surf_a[0] + surf_a[1] v, 0, 1) and the per-channel intensity
   * I_s = surf_i[c][0] + surf_i[c][1] v + surf_i[c][2] w(v), w = exp(-((1-v) surf_k)^2 / 2). */
  int32_t dim;             /* 3 (or 0): volume forest; 2: surface forest */
  double surf_a[2], surf_i[3][3], surf_k;
} orc_scene;

typedef struct {
  int32_t projection;      /* 0 perspective, 1 orthographic */
  double origin[3], view[3], right[3], up[3];
  double pixel_size, far_dist;
  int32_t width, height;
} orc_camera;

/* One (element, pixel) segment record produced by orc_render. */
typedef struct {
  int64_t elem;        /* leaf index in the scene */
  int32_t pixel;       /* j*w + i */
  int32_t flags;       /* ORC_HIT | ORC_AMBIGUOUS | ORC_NEWTON_FAIL */
  double alpha_near, alpha_far, a, b[3];
} orc_hit;

enum { ORC_HIT = 1, ORC_AMBIGUOUS = 2, ORC_NEWTON_FAIL = 4, ORC_OVERFLOW = 8, ORC_SPLIT_NEAR = 16 };
enum { ORC_GL = 0, ORC_EULER = 1, ORC_HEUN2 = 2, ORC_HEUN3 = 3, ORC_RK4 = 4, ORC_GAUSS2 = 5, ORC_SIMPSON = 6 };

/* ---- segment algebra, PAPER.md:386-558 ---- */
void orc_combine(double an, double bn, double af, double bf, double* a, double* b);
int  orc_inverse(double a, double b, double* ai, double* bi);
int  orc_split(double a, double b, double dx1, double dx2, double out[4]);
void orc_average(double a1, double b1, double a2, double b2, double* a, double* b);
void orc_from_constant(double beta, double gamma, double dx, double* a, double* b);
double orc_background(double a, double b, double Ib);

/* ---- quadrature ---- */
void orc_gauss_legendre(int N, double* u, double* w);
void orc_lagrange_integrals(int N, const double* u, double* S);
typedef void (*orc_medium_fn)(void* ctx, double s, double* kappa, double* q3);
int  orc_segment_exact(orc_medium_fn fn, void* ctx, double L, double* a, double b[3]);
void orc_segment_rule(int N, orc_medium_fn fn, void* ctx, double L, double* a, double b[3]);
/* Alg. 1 adaptive integration with a scheme (ORC_*); returns the recursion
 * depth reached; *flags: 1 = depth cap hit, 2 = a split decision within 1e-4
 * of c_RK.  orc_set_scheme selects the scheme of orc_render mode 3. */
int  orc_segment_scheme(int scheme, int N, double c_rk, int max_depth, orc_medium_fn fn, void* ctx, double L,
                        double* a, double b[3], int* flags);
void orc_set_scheme(int scheme, double c_rk, int max_depth);
long long orc_medium_evals(int reset);   /* field evaluations of orc_render so far (diagnostic) */

/* ---- geometry / camera ---- */
void orc_gll(int R, double* eta);
void orc_lagrange(int R, const double* eta, double t, double* psi, double* dpsi);
void orc_tree_map(const orc_scene* sc, int k, const double t[3], double x[3]);
void orc_element_map(const orc_scene* sc, int64_t e, const double xi[3], double x[3], double J[9]);
void orc_camera_transform(const orc_camera* cam, const double x[3], double X[3]);
void orc_ray(const orc_camera* cam, int i, int j, double o[3], double r[3]);
int  orc_element_aabb(const orc_scene* sc, const orc_camera* cam, int64_t e, double lo[3], double hi[3]);
int  orc_pixel_rect(const orc_camera* cam, const double lo[3], const double hi[3], int32_t rect[4]);
void orc_cull(const orc_scene* sc, const orc_camera* cam, int8_t* visible, int8_t* ambiguous,
              int32_t* rects);
double orc_field(const orc_scene* sc, int64_t e, const double xi[3]);
int  orc_inverse_map(const orc_scene* sc, int64_t e, const double x[3], double xi[3]);

/* ---- intersection: segments of pixel (i,j)'s ray inside element e ---- */
int  orc_intersect(const orc_scene* sc, const orc_camera* cam, int64_t e, int i, int j,
                   int max_seg, double* seg /* [max_seg][2] */, int* flags);

void orc_set_force_general(int on);

/* ---- full render of a pixel subset ---- */
int64_t orc_render(const orc_scene* sc, const orc_camera* cam, int mode /*0 exact,1 rule*/, int N,
                   const double background[3], int64_t npix, const int32_t* pixels,
                   double* rgba /*[npix][4]*/, int32_t* nhits /*[npix]*/, int32_t* namb /*[npix]*/,
                   int32_t cap, orc_hit* hits /*[npix][cap] or NULL*/, int nthreads);

/* As orc_render, plus (each optional): the culled list of orc_cull
 * (visible[n], ambiguous[n]) and, per rendered pixel, the (elem, flags) of
 * every candidate pair that hits or is eps-ambiguous (CSR, allocated here,
 * released by orc_pairs_free).  mode 2 = hit lists only (no integration;
 * rgba = 0).  rects_in (optional, [n][4]): the rectangles of an earlier
 * orc_cull of the same scene and camera, reused instead of culling again
 * (visible / ambiguous are then not written). */
typedef struct {
  int64_t npix;
  int64_t* off;      /* [npix+1] */
  int64_t* elem;     /* [off[npix]] */
  int32_t* flags;    /* [off[npix]] ORC_HIT | ORC_AMBIGUOUS */
} orc_pairs;
int64_t orc_render_ex(const orc_scene* sc, const orc_camera* cam, int mode, int N, const double background[3],
                      int64_t npix, const int32_t* pixels, double* rgba, int32_t* nhits, int32_t* namb,
                      int nthreads, int8_t* visible, int8_t* ambiguous, orc_pairs* pairs,
                      const int32_t* rects_in);
void orc_pairs_free(orc_pairs* p);

/* Fold a caller-given list of segments of one pixel (any order): sort by
 * (alpha_near, elem), resolve clusters of overlapping segments (Eq. segsplit /
 * segaverage at every end point of the cluster, D14) with
 * tolerance tau, fold back to front. */
void orc_fold_pixel(int n, orc_hit* segs, double tau, const double background[3], double rgba[4],
                    double ab[4]);

/* Surface forests (App. A.1): all s in [lo, hi)^2 with
 * X(s) = o + alpha r on the bilinear patch with corners P [2][2][3]
 * ([m2][m1][xyz]); writes s_out [count][2] and returns the count (<= 2). */
int orc_surface_roots(const double* P, const double o[3], const double r[3], double lo, double hi, double* s_out);

#ifdef __cplusplus
}
#endif
#endif
