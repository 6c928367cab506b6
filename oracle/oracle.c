/* oracle.c -- plain, slow, obviously-correct fp64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Everything here is IEEE fp64,
 * no fast-math, no blocking or fusion beyond the definitions it cites.
 * Readings of the paper where it is silent are those of SURVEY.md §8(c)
 * (R1..R24) and are listed in DESIGN.md §3.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EPS_AMBIG 1e-6   /* epsilon = 1e-6 world units      */
#define TAU_OV    1e-12  /* oracle overlap tolerance          */
#define MAXL 18

/* ======================================================================
 * Segment algebra.  PAPER.md:386-394 (Eq. aggregate), 398-404 (Eq.
 * identityinverse), 506-516 (Eq. segsplit), 529-538 (Eq. segaverage),
 * 364-375 (Eq. ABconstant), 481-488 (background).
 * Orientation: "near" is the segment closer to the camera =
 * (A2,B2) of Eq. aggregate; "far" is (A1,B1).
 * ==================================================================== */
void orc_combine(double an, double bn, double af, double bf, double* a, double* b) {
  *a = an * af;          /* A2 A1      */
  *b = bn + an * bf;     /* B2 + A2 B1 */
}

int orc_inverse(double a, double b, double* ai, double* bi) {
  if (!(a > 0.0)) return -1;         /* opaque segments have no inverse */
  *ai = 1.0 / a;
  *bi = -b / a;
  return 0;
}

/* Split (A,B) of length dx1+dx2 into pieces of lengths dx1, dx2 (Eq. segsplit). */
int orc_split(double a, double b, double dx1, double dx2, double out[4]) {
  if (dx1 < 0.0 || dx2 < 0.0 || !(dx1 + dx2 > 0.0)) return -1;
  double dx = dx1 + dx2;
  double d[2] = {dx1, dx2};
  for (int i = 0; i < 2; ++i) {
    double ai = pow(a, d[i] / dx);
    double bi = (a == 1.0) ? b * d[i] / dx            /* special case A = 1 */
                           : b * (1.0 - ai) / (1.0 - a);
    out[2 * i] = ai;
    out[2 * i + 1] = bi;
  }
  return 0;
}

void orc_average(double a1, double b1, double a2, double b2, double* a, double* b) {
  *a = sqrt(a1 * a2);
  *b = 0.5 * (b1 + b2);
}

void orc_from_constant(double beta, double gamma, double dx, double* a, double* b) {
  *a = exp(-beta * dx);
  *b = (beta == 0.0) ? gamma * dx : gamma / beta * (1.0 - *a);   /* beta -> 0 limit */
}

double orc_background(double a, double b, double Ib) { return a * Ib + b; }

/* ======================================================================
 * Quadrature.  Gauss-Legendre on [0,1] (textbook Newton on P_N) and the
 * Lagrange-basis integral table S_jk = int_0^{u_j} l_k(u) du.
 * ==================================================================== */
void orc_gauss_legendre(int N, double* u, double* w) {
  for (int i = 0; i < N; ++i) {
    double x = cos(M_PI * (i + 0.75) / (N + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (N == 1) { p1 = x; p0 = 1.0; }
      dp = N * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (fabs(dx) < 1e-16) break;
    }
    /* recompute derivative at the converged root */
    {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= N; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (N == 1) { p1 = x; p0 = 1.0; }
      dp = N * (x * p1 - p0) / (x * x - 1.0);
    }
    /* x descending in i -> u ascending */
    u[i] = 0.5 * (1.0 - x);
    w[i] = 1.0 / ((1.0 - x * x) * dp * dp);   /* (2/((1-x^2)P'^2)) / 2 */
  }
}

static double lagrange_basis_at(int N, const double* u, int k, double t) {
  double v = 1.0;
  for (int m = 0; m < N; ++m)
    if (m != k) v *= (t - u[m]) / (u[k] - u[m]);
  return v;
}

void orc_lagrange_integrals(int N, const double* u, double* S) {
  double gu[64], gw[64];
  orc_gauss_legendre(N, gu, gw);   /* N-point GL is exact for degree N-1 basis polys */
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
      for (int q = 0; q < N; ++q) s += gw[q] * u[j] * lagrange_basis_at(N, u, k, u[j] * gu[q]);
      S[j * N + k] = s;
    }
}

/* Eq. ABgeneral with s measured from the near (downstream,
 * camera-side) end x2: a = exp(-int_0^L kappa),
 * b_c = int_0^L q_c(s) exp(-int_0^s kappa) ds.  Composite 16-point
 * Gauss-Legendre panels, panel count doubled until two successive estimates
 * agree to 1e-13 (the "exact mode" of SURVEY §8(c) step 5). */
#define EX_NQ 16
static void composite_eval(orc_medium_fn fn, void* ctx, double L, int M, const double* u,
                           const double* w, const double* S, double* a, double b[3]) {
  double tau0 = 0.0, bb[3] = {0, 0, 0};
  double h = L / M;
  for (int m = 0; m < M; ++m) {
    double kap[EX_NQ], q[EX_NQ][3];
    for (int j = 0; j < EX_NQ; ++j) fn(ctx, (m + u[j]) * h, &kap[j], q[j]);
    double panel = 0.0;
    for (int j = 0; j < EX_NQ; ++j) panel += w[j] * kap[j];
    panel *= h;
    for (int j = 0; j < EX_NQ; ++j) {
      double part = 0.0;
      for (int k = 0; k < EX_NQ; ++k) part += S[j * EX_NQ + k] * kap[k];
      double tau = tau0 + h * part;
      double att = exp(-tau);
      for (int c = 0; c < 3; ++c) bb[c] += h * w[j] * q[j][c] * att;
    }
    tau0 += panel;
  }
  *a = exp(-tau0);
  for (int c = 0; c < 3; ++c) b[c] = bb[c];
}

int orc_segment_exact(orc_medium_fn fn, void* ctx, double L, double* a, double b[3]) {
  double u[EX_NQ], w[EX_NQ], S[EX_NQ * EX_NQ];
  orc_gauss_legendre(EX_NQ, u, w);
  orc_lagrange_integrals(EX_NQ, u, S);
  if (!(L > 0.0)) {
    *a = 1.0;
    b[0] = b[1] = b[2] = 0.0;
    return 0;
  }
  double ap, bp[3];
  composite_eval(fn, ctx, L, 1, u, w, S, &ap, bp);
  for (int M = 2; M <= 1024; M *= 2) {
    double ac, bc[3];
    composite_eval(fn, ctx, L, M, u, w, S, &ac, bc);
    int ok = fabs(ac - ap) <= 1e-13;
    for (int c = 0; c < 3; ++c) ok = ok && fabs(bc[c] - bp[c]) <= 1e-13 * fmax(1.0, fabs(bc[c]));
    ap = ac;
    memcpy(bp, bc, sizeof bp);
    if (ok) {
      *a = ap;
      memcpy(b, bp, sizeof bp);
      return M;
    }
  }
  *a = ap;
  memcpy(b, bp, sizeof bp);
  return -1;
}

/* SURVEY §8(c) R13, written out step by step in fp64 ("rule mode"). */
void orc_segment_rule(int N, orc_medium_fn fn, void* ctx, double L, double* a, double b[3]) {
  double u[64], w[64], S[64 * 64], kap[64], q[64][3];
  orc_gauss_legendre(N, u, w);
  orc_lagrange_integrals(N, u, S);
  for (int j = 0; j < N; ++j) fn(ctx, u[j] * L, &kap[j], q[j]);
  double sum = 0.0;
  for (int j = 0; j < N; ++j) sum += w[j] * kap[j];
  *a = exp(-L * sum);
  double bb[3] = {0, 0, 0};
  for (int j = 0; j < N; ++j) {
    double tau = 0.0;
    for (int k = 0; k < N; ++k) tau += S[j * N + k] * kap[k];
    tau *= L;
    for (int c = 0; c < 3; ++c) bb[c] += w[j] * q[j][c] * exp(-tau);
  }
  for (int c = 0; c < 3; ++c) b[c] = L * bb[c];
}

/* ======================================================================
 * The paper's per-segment integrators with the adaptive recursion of Alg. 1
 * (§2.7): explicit RK
 * (Eq. RKresultAB: Euler, Heun 2, Heun 3, classical RK4), the implicit
 * Gauss method of order 4 (Eq. gaussAB / gaussABab), Simpson's rule on the
 * closed form (Eq. simpson) and the N-point GL rule of SURVEY R13.  x runs
 * from the upstream (far) end x1 to the downstream (near) end x2;
 * the medium callback takes s = distance from the near end: s = L - x.
 * Alg. 1: a step of length dx whose computation evaluates dx beta > c_RK is
 * abandoned and replaced by segeval(x_1/2, x2) (+) segeval(x1, x_1/2).  The
 * same test at the scheme's own nodes applies to Gauss-2, Simpson and GL
 * (D17).  c_RK <= 0: no recursion.
 * ==================================================================== */
typedef struct {
  int M;
  double c[4], a[4][4], b[4];
} rk_tableau;
static const rk_tableau RK_TAB[5] = {
    {0, {0}, {{0}}, {0}},
    {1, {0}, {{0}}, {1}},                                                            /* explicit Euler  */
    {2, {0, 1}, {{0}, {1}}, {0.5, 0.5}},                                             /* Heun, order 2   */
    {3, {0, 1.0 / 3, 2.0 / 3}, {{0}, {1.0 / 3}, {0, 2.0 / 3}}, {0.25, 0, 0.75}},     /* Heun, order 3   */
    {4, {0, 0.5, 0.5, 1}, {{0}, {0.5}, {0, 0.5}, {0, 0, 1}}, {1.0 / 6, 1.0 / 3, 1.0 / 3, 1.0 / 6}}, /* RK4 */
};

typedef struct {
  int scheme, N, max_depth;
  double c_rk, L;
  orc_medium_fn fn;
  void* ctx;
  int depth, capped, near_threshold;
} seg_scheme;

static void bg_at(seg_scheme* q, double x, double* beta, double gamma[3]) { q->fn(q->ctx, q->L - x, beta, gamma); }

/* the split test of Alg. 1; flags decisions within 1e-4 of the threshold */
static int split_test(seg_scheme* q, double dx, double beta) {
  if (!(q->c_rk > 0.0)) return 0;
  if (fabs(dx * beta - q->c_rk) <= 1e-4 * q->c_rk) q->near_threshold = 1;
  return dx * beta > q->c_rk;
}

static void segeval(seg_scheme* q, double x1, double x2, int d, double* A, double B[3]) {
  const double dx = x2 - x1;
  if (d > q->depth) q->depth = d;
  int split = 0;
  double beta[64], gamma[64][3];
  if (q->scheme >= ORC_EULER && q->scheme <= ORC_RK4) {
    const rk_tableau* T = &RK_TAB[q->scheme];
    double Ab[5], Bb[5][3];
    for (int i = 0; i <= T->M && !split; ++i) {
      /* stage i, Eq. RKresultAB (a_Mj = b_j for the final values) */
      Ab[i] = 1.0;
      Bb[i][0] = Bb[i][1] = Bb[i][2] = 0.0;
      for (int j = 0; j < i; ++j) {
        const double aij = (i == T->M) ? T->b[j] : T->a[i][j];
        Ab[i] += dx * aij * (-beta[j] * Ab[j]);
        for (int c = 0; c < 3; ++c) Bb[i][c] += dx * aij * (gamma[j][c] - beta[j] * Bb[j][c]);
      }
      if (i > 0 && split_test(q, dx, beta[i - 1])) split = 1;   /* Alg. 1 */
      if (!split && i < T->M) bg_at(q, x1 + T->c[i] * dx, &beta[i], gamma[i]);
    }
    if (!split) {
      *A = Ab[T->M];
      for (int c = 0; c < 3; ++c) B[c] = Bb[T->M][c];
    }
  } else if (q->scheme == ORC_GAUSS2) {
    const double xi[2] = {0.5 - sqrt(3.0) / 6.0, 0.5 + sqrt(3.0) / 6.0};   /* DESIGN.md D6 */
    for (int j = 0; j < 2; ++j) {
      bg_at(q, x1 + xi[j] * dx, &beta[j], gamma[j]);
      split |= split_test(q, dx, beta[j]);
    }
    if (!split) {   /* Eq. gaussAB, Eq. gaussABab */
      const double a1 = dx * (beta[0] + beta[1]) / 4.0, a2 = dx * dx * beta[0] * beta[1] / 12.0;
      *A = (1.0 - a1 + a2) / (1.0 + a1 + a2);
      for (int c = 0; c < 3; ++c) {
        const double b1 = dx * (gamma[0][c] + gamma[1][c]) / 2.0;
        const double b2 = dx * dx * (beta[0] * gamma[1][c] - beta[1] * gamma[0][c]) * sqrt(3.0) / 12.0;
        B[c] = (b1 + b2) / (1.0 + a1 + a2);
      }
    }
  } else if (q->scheme == ORC_SIMPSON) {
    const double cj[3] = {0.0, 0.5, 1.0}, bj[3] = {1.0 / 6, 4.0 / 6, 1.0 / 6};
    for (int j = 0; j < 3; ++j) {
      bg_at(q, x1 + cj[j] * dx, &beta[j], gamma[j]);
      split |= split_test(q, dx, beta[j]);
    }
    if (!split) {   /* Eq. simpson */
      double sb = 0.0;
      for (int j = 0; j < 3; ++j) sb += bj[j] * beta[j];
      *A = exp(-dx * sb);
      for (int c = 0; c < 3; ++c)
        B[c] = dx * (bj[0] * *A * gamma[0][c] + bj[1] * sqrt(*A) * gamma[1][c] + bj[2] * gamma[2][c]);
    }
  } else {   /* ORC_GL: the R13 rule on [x1, x2], nodes u_j from the downstream (near) end */
    double u[64], w[64], S[64 * 64];
    orc_gauss_legendre(q->N, u, w);
    orc_lagrange_integrals(q->N, u, S);
    for (int j = 0; j < q->N; ++j) {
      bg_at(q, x2 - u[j] * dx, &beta[j], gamma[j]);
      split |= split_test(q, dx, beta[j]);
    }
    if (!split) {
      double sum = 0.0;
      for (int j = 0; j < q->N; ++j) sum += w[j] * beta[j];
      *A = exp(-dx * sum);
      B[0] = B[1] = B[2] = 0.0;
      for (int j = 0; j < q->N; ++j) {
        double tau = 0.0;
        for (int k = 0; k < q->N; ++k) tau += S[j * q->N + k] * beta[k];
        for (int c = 0; c < 3; ++c) B[c] += dx * w[j] * gamma[j][c] * exp(-dx * tau);
      }
    }
  }
  if (split) {
    if (d >= q->max_depth) {   /* depth cap: report, and take the step without the test */
      q->capped = 1;
      const double keep = q->c_rk;
      q->c_rk = 0.0;
      segeval(q, x1, x2, d, A, B);
      q->c_rk = keep;
      return;
    }
    const double xm = 0.5 * (x1 + x2);
    double An, Bn[3], Af, Bf[3];
    segeval(q, xm, x2, d + 1, &An, Bn);   /* downstream (near) half */
    segeval(q, x1, xm, d + 1, &Af, Bf);   /* upstream (far) half */
    for (int c = 0; c < 3; ++c) orc_combine(An, Bn[c], Af, Bf[c], A, &B[c]);   /* near (+) far */
  }
}

int orc_segment_scheme(int scheme, int N, double c_rk, int max_depth, orc_medium_fn fn, void* ctx, double L,
                       double* a, double b[3], int* flags) {
  seg_scheme q = {scheme, N, max_depth, c_rk, L, fn, ctx, 0, 0, 0};
  if (!(L > 0.0)) {
    *a = 1.0;
    b[0] = b[1] = b[2] = 0.0;
    if (flags) *flags = 0;
    return 0;
  }
  segeval(&q, 0.0, L, 0, a, b);
  if (flags) *flags = (q.capped ? 1 : 0) | (q.near_threshold ? 2 : 0);
  return q.depth;
}

static int g_scheme = ORC_GL, g_scheme_depth = 24;
static double g_scheme_crk = 0.0;
void orc_set_scheme(int scheme, double c_rk, int max_depth) {
  g_scheme = scheme;
  g_scheme_crk = c_rk;
  g_scheme_depth = max_depth;
}

/* ======================================================================
 * Geometry.  Gauss-Lobatto nodes, Lagrange
 * basis (Eq. nodal), tensor-product map (Eq. tensorgeom),
 * element = subcube of the tree.
 * ==================================================================== */
void orc_gll(int R, double* eta) {
  if (R == 1) { eta[0] = 0.0; eta[1] = 1.0; }
  else { eta[0] = 0.0; eta[1] = 0.5; eta[2] = 1.0; }   /* R = 2 */
}

void orc_lagrange(int R, const double* eta, double t, double* psi, double* dpsi) {
  for (int m = 0; m <= R; ++m) {
    double v = 1.0, dv = 0.0;
    for (int q = 0; q <= R; ++q) {
      if (q == m) continue;
      double f = (t - eta[q]) / (eta[m] - eta[q]);
      double df = 1.0 / (eta[m] - eta[q]);
      dv = dv * f + v * df;
      v *= f;
    }
    psi[m] = v;
    if (dpsi) dpsi[m] = dv;
  }
}

static void tree_map_jac(const orc_scene* sc, int k, const double t[3], double x[3], double dxdt[9]) {
  int R = sc->R, n1 = R + 1;
  double eta[3], p[3][3], dp[3][3];
  orc_gll(R, eta);
  for (int d = 0; d < 3; ++d) orc_lagrange(R, eta, t[d], p[d], dp[d]);
  for (int c = 0; c < 3; ++c) x[c] = 0.0;
  if (dxdt) for (int c = 0; c < 9; ++c) dxdt[c] = 0.0;
  const double* z = sc->tree_ctrl + (size_t)k * n1 * n1 * n1 * 3;
  for (int m3 = 0; m3 < n1; ++m3)
    for (int m2 = 0; m2 < n1; ++m2)
      for (int m1 = 0; m1 < n1; ++m1) {
        const double* zz = z + ((m3 * n1 + m2) * n1 + m1) * 3;
        double s = p[0][m1] * p[1][m2] * p[2][m3];
        double s1 = dp[0][m1] * p[1][m2] * p[2][m3];
        double s2 = p[0][m1] * dp[1][m2] * p[2][m3];
        double s3 = p[0][m1] * p[1][m2] * dp[2][m3];
        for (int c = 0; c < 3; ++c) {
          x[c] += zz[c] * s;
          if (dxdt) {
            dxdt[c * 3 + 0] += zz[c] * s1;
            dxdt[c * 3 + 1] += zz[c] * s2;
            dxdt[c * 3 + 2] += zz[c] * s3;
          }
        }
      }
}

void orc_tree_map(const orc_scene* sc, int k, const double t[3], double x[3]) {
  tree_map_jac(sc, k, t, x, NULL);
}

static double elem_h(const orc_scene* sc, int64_t e) { return ldexp(1.0, -(int)sc->level[e]); }

/* X_E(xi) = J_k(a 2^-18 + 2^-l xi); J = dX_E/dxi (row c, column d). */
void orc_element_map(const orc_scene* sc, int64_t e, const double xi[3], double x[3], double J[9]) {
  double h = elem_h(sc, e), t[3], dt[9];
  for (int d = 0; d < 3; ++d) t[d] = ldexp((double)sc->anchor[3 * e + d], -MAXL) + h * xi[d];
  tree_map_jac(sc, sc->tree[e], t, x, J ? dt : NULL);
  if (J) for (int c = 0; c < 9; ++c) J[c] = h * dt[c];
}

/* Eq. camerageometry; orthographic per SURVEY R4. */
void orc_camera_transform(const orc_camera* cam, const double x[3], double X[3]) {
  double d[3] = {x[0] - cam->origin[0], x[1] - cam->origin[1], x[2] - cam->origin[2]};
  double n = sqrt(cam->view[0] * cam->view[0] + cam->view[1] * cam->view[1] + cam->view[2] * cam->view[2]);
  X[0] = cam->right[0] * d[0] + cam->right[1] * d[1] + cam->right[2] * d[2];
  X[1] = cam->up[0] * d[0] + cam->up[1] * d[1] + cam->up[2] * d[2];
  X[2] = (cam->view[0] * d[0] + cam->view[1] * d[1] + cam->view[2] * d[2]) / n;
}

/* Eq. ray: o + alpha r, r = v + l((i-(w-1)/2) t + (j-(h-1)/2) u).
 * Orthographic: origin P0 + l(...), direction d. */
void orc_ray(const orc_camera* cam, int i, int j, double o[3], double r[3]) {
  double di = cam->pixel_size * (i - 0.5 * (cam->width - 1));
  double dj = cam->pixel_size * (j - 0.5 * (cam->height - 1));
  for (int c = 0; c < 3; ++c) {
    double off = di * cam->right[c] + dj * cam->up[c];
    if (cam->projection == 0) {
      o[c] = cam->origin[c];
      r[c] = cam->view[c] + off;
    } else {
      o[c] = cam->origin[c] + off;
      r[c] = cam->view[c];
    }
  }
}

static double cam_n(const orc_camera* cam) {
  return sqrt(cam->view[0] * cam->view[0] + cam->view[1] * cam->view[1] + cam->view[2] * cam->view[2]);
}
static void alpha_range(const orc_camera* cam, double* amin, double* amax) {
  if (cam->projection == 0) { *amin = 1.0; *amax = cam->far_dist / cam_n(cam); }   /* Z in [n,f] */
  else { *amin = 0.0; *amax = cam->far_dist; }
}

/* Bernstein-Bezier control points of the element map restricted to the
 * parameter box [lo,hi]^3 (for R=2 per axis b1 = 2 y(1/2) - (y0+y2)/2;
 * SURVEY R6).  Lagrange values are plain evaluations of X_E. */
static void element_bezier(const orc_scene* sc, int64_t e, const double lo[3], const double hi[3],
                           double B[27][3]) {
  int R = sc->R, n1 = R + 1;
  double eta[3];
  orc_gll(R, eta);
  double Y[27][3];
  for (int m3 = 0; m3 < n1; ++m3)
    for (int m2 = 0; m2 < n1; ++m2)
      for (int m1 = 0; m1 < n1; ++m1) {
        double xi[3] = {lo[0] + (hi[0] - lo[0]) * eta[m1], lo[1] + (hi[1] - lo[1]) * eta[m2],
                        lo[2] + (hi[2] - lo[2]) * eta[m3]};
        orc_element_map(sc, e, xi, Y[(m3 * n1 + m2) * n1 + m1], NULL);
      }
  memcpy(B, Y, sizeof(double) * 3 * n1 * n1 * n1);
  if (R == 2) {
    /* apply the 1D Lagrange->Bernstein conversion along each axis */
    for (int ax = 0; ax < 3; ++ax)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          int idx[3];
          for (int m = 0; m < 3; ++m) {
            int c3[3];
            c3[ax] = m;
            c3[(ax + 1) % 3] = a;
            c3[(ax + 2) % 3] = b;
            idx[m] = (c3[2] * 3 + c3[1]) * 3 + c3[0];
          }
          for (int c = 0; c < 3; ++c)
            B[idx[1]][c] = 2.0 * B[idx[1]][c] - 0.5 * (B[idx[0]][c] + B[idx[2]][c]);
        }
  }
}

/* Camera-space AABB of the element's Bezier points. */
static void surface_corners(const orc_scene* sc, int64_t e, double P[2][2][3]);
static int is_surface(const orc_scene* sc);
int orc_element_aabb(const orc_scene* sc, const orc_camera* cam, int64_t e, double lo[3], double hi[3]) {
  if (is_surface(sc)) {   /* a bilinear patch lies in the convex hull of its four corners */
    double P[2][2][3];
    surface_corners(sc, e, P);
    for (int c = 0; c < 3; ++c) { lo[c] = INFINITY; hi[c] = -INFINITY; }
    for (int q = 0; q < 4; ++q) {
      double X[3];
      orc_camera_transform(cam, P[q / 2][q % 2], X);
      for (int c = 0; c < 3; ++c) { lo[c] = fmin(lo[c], X[c]); hi[c] = fmax(hi[c], X[c]); }
    }
    return 0;
  }
  double B[27][3], plo[3] = {0, 0, 0}, phi[3] = {1, 1, 1};
  element_bezier(sc, e, plo, phi, B);
  int np = (sc->R + 1) * (sc->R + 1) * (sc->R + 1);
  for (int c = 0; c < 3; ++c) { lo[c] = INFINITY; hi[c] = -INFINITY; }
  for (int m = 0; m < np; ++m) {
    double X[3];
    orc_camera_transform(cam, B[m], X);
    for (int c = 0; c < 3; ++c) { lo[c] = fmin(lo[c], X[c]); hi[c] = fmax(hi[c], X[c]); }
  }
  return 0;
}

/* Pixel-centre rectangle of a camera-space AABB:
 * p = (n/l) X/Z + (w-1)/2 with Z clamped >= n (perspective), p = X/l + (w-1)/2
 * (orthographic); rect = [ceil pmin, floor pmax] clipped to the image.
 * Returns 1 if non-empty. */
int orc_pixel_rect(const orc_camera* cam, const double lo[3], const double hi[3], int32_t rect[4]) {
  double n = cam_n(cam), l = cam->pixel_size;
  double pmin[2], pmax[2];
  int dims[2] = {cam->width, cam->height};
  rect[0] = 0; rect[1] = -1; rect[2] = 0; rect[3] = -1;
  if (cam->projection == 0) {
    if (hi[2] < n || lo[2] > cam->far_dist) return 0;
    double Z[2] = {fmax(lo[2], n), fmax(hi[2], n)};
    for (int d = 0; d < 2; ++d) {
      double X[2] = {lo[d], hi[d]};
      pmin[d] = INFINITY; pmax[d] = -INFINITY;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          double p = (n / l) * X[a] / Z[b] + 0.5 * (dims[d] - 1);
          pmin[d] = fmin(pmin[d], p);
          pmax[d] = fmax(pmax[d], p);
        }
    }
  } else {
    if (hi[2] < 0.0 || lo[2] > cam->far_dist) return 0;
    for (int d = 0; d < 2; ++d) {
      pmin[d] = lo[d] / l + 0.5 * (dims[d] - 1);
      pmax[d] = hi[d] / l + 0.5 * (dims[d] - 1);
    }
  }
  for (int d = 0; d < 2; ++d) {
    double a = ceil(pmin[d]), b = floor(pmax[d]);
    if (a < 0) a = 0;
    if (b > dims[d] - 1) b = dims[d] - 1;
    if (a > b) return 0;
    rect[2 * d] = (int32_t)a;
    rect[2 * d + 1] = (int32_t)b;
  }
  return 1;
}

/* Culled list: visible iff the pixel-centre rect is
 * non-empty; ambiguous iff the decision differs for the AABB inflated and
 * deflated by EPS_AMBIG.  rects[4n] receives the EPS-inflated rect (superset
 * used for candidate pairs). */
void orc_cull(const orc_scene* sc, const orc_camera* cam, int8_t* visible, int8_t* ambiguous,
              int32_t* rects) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < sc->n; ++e) {
    double lo[3], hi[3], lp[3], hp[3], lm[3], hm[3];
    int32_t r0[4], rp[4], rm[4];
    orc_element_aabb(sc, cam, e, lo, hi);
    for (int c = 0; c < 3; ++c) {
      lp[c] = lo[c] - EPS_AMBIG; hp[c] = hi[c] + EPS_AMBIG;
      lm[c] = lo[c] + EPS_AMBIG; hm[c] = hi[c] - EPS_AMBIG;
    }
    int v0 = orc_pixel_rect(cam, lo, hi, r0);
    int vp = orc_pixel_rect(cam, lp, hp, rp);
    int vm = orc_pixel_rect(cam, lm, hm, rm);
    visible[e] = (int8_t)v0;
    ambiguous[e] = (int8_t)(vp != vm);
    if (rects) {
      if (vp) memcpy(rects + 4 * e, rp, sizeof rp);
      else { rects[4 * e] = 0; rects[4 * e + 1] = -1; rects[4 * e + 2] = 0; rects[4 * e + 3] = -1; }
    }
  }
}

/* Nodal field interpolation at element-local GLL nodes. */
double orc_field(const orc_scene* sc, int64_t e, const double xi[3]) {
  int P = sc->P, n1 = P + 1;
  double eta[3], p[3][3];
  orc_gll(P, eta);
  for (int d = 0; d < 3; ++d) orc_lagrange(P, eta, xi[d], p[d], NULL);
  const float* f = sc->field + (size_t)e * n1 * n1 * n1;
  double v = 0.0;
  for (int k3 = 0; k3 < n1; ++k3)
    for (int k2 = 0; k2 < n1; ++k2)
      for (int k1 = 0; k1 < n1; ++k1) v += (double)f[(k3 * n1 + k2) * n1 + k1] * p[0][k1] * p[1][k2] * p[2][k3];
  return v;
}

static int solve3(const double A[9], const double b[3], double x[3]) {
  double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
               A[2] * (A[3] * A[7] - A[4] * A[6]);
  if (det == 0.0 || !isfinite(det)) return -1;
  double inv[9];
  inv[0] = (A[4] * A[8] - A[5] * A[7]) / det;
  inv[1] = (A[2] * A[7] - A[1] * A[8]) / det;
  inv[2] = (A[1] * A[5] - A[2] * A[4]) / det;
  inv[3] = (A[5] * A[6] - A[3] * A[8]) / det;
  inv[4] = (A[0] * A[8] - A[2] * A[6]) / det;
  inv[5] = (A[2] * A[3] - A[0] * A[5]) / det;
  inv[6] = (A[3] * A[7] - A[4] * A[6]) / det;
  inv[7] = (A[1] * A[6] - A[0] * A[7]) / det;
  inv[8] = (A[0] * A[4] - A[1] * A[3]) / det;
  for (int r = 0; r < 3; ++r) x[r] = inv[3 * r] * b[0] + inv[3 * r + 1] * b[1] + inv[3 * r + 2] * b[2];
  return 0;
}

/* xi with X_E(xi) = x by Newton in fp64, started from the
 * affine model at the element centre.  Returns 0 on convergence. */
int orc_inverse_map(const orc_scene* sc, int64_t e, const double x[3], double xi[3]) {
  double c[3] = {0.5, 0.5, 0.5}, X[3], J[9], rhs[3], d[3];
  orc_element_map(sc, e, c, X, J);
  for (int k = 0; k < 3; ++k) rhs[k] = x[k] - X[k];
  if (solve3(J, rhs, d)) return -1;
  for (int k = 0; k < 3; ++k) xi[k] = 0.5 + d[k];
  double prev = INFINITY;
  for (int it = 0; it < 80; ++it) {
    orc_element_map(sc, e, xi, X, J);
    for (int k = 0; k < 3; ++k) rhs[k] = x[k] - X[k];
    if (solve3(J, rhs, d)) return -1;
    for (int k = 0; k < 3; ++k) xi[k] += d[k];
    double st = fmax(fabs(d[0]), fmax(fabs(d[1]), fabs(d[2])));
    /* converged: step below 1e-12, or stagnating at the fp64 rounding floor
     * (|x| ~ 1 against elements of size h gives ~1e-16/h noise in xi) */
    if (st < 1e-12 || (st < 1e-9 && st >= 0.5 * prev)) return 0;
    prev = st;
    if (!(fabs(xi[0]) < 1e6 && fabs(xi[1]) < 1e6 && fabs(xi[2]) < 1e6)) return -1;
  }
  return -2;
}

/* ======================================================================
 * Intersection (App. A.1).
 * Affine trees: slab test in reference coordinates.  General trees: all
 * roots on each face by Bezier subdivision of the projected patch (Eq.
 * intersectiontwod, d1,d2 perpendicular to r) + fp64 Newton; inside/outside
 * of each interval between consecutive roots decided by the inverse map.
 * ==================================================================== */
static int g_force_general = 0;
/* test hook: route affine trees through the general face-root path */
void orc_set_force_general(int on) { g_force_general = on; }

static int tree_affine(const orc_scene* sc, int k, double c[3], double M[9]) {
  if (g_force_general) return 0;
  double t0[3] = {0, 0, 0}, x[3];
  orc_tree_map(sc, k, t0, c);
  for (int d = 0; d < 3; ++d) {
    double t[3] = {0, 0, 0};
    t[d] = 1.0;
    orc_tree_map(sc, k, t, x);
    for (int q = 0; q < 3; ++q) M[q * 3 + d] = x[q] - c[q];
  }
  int R = sc->R, n1 = R + 1;
  double eta[3];
  orc_gll(R, eta);
  const double* z = sc->tree_ctrl + (size_t)k * n1 * n1 * n1 * 3;
  for (int m3 = 0; m3 < n1; ++m3)
    for (int m2 = 0; m2 < n1; ++m2)
      for (int m1 = 0; m1 < n1; ++m1) {
        const double* zz = z + ((m3 * n1 + m2) * n1 + m1) * 3;
        double et[3] = {eta[m1], eta[m2], eta[m3]};
        for (int q = 0; q < 3; ++q) {
          double v = c[q] + M[q * 3] * et[0] + M[q * 3 + 1] * et[1] + M[q * 3 + 2] * et[2];
          if (fabs(v - zz[q]) > 1e-13 * (1.0 + fabs(zz[q]))) return 0;
        }
      }
  return 1;
}

static void inv3(const double A[9], double inv[9]) {
  double e[3], x[3];
  for (int col = 0; col < 3; ++col) {
    e[0] = e[1] = e[2] = 0.0;
    e[col] = 1.0;
    solve3(A, e, x);
    for (int r = 0; r < 3; ++r) inv[r * 3 + col] = x[r];
  }
}

/* slab test of the ray against xi in [lo_k, hi_k]; returns 1 and [a0,a1] on hit */
static int slab(const double xi0[3], const double dxi[3], const double lo[3], const double hi[3],
                double amin, double amax, double* a0, double* a1) {
  double enter = amin, exit_ = amax;
  for (int k = 0; k < 3; ++k) {
    if (dxi[k] == 0.0) {
      if (xi0[k] < lo[k] || xi0[k] > hi[k]) return 0;
      continue;
    }
    double t0 = (lo[k] - xi0[k]) / dxi[k], t1 = (hi[k] - xi0[k]) / dxi[k];
    if (t0 > t1) { double tt = t0; t0 = t1; t1 = tt; }
    if (t0 > enter) enter = t0;
    if (t1 < exit_) exit_ = t1;
  }
  if (exit_ > enter) { *a0 = enter; *a1 = exit_; return 1; }
  return 0;
}

typedef struct { double alpha, cosphi, xi[3]; } froot;

typedef struct {
  const orc_scene* sc; int64_t e; int fixk; double fixv; int ax, bx;
  double lo_a, hi_a, lo_b, hi_b;
  double o[3], r[3], d1[3], d2[3];
  froot* roots; int nroots, cap, boxes, fail;
} face_ctx;

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

static void face_point(face_ctx* f, double s1, double s2, double xi[3]) {
  xi[f->fixk] = f->fixv;
  xi[f->ax] = f->lo_a + (f->hi_a - f->lo_a) * s1;
  xi[f->bx] = f->lo_b + (f->hi_b - f->lo_b) * s2;
}

/* Newton on the projected system G(xi_a, xi_b) = (d1.(X-o), d2.(X-o)) = 0 */
static int face_newton(face_ctx* f, double s1, double s2, froot* out, double* so1, double* so2) {
  double xi[3], X[3], J[9];
  face_point(f, s1, s2, xi);
  double prev = INFINITY;
  for (int it = 0; it < 60; ++it) {
    orc_element_map(f->sc, f->e, xi, X, J);
    double dx[3] = {X[0] - f->o[0], X[1] - f->o[1], X[2] - f->o[2]};
    double g1 = dot3(f->d1, dx), g2 = dot3(f->d2, dx);
    double Xa[3] = {J[f->ax], J[3 + f->ax], J[6 + f->ax]};
    double Xb[3] = {J[f->bx], J[3 + f->bx], J[6 + f->bx]};
    double j11 = dot3(f->d1, Xa), j12 = dot3(f->d1, Xb), j21 = dot3(f->d2, Xa), j22 = dot3(f->d2, Xb);
    double det = j11 * j22 - j12 * j21;
    if (det == 0.0 || !isfinite(det)) return -1;
    double da = (g1 * j22 - g2 * j12) / det, db = (j11 * g2 - j21 * g1) / det;
    xi[f->ax] -= da;
    xi[f->bx] -= db;
    if (!(fabs(xi[f->ax]) < 10 && fabs(xi[f->bx]) < 10)) return -1;
    double st = fmax(fabs(da), fabs(db));
    if (st < 1e-12 || (st < 1e-9 && st >= 0.5 * prev)) {   /* see orc_inverse_map */
      orc_element_map(f->sc, f->e, xi, X, J);
      double Xa2[3] = {J[f->ax], J[3 + f->ax], J[6 + f->ax]};
      double Xb2[3] = {J[f->bx], J[3 + f->bx], J[6 + f->bx]};
      double nrm[3];
      cross3(Xa2, Xb2, nrm);
      double rr = dot3(f->r, f->r);
      out->alpha = dot3(f->r, (double[3]){X[0] - f->o[0], X[1] - f->o[1], X[2] - f->o[2]}) / rr;
      out->cosphi = fabs(dot3(nrm, f->r)) / (sqrt(dot3(nrm, nrm)) * sqrt(rr));
      memcpy(out->xi, xi, sizeof xi);
      *so1 = (xi[f->ax] - f->lo_a) / (f->hi_a - f->lo_a);
      *so2 = (xi[f->bx] - f->lo_b) / (f->hi_b - f->lo_b);
      return 0;
    }
    prev = st;
  }
  return -2;
}

/* de Casteljau split of a degree-R Bernstein patch g[(R+1)^2][2] along s1
 * (dir 0) or s2 (dir 1) at 1/2. */
static void bz_split(int R, const double g[9][2], int dir, double L[9][2], double H[9][2]) {
  int n1 = R + 1;
  for (int o = 0; o < n1; ++o) {
    double row[3][2];
    for (int m = 0; m < n1; ++m) {
      int idx = dir == 0 ? o * n1 + m : m * n1 + o;
      row[m][0] = g[idx][0];
      row[m][1] = g[idx][1];
    }
    double lo[3][2], hi[3][2];
    if (R == 1) {
      double mid[2] = {0.5 * (row[0][0] + row[1][0]), 0.5 * (row[0][1] + row[1][1])};
      lo[0][0] = row[0][0]; lo[0][1] = row[0][1]; lo[1][0] = mid[0]; lo[1][1] = mid[1];
      hi[0][0] = mid[0]; hi[0][1] = mid[1]; hi[1][0] = row[1][0]; hi[1][1] = row[1][1];
    } else {
      for (int c = 0; c < 2; ++c) {
        double a01 = 0.5 * (row[0][c] + row[1][c]), a12 = 0.5 * (row[1][c] + row[2][c]);
        double a = 0.5 * (a01 + a12);
        lo[0][c] = row[0][c]; lo[1][c] = a01; lo[2][c] = a;
        hi[0][c] = a; hi[1][c] = a12; hi[2][c] = row[2][c];
      }
    }
    for (int m = 0; m < n1; ++m) {
      int idx = dir == 0 ? o * n1 + m : m * n1 + o;
      L[idx][0] = lo[m][0]; L[idx][1] = lo[m][1];
      H[idx][0] = hi[m][0]; H[idx][1] = hi[m][1];
    }
  }
}

static void face_subdiv(face_ctx* f, const double g[9][2], double s1a, double s1b, double s2a,
                        double s2b) {
  int R = f->sc->R, np = (R + 1) * (R + 1);
  if (++f->boxes > 400000) { if (getenv("ORC_DEBUG")) fprintf(stderr, "box limit face %d\n", f->fixk); f->fail = 1; return; }
  double mn[2] = {INFINITY, INFINITY}, mx[2] = {-INFINITY, -INFINITY};
  for (int m = 0; m < np; ++m)
    for (int c = 0; c < 2; ++c) { mn[c] = fmin(mn[c], g[m][c]); mx[c] = fmax(mx[c], g[m][c]); }
  if (mn[0] > 0 || mx[0] < 0 || mn[1] > 0 || mx[1] < 0) return;   /* hull excludes the ray */
  double width = fmax(s1b - s1a, s2b - s2a);
  if (width < 1e-3) {
    /* Newton from the box centre; a root it lands on inside this box is
     * accepted.  If it leaves the box (ill-conditioned grazing rays can jump
     * to another root), keep subdividing: the hull test alone converges to
     * every root (exhaustive Bezier subdivision). */
    froot rt;
    double so1, so2;
    if (face_newton(f, 0.5 * (s1a + s1b), 0.5 * (s2a + s2b), &rt, &so1, &so2) == 0) {
      double tol = 1e-9;
      if (so1 >= s1a - tol && so1 <= s1b + tol && so2 >= s2a - tol && so2 <= s2b + tol) {
        if (so1 >= -1e-12 && so1 <= 1 + 1e-12 && so2 >= -1e-12 && so2 <= 1 + 1e-12) {
          if (f->nroots < f->cap) f->roots[f->nroots++] = rt;
          else f->fail = 1;
        }
        return;
      }
    }
    if (width < 1e-11) {   /* converged by subdivision alone: accept the box centre */
      double xi[3], X[3], J[9], nrm[3];
      face_point(f, 0.5 * (s1a + s1b), 0.5 * (s2a + s2b), xi);
      orc_element_map(f->sc, f->e, xi, X, J);
      double Xa[3] = {J[f->ax], J[3 + f->ax], J[6 + f->ax]}, Xb[3] = {J[f->bx], J[3 + f->bx], J[6 + f->bx]};
      cross3(Xa, Xb, nrm);
      double rr = dot3(f->r, f->r);
      froot rt2;
      rt2.alpha = dot3(f->r, (double[3]){X[0] - f->o[0], X[1] - f->o[1], X[2] - f->o[2]}) / rr;
      rt2.cosphi = fabs(dot3(nrm, f->r)) / (sqrt(dot3(nrm, nrm)) * sqrt(rr));
      memcpy(rt2.xi, xi, sizeof xi);
      double m1 = 0.5 * (s1a + s1b), m2 = 0.5 * (s2a + s2b);
      if (m1 >= 0 && m1 <= 1 && m2 >= 0 && m2 <= 1) {
        if (f->nroots < f->cap) f->roots[f->nroots++] = rt2;
        else f->fail = 1;
      }
      return;
    }
  }
  double L[9][2], H[9][2];
  if (s1b - s1a >= s2b - s2a) {
    bz_split(R, g, 0, L, H);
    double sm = 0.5 * (s1a + s1b);
    face_subdiv(f, L, s1a, sm, s2a, s2b);
    face_subdiv(f, H, sm, s1b, s2a, s2b);
  } else {
    bz_split(R, g, 1, L, H);
    double sm = 0.5 * (s2a + s2b);
    face_subdiv(f, L, s1a, s1b, s2a, sm);
    face_subdiv(f, H, s1a, s1b, sm, s2b);
  }
}

static int cmp_froot(const void* a, const void* b) {
  double x = ((const froot*)a)->alpha, y = ((const froot*)b)->alpha;
  return (x > y) - (x < y);
}

static int inside_elem(const orc_scene* sc, int64_t e, const double lo[3], const double hi[3],
                       const double wlo[3], const double whi[3], const double p[3], int* fail) {
  for (int c = 0; c < 3; ++c)
    if (p[c] < wlo[c] || p[c] > whi[c]) return 0;
  double xi[3];
  if (orc_inverse_map(sc, e, p, xi) != 0) { if (getenv("ORC_DEBUG")) fprintf(stderr, "inverse map fail\n"); *fail = 1; return 0; }
  for (int k = 0; k < 3; ++k)
    if (xi[k] < lo[k] || xi[k] > hi[k]) return 0;
  return 1;
}

/* general-geometry intersection with parameter domain [lo,hi]^3 */
static int general_segments(const orc_scene* sc, int64_t e, const double o[3], const double r[3],
                            double amin, double amax, const double lo[3], const double hi[3], int max_seg,
                            double* seg, int* flags) {
  froot roots[96];
  int nr = 0, fail = 0;
  double d1[3], d2[3], ax[3] = {0, 0, 0};
  /* d1, d2 orthonormal, perpendicular to r */
  int im = 0;
  for (int c = 1; c < 3; ++c)
    if (fabs(r[c]) < fabs(r[im])) im = c;
  ax[im] = 1.0;
  cross3(r, ax, d1);
  double nd = sqrt(dot3(d1, d1));
  for (int c = 0; c < 3; ++c) d1[c] /= nd;
  cross3(r, d1, d2);
  nd = sqrt(dot3(d2, d2));
  for (int c = 0; c < 3; ++c) d2[c] /= nd;

  int R = sc->R, n1 = R + 1;
  double eta[3];
  orc_gll(R, eta);
  for (int fidx = 0; fidx < 6; ++fidx) {
    face_ctx f;
    memset(&f, 0, sizeof f);
    f.sc = sc; f.e = e; f.fixk = fidx / 2;
    f.fixv = (fidx % 2) ? hi[f.fixk] : lo[f.fixk];
    f.ax = (f.fixk + 1) % 3; f.bx = (f.fixk + 2) % 3;
    f.lo_a = lo[f.ax]; f.hi_a = hi[f.ax]; f.lo_b = lo[f.bx]; f.hi_b = hi[f.bx];
    memcpy(f.o, o, sizeof f.o); memcpy(f.r, r, sizeof f.r);
    memcpy(f.d1, d1, sizeof d1); memcpy(f.d2, d2, sizeof d2);
    f.roots = roots + nr;
    f.cap = 96 - nr;
    /* projected face polynomial in Bernstein form (affine projection commutes) */
    double g[9][2];
    for (int m2 = 0; m2 < n1; ++m2)
      for (int m1 = 0; m1 < n1; ++m1) {
        double xi[3], X[3];
        face_point(&f, eta[m1], eta[m2], xi);
        orc_element_map(sc, e, xi, X, NULL);
        double dx[3] = {X[0] - o[0], X[1] - o[1], X[2] - o[2]};
        g[m2 * n1 + m1][0] = dot3(d1, dx);
        g[m2 * n1 + m1][1] = dot3(d2, dx);
      }
    if (R == 2) {
      for (int row = 0; row < 3; ++row)
        for (int c = 0; c < 2; ++c) {
          g[row * 3 + 1][c] = 2 * g[row * 3 + 1][c] - 0.5 * (g[row * 3][c] + g[row * 3 + 2][c]);
        }
      for (int col = 0; col < 3; ++col)
        for (int c = 0; c < 2; ++c) {
          g[3 + col][c] = 2 * g[3 + col][c] - 0.5 * (g[col][c] + g[6 + col][c]);
        }
    }
    face_subdiv(&f, g, 0.0, 1.0, 0.0, 1.0);
    nr += f.nroots;
    fail |= f.fail;
  }
  qsort(roots, nr, sizeof(froot), cmp_froot);
  if (getenv("ORC_DEBUG")) {
    fprintf(stderr, "roots %d:", nr);
    for (int q = 0; q < nr; ++q) fprintf(stderr, " (%.9f c%.2e xi %.4f %.4f %.4f)", roots[q].alpha, roots[q].cosphi, roots[q].xi[0], roots[q].xi[1], roots[q].xi[2]);
    fprintf(stderr, "\n");
  }
  /* dedupe roots found on several faces / sub-boxes */
  double rn = sqrt(dot3(r, r));
  int m = 0;
  for (int q = 0; q < nr; ++q) {
    if (m > 0 && fabs(roots[q].alpha - roots[m - 1].alpha) * rn < 1e-10) continue;
    roots[m++] = roots[q];
  }
  nr = m;
  for (int q = 0; q < nr; ++q)
    if (roots[q].cosphi < 1e-6) *flags |= ORC_AMBIGUOUS;   /* tangent */
  /* world AABB of the element restricted to [lo,hi] for a cheap outside test */
  double B[27][3], wlo[3], whi[3];
  element_bezier(sc, e, lo, hi, B);
  int np = n1 * n1 * n1;
  for (int c = 0; c < 3; ++c) { wlo[c] = INFINITY; whi[c] = -INFINITY; }
  for (int q = 0; q < np; ++q)
    for (int c = 0; c < 3; ++c) { wlo[c] = fmin(wlo[c], B[q][c]); whi[c] = fmax(whi[c], B[q][c]); }
  for (int c = 0; c < 3; ++c) { wlo[c] -= 1e-12; whi[c] += 1e-12; }
  /* breakpoints */
  double bp[100];
  int nb = 0;
  bp[nb++] = amin;
  for (int q = 0; q < nr; ++q)
    if (roots[q].alpha > amin && roots[q].alpha < amax) bp[nb++] = roots[q].alpha;
  bp[nb++] = amax;
  int nseg = 0, open = 0;
  double start = 0;
  for (int q = 0; q + 1 < nb; ++q) {
    double am = 0.5 * (bp[q] + bp[q + 1]);
    double p[3] = {o[0] + am * r[0], o[1] + am * r[1], o[2] + am * r[2]};
    int in = inside_elem(sc, e, lo, hi, wlo, whi, p, &fail);
    if (in && !open) { open = 1; start = bp[q]; }
    if (!in && open) {
      open = 0;
      if (nseg < max_seg) { seg[2 * nseg] = start; seg[2 * nseg + 1] = bp[q]; }
      nseg++;
    }
  }
  if (open) {
    if (nseg < max_seg) { seg[2 * nseg] = start; seg[2 * nseg + 1] = bp[nb - 1]; }
    nseg++;
  }
  if (fail) *flags |= ORC_NEWTON_FAIL | ORC_AMBIGUOUS;
  if (nseg > max_seg) { *flags |= ORC_OVERFLOW; nseg = max_seg; }
  return nseg;
}

static double min_edge(const orc_scene* sc, int64_t e, int k) {
  /* minimum length of the 4 element edges parallel to xi_k (corner chords) */
  double best = INFINITY;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double x0[3], x1[3], p0[3], p1[3];
      p0[k] = 0; p1[k] = 1;
      p0[(k + 1) % 3] = p1[(k + 1) % 3] = a;
      p0[(k + 2) % 3] = p1[(k + 2) % 3] = b;
      orc_element_map(sc, e, p0, x0, NULL);
      orc_element_map(sc, e, p1, x1, NULL);
      double d[3] = {x1[0] - x0[0], x1[1] - x0[1], x1[2] - x0[2]};
      best = fmin(best, sqrt(dot3(d, d)));
    }
  return best;
}

/* debug/test export: general-path segments with the parameter domain
 * [-delta, 1+delta]^3 (E+ for delta > 0, E- for delta < 0). */
int orc_intersect_domain(const orc_scene* sc, const orc_camera* cam, int64_t e, int i, int j, double delta,
                         int max_seg, double* seg, int* flags) {
  double o[3], r[3], amin, amax, lo[3], hi[3];
  orc_ray(cam, i, j, o, r);
  alpha_range(cam, &amin, &amax);
  for (int k = 0; k < 3; ++k) { lo[k] = -delta; hi[k] = 1 + delta; }
  *flags = 0;
  return general_segments(sc, e, o, r, amin, amax, lo, hi, max_seg, seg, flags);
}

/* Segments of the ray of pixel (i,j) inside element e (E0), with the
 * ambiguity classification of SURVEY R7: hit(E+) != hit(E-) where E+/- is
 * the element with its boundary pushed out/in by EPS_AMBIG, or a chord
 * < EPS_AMBIG, or a tangent root. */
/* ======================================================================
 * Surface forests (§2.8 "Visualization of surfaces", App.
 * A.1 PAPER.md:1473-1514).  An element is the bilinear
 * patch X_E(s) = J_k(a 2^-18 + 2^-l s), s in [0,1)^2, of its tree's bilinear
 * map (tree_ctrl [k][m2][m1][xyz]).  A ray meets it in points: projected on
 * d1, d2 perpendicular to r (Eq. intersectiontwod) the patch is the 2D
 * bilinear map g(s) = a + b s1 + c s2 + d s1 s2, and g(s) = 0 is a quadratic
 * in s2 after eliminating s1 (App. A.1).  Each point is a zero-length segment
 * with Eq. ABphi: A_phi = A_s^(1/cos phi), B_phi = I_s (1 - A_phi)
 * (Eq. BIrelation), phi the angle between the ray and the patch normal.
 * ==================================================================== */
static int is_surface(const orc_scene* sc) { return sc->dim == 2; }

/* corner points P[m2][m1] of the element's patch */
static void surface_corners(const orc_scene* sc, int64_t e, double P[2][2][3]) {
  const double* z = sc->tree_ctrl + (size_t)sc->tree[e] * 12;   /* [m2][m1][xyz] */
  const double h = elem_h(sc, e);
  for (int q2 = 0; q2 < 2; ++q2)
    for (int q1 = 0; q1 < 2; ++q1) {
      const double t1 = ldexp((double)sc->anchor[3 * e], -MAXL) + h * q1;
      const double t2 = ldexp((double)sc->anchor[3 * e + 1], -MAXL) + h * q2;
      for (int c = 0; c < 3; ++c)
        P[q2][q1][c] = (1 - t2) * ((1 - t1) * z[0 * 3 + c] + t1 * z[1 * 3 + c]) +
                       t2 * ((1 - t1) * z[2 * 3 + c] + t1 * z[3 * 3 + c]);
    }
}

static void surface_point(const double P[2][2][3], double s1, double s2, double X[3], double n[3]) {
  double d1[3], d2[3];
  for (int c = 0; c < 3; ++c) {
    X[c] = (1 - s2) * ((1 - s1) * P[0][0][c] + s1 * P[0][1][c]) + s2 * ((1 - s1) * P[1][0][c] + s1 * P[1][1][c]);
    d1[c] = (1 - s2) * (P[0][1][c] - P[0][0][c]) + s2 * (P[1][1][c] - P[1][0][c]);
    d2[c] = (1 - s1) * (P[1][0][c] - P[0][0][c]) + s1 * (P[1][1][c] - P[0][1][c]);
  }
  n[0] = d1[1] * d2[2] - d1[2] * d2[1];
  n[1] = d1[2] * d2[0] - d1[0] * d2[2];
  n[2] = d1[0] * d2[1] - d1[1] * d2[0];
}

/* All s in [lo, hi)^2 with X(s) on the ray line; returns the count (<= 2). */
static int surface_roots(const double P[2][2][3], const double o[3], const double r[3], double lo, double hi,
                         double s_out[2][2]) {
  double ax[3] = {0, 0, 0};   /* the coordinate axis least aligned with r */
  {
    const double a0 = fabs(r[0]), a1 = fabs(r[1]), a2 = fabs(r[2]);
    ax[(a0 <= a1 && a0 <= a2) ? 0 : (a1 <= a2 ? 1 : 2)] = 1.0;
  }
  double d1[3] = {r[1] * ax[2] - r[2] * ax[1], r[2] * ax[0] - r[0] * ax[2], r[0] * ax[1] - r[1] * ax[0]};
  double n1 = sqrt(dot3(d1, d1));
  for (int c = 0; c < 3; ++c) d1[c] /= n1;
  double d2[3] = {r[1] * d1[2] - r[2] * d1[1], r[2] * d1[0] - r[0] * d1[2], r[0] * d1[1] - r[1] * d1[0]};
  double n2 = sqrt(dot3(d2, d2));
  for (int c = 0; c < 3; ++c) d2[c] /= n2;
  double g[2][2][2];   /* projected corners [m2][m1][k] relative to the ray */
  for (int q2 = 0; q2 < 2; ++q2)
    for (int q1 = 0; q1 < 2; ++q1) {
      double rel[3] = {P[q2][q1][0] - o[0], P[q2][q1][1] - o[1], P[q2][q1][2] - o[2]};
      g[q2][q1][0] = dot3(d1, rel);
      g[q2][q1][1] = dot3(d2, rel);
    }
  double a[2], b[2], c[2], d[2];
  for (int k = 0; k < 2; ++k) {
    a[k] = g[0][0][k];
    b[k] = g[0][1][k] - g[0][0][k];
    c[k] = g[1][0][k] - g[0][0][k];
    d[k] = g[1][1][k] - g[1][0][k] - g[0][1][k] + g[0][0][k];
  }
  /* (a + c s2) x (b + d s2) = 0: q2 s2^2 + q1 s2 + q0 = 0 */
  const double q0 = a[0] * b[1] - a[1] * b[0];
  const double q1 = a[0] * d[1] - a[1] * d[0] + c[0] * b[1] - c[1] * b[0];
  const double qq = c[0] * d[1] - c[1] * d[0];
  double roots[2];
  int nr = 0;
  const double scale = fabs(q0) + fabs(q1) + fabs(qq);
  if (fabs(qq) <= 1e-14 * scale) {
    if (fabs(q1) > 0) roots[nr++] = -q0 / q1;
  } else {
    const double disc = q1 * q1 - 4 * qq * q0;
    if (disc >= 0) {
      const double sq = sqrt(disc);
      const double t = -0.5 * (q1 + (q1 >= 0 ? sq : -sq));   /* stable quadratic formula */
      roots[nr++] = t / qq;
      if (t != 0) roots[nr++] = q0 / t;
    }
  }
  int ns = 0;
  for (int k = 0; k < nr; ++k) {
    const double s2 = roots[k];
    if (!(s2 >= lo && s2 < hi)) continue;
    const double u[2] = {b[0] + d[0] * s2, b[1] + d[1] * s2};
    const double w[2] = {a[0] + c[0] * s2, a[1] + c[1] * s2};
    const double uu = u[0] * u[0] + u[1] * u[1];
    if (!(uu > 0)) continue;
    const double s1 = -(w[0] * u[0] + w[1] * u[1]) / uu;
    if (!(s1 >= lo && s1 < hi)) continue;
    s_out[ns][0] = s1;
    s_out[ns][1] = s2;
    ++ns;
  }
  return ns;
}

/* exported for the pins: P [2][2][3] ([m2][m1][xyz]), s_out [2][2] */
int orc_surface_roots(const double* P, const double o[3], const double r[3], double lo, double hi, double* s_out) {
  double Q[2][2][3], S[2][2];
  memcpy(Q, P, sizeof Q);
  const int ns = surface_roots(Q, o, r, lo, hi, S);
  memcpy(s_out, S, sizeof(double) * 2 * ns);
  return ns;
}

/* Surface hits of pixel (i,j)'s ray on element e: alpha and (a, b[3]) per point
 * (Eq. ABphi), at most 2; ambiguity as SURVEY R7 (s within eps / edge length of
 * the boundary, or |cos phi| < 1e-6). */
static int surface_hits(const orc_scene* sc, const orc_camera* cam, int64_t e, int i, int j, double* alpha,
                        double (*ab)[4], int* flags) {
  double o[3], r[3], amin, amax, P[2][2][3];
  orc_ray(cam, i, j, o, r);
  alpha_range(cam, &amin, &amax);
  surface_corners(sc, e, P);
  double emin = INFINITY;
  for (int q = 0; q < 2; ++q) {
    double e1[3], e2[3];
    for (int c = 0; c < 3; ++c) {
      e1[c] = P[q][1][c] - P[q][0][c];
      e2[c] = P[1][q][c] - P[0][q][c];
    }
    emin = fmin(emin, fmin(sqrt(dot3(e1, e1)), sqrt(dot3(e2, e2))));
  }
  const double delta = EPS_AMBIG / emin;
  double s[2][2], sp[2][2], sm[2][2];
  const int ns = surface_roots(P, o, r, 0.0, 1.0, s);
  const int np = surface_roots(P, o, r, -delta, 1.0 + delta, sp);
  const int nm = surface_roots(P, o, r, delta, 1.0 - delta, sm);
  (void)sp;
  (void)sm;
  *flags = 0;
  if (np != nm) *flags |= ORC_AMBIGUOUS;
  const double rr = dot3(r, r), rn = sqrt(rr);
  int nh = 0;
  for (int k = 0; k < ns; ++k) {
    double X[3], n[3];
    surface_point(P, s[k][0], s[k][1], X, n);
    const double al = ((X[0] - o[0]) * r[0] + (X[1] - o[1]) * r[1] + (X[2] - o[2]) * r[2]) / rr;
    if (!(al >= amin && al <= amax)) continue;
    const double cphi = fabs(dot3(n, r)) / (sqrt(dot3(n, n)) * rn);
    if (cphi < 1e-6) *flags |= ORC_AMBIGUOUS;
    /* the nodal value (bilinear in s, corners [k2][k1]) and the surface transfer */
    const float* f = sc->field + 4 * e;
    const double v = (1 - s[k][1]) * ((1 - s[k][0]) * f[0] + s[k][0] * f[1]) +
                     s[k][1] * ((1 - s[k][0]) * f[2] + s[k][0] * f[3]);
    double As = sc->surf_a[0] + sc->surf_a[1] * v;
    As = fmin(1.0, fmax(0.0, As));
    const double w = exp(-0.5 * ((1 - v) * sc->surf_k) * ((1 - v) * sc->surf_k));
    const double Aphi = (As == 0.0) ? 0.0 : pow(As, 1.0 / cphi);   /* Eq. ABphi (A_s = 0: opaque) */
    alpha[nh] = al;
    ab[nh][0] = Aphi;
    for (int c = 0; c < 3; ++c) {
      const double Is = sc->surf_i[c][0] + sc->surf_i[c][1] * v + sc->surf_i[c][2] * w;
      ab[nh][1 + c] = Is * (1.0 - Aphi);   /* Eq. BIrelation */
    }
    ++nh;
  }
  if (nh > 0) *flags |= ORC_HIT;
  return nh;
}

int orc_intersect(const orc_scene* sc, const orc_camera* cam, int64_t e, int i, int j, int max_seg,
                  double* seg, int* flags) {
  double o[3], r[3], amin, amax;
  orc_ray(cam, i, j, o, r);
  alpha_range(cam, &amin, &amax);
  *flags = 0;
  double rn = sqrt(dot3(r, r));
  double c[3], M[9];
  int nseg;
  int hitp, hitm;
  if (tree_affine(sc, sc->tree[e], c, M)) {
    double Mi[9], h = elem_h(sc, e), q0[3], dq[3], xi0[3], dxi[3];
    inv3(M, Mi);
    for (int k = 0; k < 3; ++k) {
      q0[k] = Mi[3 * k] * (o[0] - c[0]) + Mi[3 * k + 1] * (o[1] - c[1]) + Mi[3 * k + 2] * (o[2] - c[2]);
      dq[k] = Mi[3 * k] * r[0] + Mi[3 * k + 1] * r[1] + Mi[3 * k + 2] * r[2];
      xi0[k] = (q0[k] - ldexp((double)sc->anchor[3 * e + k], -MAXL)) / h;
      dxi[k] = dq[k] / h;
    }
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1}, lp[3], hp[3], lm[3], hm[3], a0, a1;
    for (int k = 0; k < 3; ++k) {
      double rowk = sqrt(Mi[3 * k] * Mi[3 * k] + Mi[3 * k + 1] * Mi[3 * k + 1] + Mi[3 * k + 2] * Mi[3 * k + 2]);
      double dk = EPS_AMBIG * rowk / h;
      lp[k] = -dk; hp[k] = 1 + dk; lm[k] = dk; hm[k] = 1 - dk;
    }
    nseg = slab(xi0, dxi, lo, hi, amin, amax, &a0, &a1);
    if (nseg && max_seg > 0) { seg[0] = a0; seg[1] = a1; }
    if (nseg && (a1 - a0) * rn < EPS_AMBIG) *flags |= ORC_AMBIGUOUS;
    hitp = slab(xi0, dxi, lp, hp, amin, amax, &a0, &a1);
    hitm = slab(xi0, dxi, lm, hm, amin, amax, &a0, &a1);
  } else {
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1}, lp[3], hp[3], lm[3], hm[3], tmp[16];
    for (int k = 0; k < 3; ++k) {
      double dk = EPS_AMBIG / min_edge(sc, e, k);
      lp[k] = -dk; hp[k] = 1 + dk; lm[k] = dk; hm[k] = 1 - dk;
    }
    int fl = 0;
    nseg = general_segments(sc, e, o, r, amin, amax, lo, hi, max_seg, seg, &fl);
    *flags |= fl;
    for (int q = 0; q < nseg && q < max_seg; ++q)
      if ((seg[2 * q + 1] - seg[2 * q]) * rn < EPS_AMBIG) *flags |= ORC_AMBIGUOUS;
    fl = 0;
    hitp = general_segments(sc, e, o, r, amin, amax, lp, hp, 8, tmp, &fl) > 0;
    *flags |= fl & (ORC_AMBIGUOUS | ORC_NEWTON_FAIL);
    fl = 0;
    hitm = general_segments(sc, e, o, r, amin, amax, lm, hm, 8, tmp, &fl) > 0;
    *flags |= fl & (ORC_AMBIGUOUS | ORC_NEWTON_FAIL);
  }
  if (hitp != hitm) *flags |= ORC_AMBIGUOUS;
  if (nseg > 0) *flags |= ORC_HIT;
  return nseg;
}

/* ======================================================================
 * Medium along a segment: kappa = kappa0 (f/F)^2,
 * q = q0 ((1+f~)/2, (1-f~)/2, 1/2); s measured from the near end.
 * ==================================================================== */
typedef struct {
  const orc_scene* sc; int64_t e; double o[3], r[3], alpha_near, rn;
} medium_ctx;

static long long g_medium_evals = 0;   /* field evaluations of orc_render (diagnostic) */
long long orc_medium_evals(int reset) {
  long long v = g_medium_evals;
  if (reset) g_medium_evals = 0;
  return v;
}

static void medium_eval(void* vctx, double s, double* kappa, double* q3) {
  medium_ctx* m = (medium_ctx*)vctx;
#pragma omp atomic
  g_medium_evals++;
  double al = m->alpha_near + s / m->rn;
  double p[3] = {m->o[0] + al * m->r[0], m->o[1] + al * m->r[1], m->o[2] + al * m->r[2]};
  double xi[3];
  orc_inverse_map(m->sc, m->e, p, xi);
  double ft = orc_field(m->sc, m->e, xi) * m->sc->inv_F;
  *kappa = m->sc->kappa0 * ft * ft;
  q3[0] = m->sc->q0 * 0.5 * (1.0 + ft);
  q3[1] = m->sc->q0 * 0.5 * (1.0 - ft);
  q3[2] = m->sc->q0 * 0.5;
}

/* ======================================================================
 * Per-pixel fold: sort by (alpha_near, elem), cut + average
 * overlaps, then the sequential
 * back-to-front composite I <- A_k I + B_k.
 * ==================================================================== */
static int cmp_hit(const void* x, const void* y) {
  const orc_hit* a = (const orc_hit*)x;
  const orc_hit* b = (const orc_hit*)y;
  if (a->alpha_near != b->alpha_near) return (a->alpha_near > b->alpha_near) - (a->alpha_near < b->alpha_near);
  return (a->elem > b->elem) - (a->elem < b->elem);
}

/* The piece of segment s on [x, y] (an <= x < y <= af): Eq. segsplit
 * applied twice -- cut at x and keep the far part, cut
 * that at y and keep the near part. */
static orc_hit sub_hit(const orc_hit* s, double x, double y) {
  orc_hit p = *s;
  double out[4];
  if (x > s->alpha_near) {          /* far part of the cut at x */
    orc_split(p.a, 0.0, x - p.alpha_near, p.alpha_far - x, out);
    double a_far = out[2];
    for (int c = 0; c < 3; ++c) {
      orc_split(p.a, p.b[c], x - p.alpha_near, p.alpha_far - x, out);
      p.b[c] = out[3];
    }
    p.a = a_far;
    p.alpha_near = x;
  }
  if (y < p.alpha_far) {            /* near part of the cut at y */
    orc_split(p.a, 0.0, y - p.alpha_near, p.alpha_far - y, out);
    double a_near = out[0];
    for (int c = 0; c < 3; ++c) {
      orc_split(p.a, p.b[c], y - p.alpha_near, p.alpha_far - y, out);
      p.b[c] = out[1];
    }
    p.a = a_near;
    p.alpha_far = y;
  }
  return p;
}

static int cmp_double(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* Per-pixel fold (PAPER.md:295-301 back to front, Eq. aggregate
 * PAPER.md:386-394) with the overlap resolution of PAPER.md:495-558 ("cutting
 * the segments into pieces to isolate the overlapping section and then
 * averaging the segment values in the overlapping interval"), read for any
 * number of mutually overlapping segments as DESIGN.md D14:
 *  - sort by (alpha_near, elem);
 *  - a cluster is a maximal run of the sorted list in which every segment
 *    starts more than tol = tau max(1,|alpha|) before the largest alpha_far of
 *    the segments before it in the run (overlap beyond the tolerance, R15);
 *  - every member of a cluster is cut (Eq. segsplit) at all end points of the
 *    cluster; on each elementary interval between consecutive end points the
 *    pieces covering it are averaged, geometric mean of A and arithmetic mean
 *    of B (Eq. segaverage; for m pieces: (prod A)^(1/m), sum B / m);
 *  - an elementary interval covered by no piece is an empty gap (identity,
 *    PAPER.md:427). */
void orc_fold_pixel(int n, orc_hit* segs, double tau, const double background[3], double rgba[4],
                    double ab[4]) {
  qsort(segs, n, sizeof(orc_hit), cmp_hit);
  orc_hit* out = (orc_hit*)malloc(sizeof(orc_hit) * (4 * n + 4));
  double* pts = (double*)malloc(sizeof(double) * (2 * n + 2));
  int m = 0;
  int k = 0;
  while (k < n) {
    int j = k + 1;
    double far = segs[k].alpha_far;
    while (j < n && segs[j].alpha_near < far - tau * fmax(1.0, fabs(segs[j].alpha_near))) {
      if (segs[j].alpha_far > far) far = segs[j].alpha_far;
      ++j;
    }
    if (j == k + 1) {                 /* no overlap: the segment as it is */
      out[m++] = segs[k];
      k = j;
      continue;
    }
    int np = 0;
    for (int t = k; t < j; ++t) {
      pts[np++] = segs[t].alpha_near;
      pts[np++] = segs[t].alpha_far;
    }
    qsort(pts, np, sizeof(double), cmp_double);
    for (int q = 0; q + 1 < np; ++q) {
      double x = pts[q], y = pts[q + 1];
      if (!(y > x)) continue;
      int cnt = 0;
      double prodA = 1.0, sumB[3] = {0.0, 0.0, 0.0};
      orc_hit first;
      for (int t = k; t < j; ++t) {
        if (segs[t].alpha_near <= x && y <= segs[t].alpha_far) {
          orc_hit p = sub_hit(&segs[t], x, y);
          if (cnt == 0) first = p;
          prodA *= p.a;
          for (int c = 0; c < 3; ++c) sumB[c] += p.b[c];
          ++cnt;
        }
      }
      if (cnt == 0) continue;         /* empty gap inside the cluster */
      orc_hit av = first;
      av.alpha_near = x;
      av.alpha_far = y;
      if (cnt > 1) {
        av.a = (cnt == 2) ? sqrt(prodA) : pow(prodA, 1.0 / cnt);
        for (int c = 0; c < 3; ++c) av.b[c] = sumB[c] / cnt;
      }
      out[m++] = av;
    }
    k = j;
  }
  /* back to front */
  double I[3] = {background[0], background[1], background[2]}, B[3] = {0, 0, 0}, T = 1.0;
  for (int q = m - 1; q >= 0; --q) {
    for (int c = 0; c < 3; ++c) {
      I[c] = out[q].a * I[c] + out[q].b[c];
      B[c] = out[q].a * B[c] + out[q].b[c];
    }
    T = out[q].a * T;
  }
  rgba[0] = I[0]; rgba[1] = I[1]; rgba[2] = I[2]; rgba[3] = 1.0 - T;
  if (ab) { ab[0] = T; ab[1] = B[0]; ab[2] = B[1]; ab[3] = B[2]; }
  free(out);
  free(pts);
}

/* ======================================================================
 * Render a subset of pixels: brute force over every leaf whose EPS-inflated
 * rect contains the pixel (SURVEY §8(c) oracle steps 1-7).
 * ==================================================================== */
static int64_t render_core(const orc_scene* sc, const orc_camera* cam, int mode, int N, const double background[3],
                           int64_t npix, const int32_t* pixels, double* rgba, int32_t* nhits, int32_t* namb,
                           int32_t cap, orc_hit* hits, int nthreads, int8_t* vis_out, int8_t* amb_out,
                           orc_pairs* pairs, const int32_t* rects_in) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  int W = cam->width, H = cam->height;
  int64_t npx = (int64_t)W * H;
  int8_t* vis = (int8_t*)malloc(sc->n);
  int8_t* amb = (int8_t*)malloc(sc->n);
  int32_t* rects = (int32_t*)malloc(sizeof(int32_t) * 4 * sc->n);
  if (rects_in) {   /* the culled rectangles of an earlier orc_cull of the same scene and camera */
    memcpy(rects, rects_in, sizeof(int32_t) * 4 * sc->n);
  } else {
    orc_cull(sc, cam, vis, amb, rects);
    if (vis_out) memcpy(vis_out, vis, sc->n);
    if (amb_out) memcpy(amb_out, amb, sc->n);
  }
  /* per-pixel (elem, flags) lists of every candidate with HIT or AMBIGUOUS */
  int64_t** pe = NULL;
  int32_t** pf = NULL;
  int32_t* pn = NULL;
  if (pairs) {
    pe = (int64_t**)calloc(npix, sizeof(int64_t*));
    pf = (int32_t**)calloc(npix, sizeof(int32_t*));
    pn = (int32_t*)calloc(npix, sizeof(int32_t));
  }
  int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * npx);
  for (int64_t p = 0; p < npx; ++p) slot[p] = -1;
  for (int64_t q = 0; q < npix; ++q) slot[pixels[q]] = q;
  int64_t* cnt = (int64_t*)calloc(npix + 1, sizeof(int64_t));
  for (int64_t e = 0; e < sc->n; ++e) {
    int32_t* rc = rects + 4 * e;
    for (int jj = rc[2]; jj <= rc[3]; ++jj)
      for (int ii = rc[0]; ii <= rc[1]; ++ii) {
        int64_t s = slot[(int64_t)jj * W + ii];
        if (s >= 0) cnt[s + 1]++;
      }
  }
  for (int64_t q = 0; q < npix; ++q) cnt[q + 1] += cnt[q];
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (cnt[npix] + 1));
  int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * (npix + 1));
  memcpy(fillp, cnt, sizeof(int64_t) * (npix + 1));
  for (int64_t e = 0; e < sc->n; ++e) {   /* SFC order within each pixel list */
    int32_t* rc = rects + 4 * e;
    for (int jj = rc[2]; jj <= rc[3]; ++jj)
      for (int ii = rc[0]; ii <= rc[1]; ++ii) {
        int64_t s = slot[(int64_t)jj * W + ii];
        if (s >= 0) cand[fillp[s]++] = e;
      }
  }
  int64_t total_hits = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : total_hits)
  for (int64_t q = 0; q < npix; ++q) {
    int pix = pixels[q], i = pix % W, j = pix / W;
    int64_t nc = cnt[q + 1] - cnt[q];
    orc_hit* list = (orc_hit*)malloc(sizeof(orc_hit) * (8 * nc + 1));
    orc_hit* fold = (orc_hit*)malloc(sizeof(orc_hit) * (8 * nc + 1));
    int nl = 0, nf = 0, na = 0, nh = 0;
    double o[3], r[3];
    orc_ray(cam, i, j, o, r);
    double rn = sqrt(dot3(r, r));
    for (int64_t t = cnt[q]; t < cnt[q + 1]; ++t) {
      int64_t e = cand[t];
      double seg[16];
      int flags = 0;
      double sal[2], sab[2][4];
      int ns = is_surface(sc) ? surface_hits(sc, cam, e, i, j, sal, sab, &flags)
                              : orc_intersect(sc, cam, e, i, j, 8, seg, &flags);
      if (flags & ORC_AMBIGUOUS) na++;
      if (ns > 0) nh++;
      if (pairs && (ns > 0 || (flags & ORC_AMBIGUOUS))) {
        if (!pe[q]) {
          pe[q] = (int64_t*)malloc(sizeof(int64_t) * (nc + 1));
          pf[q] = (int32_t*)malloc(sizeof(int32_t) * (nc + 1));
        }
        pe[q][pn[q]] = e;
        pf[q][pn[q]] = flags | (ns > 0 ? ORC_HIT : 0);
        pn[q]++;
      }
      if (mode == 2) continue;   /* hit lists only: no integration */
      if (ns == 0 && (flags & ORC_AMBIGUOUS)) {
        orc_hit hh;
        memset(&hh, 0, sizeof hh);
        hh.elem = e; hh.pixel = pix; hh.flags = flags; hh.a = 1.0;
        list[nl++] = hh;
      }
      for (int s = 0; s < ns; ++s) {
        orc_hit hh;
        memset(&hh, 0, sizeof hh);
        hh.elem = e; hh.pixel = pix; hh.flags = flags;
        if (is_surface(sc)) {   /* a zero-length segment (Eq. ABphi) */
          hh.alpha_near = hh.alpha_far = sal[s];
          hh.a = sab[s][0];
          for (int c = 0; c < 3; ++c) hh.b[c] = sab[s][1 + c];
          list[nl++] = hh;
          fold[nf++] = hh;
          continue;
        }
        hh.alpha_near = seg[2 * s]; hh.alpha_far = seg[2 * s + 1];
        medium_ctx mc;
        mc.sc = sc; mc.e = e; memcpy(mc.o, o, sizeof o); memcpy(mc.r, r, sizeof r);
        mc.alpha_near = hh.alpha_near; mc.rn = rn;
        double L = (hh.alpha_far - hh.alpha_near) * rn;   /* s = alpha |r| */
        if (mode == 0) {
          if (orc_segment_exact(medium_eval, &mc, L, &hh.a, hh.b) < 0) hh.flags |= ORC_NEWTON_FAIL;
        } else if (mode == 3) {   /* the paper's integrators, Alg. 1 (orc_set_scheme) */
          int sf = 0;
          orc_segment_scheme(g_scheme, N, g_scheme_crk, g_scheme_depth, medium_eval, &mc, L, &hh.a, hh.b, &sf);
          if (sf & 1) hh.flags |= ORC_NEWTON_FAIL;
          if (sf & 2) hh.flags |= ORC_SPLIT_NEAR;
        } else {
          orc_segment_rule(N, medium_eval, &mc, L, &hh.a, hh.b);
        }
        list[nl++] = hh;
        fold[nf++] = hh;
        /* integration flags (Alg. 1 decisions near c_RK, depth cap) onto the pair's entry */
        if (pairs && (hh.flags & (ORC_SPLIT_NEAR | ORC_NEWTON_FAIL))) pf[q][pn[q] - 1] |= hh.flags & (ORC_SPLIT_NEAR | ORC_NEWTON_FAIL);
      }
    }
    if (mode == 2) { for (int c = 0; c < 4; ++c) rgba[4 * q + c] = 0.0; }
    else orc_fold_pixel(nf, fold, TAU_OV, background, rgba + 4 * q, NULL);
    nhits[q] = nh;
    namb[q] = na;
    if (hits) {
      qsort(list, nl, sizeof(orc_hit), cmp_hit);
      int nn = nl < cap ? nl : cap;
      memcpy(hits + q * cap, list, sizeof(orc_hit) * nn);
      for (int t = nn; t < cap; ++t) { memset(hits + q * cap + t, 0, sizeof(orc_hit)); hits[q * cap + t].elem = -1; }
      if (nl > cap) hits[q * cap + cap - 1].flags |= ORC_OVERFLOW;
    }
    total_hits += nh;
    free(list);
    free(fold);
  }
  free(vis); free(amb); free(rects); free(slot); free(cnt); free(cand); free(fillp);
  if (pairs) {
    pairs->npix = npix;
    pairs->off = (int64_t*)malloc(sizeof(int64_t) * (npix + 1));
    pairs->off[0] = 0;
    for (int64_t q = 0; q < npix; ++q) pairs->off[q + 1] = pairs->off[q] + pn[q];
    int64_t tot = pairs->off[npix];
    pairs->elem = (int64_t*)malloc(sizeof(int64_t) * (tot + 1));
    pairs->flags = (int32_t*)malloc(sizeof(int32_t) * (tot + 1));
    for (int64_t q = 0; q < npix; ++q) {
      if (pn[q]) {
        memcpy(pairs->elem + pairs->off[q], pe[q], sizeof(int64_t) * pn[q]);
        memcpy(pairs->flags + pairs->off[q], pf[q], sizeof(int32_t) * pn[q]);
      }
      free(pe[q]);
      free(pf[q]);
    }
    free(pe); free(pf); free(pn);
  }
  return total_hits;
}

int64_t orc_render(const orc_scene* sc, const orc_camera* cam, int mode, int N, const double background[3],
                   int64_t npix, const int32_t* pixels, double* rgba, int32_t* nhits, int32_t* namb,
                   int32_t cap, orc_hit* hits, int nthreads) {
  return render_core(sc, cam, mode, N, background, npix, pixels, rgba, nhits, namb, cap, hits, nthreads, NULL,
                     NULL, NULL, NULL);
}

int64_t orc_render_ex(const orc_scene* sc, const orc_camera* cam, int mode, int N, const double background[3],
                      int64_t npix, const int32_t* pixels, double* rgba, int32_t* nhits, int32_t* namb,
                      int nthreads, int8_t* visible, int8_t* ambiguous, orc_pairs* pairs,
                      const int32_t* rects_in) {
  return render_core(sc, cam, mode, N, background, npix, pixels, rgba, nhits, namb, 0, NULL, nthreads, visible,
                     ambiguous, pairs, rects_in);
}

void orc_pairs_free(orc_pairs* p) {
  if (!p) return;
  free(p->off); free(p->elem); free(p->flags);
  p->off = NULL; p->elem = NULL; p->flags = NULL;
}
