"""Pins of the fp64 oracle against what the paper and mathematics fix
(SURVEY.md §8(c) P1-P15).  CPU only.  Nothing here compares the oracle with
itself: each check uses a closed form, a worked value from the paper, a
library routine (numpy / scipy), an independent textbook algorithm written in
this file (3D-DDA, slab test), or brute force."""
import math
import os

import numpy as np
import pytest

import oracle
import scenegen as sg

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------------------
# Segment algebra: worked values (tests/golden/segment_algebra.txt) + theorems
# ---------------------------------------------------------------------------
def _golden_cases():
    out = []
    for line in open(os.path.join(GOLDEN, "segment_algebra.txt")):
        line = line.split("|")[0].strip()
        if not line or line.startswith("#"):
            continue
        lhs, rhs = line.split("->")
        toks = lhs.split()
        out.append((toks[0], [float(t) for t in toks[1:]], [float(t) for t in rhs.split()]))
    return out


@pytest.mark.parametrize("op,args,expect", _golden_cases())
def test_algebra_golden(op, args, expect):
    if op == "combine":
        got = oracle.combine(args[0:2], args[2:4])
    elif op == "inverse":
        got = oracle.inverse(args[0:2])
    elif op == "split":
        (a1, b1), (a2, b2) = oracle.split(args[0:2], args[2], args[3])
        got = (a1, b1, a2, b2)
    elif op == "average":
        got = oracle.average(args[0:2], args[2:4])
    elif op == "constant":
        got = oracle.from_constant(*args)
    elif op == "background":
        got = (oracle.background(args[0:2], args[2]),)
    np.testing.assert_allclose(got, expect, rtol=1e-14, atol=1e-15)


def test_group_laws_random():
    """associativity, identity (1,0), inverse (1/A,-B/A)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        s = [(rng.uniform(0.05, 1), rng.normal()) for _ in range(3)]
        left = oracle.combine(oracle.combine(s[0], s[1]), s[2])
        right = oracle.combine(s[0], oracle.combine(s[1], s[2]))
        np.testing.assert_allclose(left, right, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(oracle.combine((1.0, 0.0), s[0]), s[0], rtol=0, atol=0)
        np.testing.assert_allclose(oracle.combine(s[0], oracle.inverse(s[0])), (1.0, 0.0), atol=1e-12)
        np.testing.assert_allclose(oracle.combine(oracle.inverse(s[0]), s[0]), (1.0, 0.0), atol=1e-12)
    with pytest.raises(ValueError):
        oracle.inverse((0.0, 1.0))


def test_composition_of_constant_media():
    """Eq. aggregate composes two exact constant-medium solutions end to end:
    near (beta2,gamma2,dx2) (+) far (beta1,gamma1,dx1) equals the solution of
    Eq. Iode over the concatenated interval (closed form written out here)."""
    b1, g1, d1, b2, g2, d2 = 0.7, 0.3, 0.4, 1.9, 0.8, 0.25
    far = oracle.from_constant(b1, g1, d1)
    near = oracle.from_constant(b2, g2, d2)
    A, B = oracle.combine(near, far)
    I_mid = lambda I0: math.exp(-b1 * d1) * I0 + g1 / b1 * (1 - math.exp(-b1 * d1))
    I_end = lambda I0: math.exp(-b2 * d2) * I_mid(I0) + g2 / b2 * (1 - math.exp(-b2 * d2))
    assert abs(A - (I_end(1.0) - I_end(0.0))) < 1e-15
    assert abs(B - I_end(0.0)) < 1e-15


def test_split_round_trip_and_constant_consistency():
    """Eq. segsplit: pieces aggregate back to the segment; for constant media
    the pieces equal Eq. ABconstant over the piece lengths."""
    rng = np.random.default_rng(2)
    for _ in range(100):
        beta, gamma, dx = rng.uniform(0.1, 3), rng.uniform(-1, 2), rng.uniform(0.1, 2)
        f = rng.uniform(0.05, 0.95)
        s = oracle.from_constant(beta, gamma, dx)
        p1, p2 = oracle.split(s, f * dx, (1 - f) * dx)
        np.testing.assert_allclose(p1, oracle.from_constant(beta, gamma, f * dx), rtol=1e-12)
        np.testing.assert_allclose(p2, oracle.from_constant(beta, gamma, (1 - f) * dx), rtol=1e-12)
        np.testing.assert_allclose(oracle.combine(p1, p2), s, rtol=1e-12)
        np.testing.assert_allclose(oracle.combine(p2, p1), s, rtol=1e-12)
    with pytest.raises(ValueError):
        oracle.split((0.5, 0.1), -1.0, 2.0)


def test_average_is_interleaving_limit():
    """Eq. segaverage vs the construction in its proof:
    alternating 1/(2N)-pieces of the two segments.  The limit reproduces the
    geometric mean for A exactly; for B the proof linearises 1-A^q ~ q(1-A),
    so (B1+B2)/2 is reached only to first order in (1-A) (DESIGN.md reading
    D7).  Pin A in general and B in the regime the proof assumes."""
    def interleave(s1, s2, N=1 << 12):
        p1 = oracle.split(s1, 1.0 / (2 * N), 1.0 - 1.0 / (2 * N))[0]
        p2 = oracle.split(s2, 1.0 / (2 * N), 1.0 - 1.0 / (2 * N))[0]
        pair = oracle.combine(p2, p1)
        acc = (1.0, 0.0)
        for _ in range(N):
            acc = oracle.combine(acc, pair)
        return acc
    acc = interleave((0.25, 0.1), (1.0, 0.3))
    assert abs(acc[0] - oracle.average((0.25, 0.1), (1.0, 0.3))[0]) < 1e-12
    s1, s2 = (0.9995, 0.0012), (0.9990, 0.0031)
    acc = interleave(s1, s2)
    np.testing.assert_allclose(acc, oracle.average(s1, s2), rtol=1e-3)


def test_reversal_theorem():
    """constant negative coefficients give the inverse segment."""
    for beta, gamma, dx in [(0.7, 0.3, 1.1), (2.0, -1.0, 0.3), (0.0, 2.0, 0.5)]:
        inv = oracle.inverse(oracle.from_constant(beta, gamma, dx))
        np.testing.assert_allclose(oracle.from_constant(-beta, -gamma, dx), inv, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------------------
# Quadrature tables against numpy
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("N", list(range(1, 17)))
def test_gauss_legendre_vs_numpy(N):
    u, w = oracle.gauss_legendre(N)
    x, wx = np.polynomial.legendre.leggauss(N)
    np.testing.assert_allclose(u, (x + 1) / 2, atol=1e-15)
    np.testing.assert_allclose(w, wx / 2, atol=1e-15)


@pytest.mark.filterwarnings("ignore::scipy.integrate.IntegrationWarning")
@pytest.mark.parametrize("N", [1, 2, 4, 6, 8, 16])
def test_lagrange_integral_table_vs_scipy(N):
    """S_jk = int_0^{u_j} l_k(u) du by scipy adaptive quadrature of the product form."""
    from scipy.integrate import quad
    u, _ = oracle.gauss_legendre(N)
    S = oracle.lagrange_integrals(N, u)
    for k in range(N):
        lk = lambda t, k=k: np.prod([(t - u[m]) / (u[k] - u[m]) for m in range(N) if m != k])
        for j in range(N):
            ref = quad(lk, 0.0, u[j], epsabs=1e-15, epsrel=1e-14, limit=200)[0]
            assert abs(S[j, k] - ref) < 1e-13


# ---------------------------------------------------------------------------
# Exact-mode segment integration (Eq. ABgeneral)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("kappa,q,L", [(2.0, 1.0, 0.3), (0.05, 0.7, 2.0), (5.0, 0.2, 1.7), (1e-3, 1.0, 0.01)])
def test_exact_constant_medium_P1(kappa, q, L):
    a, b, M = oracle.segment_exact(lambda s: (kappa, q), L)
    ae = math.exp(-kappa * L)
    be = -q * math.expm1(-kappa * L) / kappa     # cancellation-free form of q(1-a)/kappa
    assert M > 0
    assert abs(a - ae) <= 1e-14 * ae
    np.testing.assert_allclose(b, be, rtol=1e-13)


def test_exact_transparent_medium_P2():
    a, b, _ = oracle.segment_exact(lambda s: (0.0, 2.0), 0.5)
    assert a == 1.0
    np.testing.assert_allclose(b, 1.0, rtol=1e-14)


def test_exact_vs_scipy_nested_quadrature():
    """B = int_0^L gamma(s) exp(-int_0^s beta) with beta = 1+3s^2 (inner integral
    s + s^3 in closed form), gamma = 2 - s + sin 3s, by scipy.integrate.quad."""
    from scipy.integrate import quad
    L = 0.9
    kap = lambda s: 1 + 3 * s * s
    gam = lambda s: 2 - s + math.sin(3 * s)
    a, b, M = oracle.segment_exact(lambda s: (kap(s), gam(s)), L)
    bref, _ = quad(lambda s: gam(s) * math.exp(-(s + s ** 3)), 0, L, epsabs=1e-15, epsrel=1e-14, limit=200)
    assert abs(a - math.exp(-(L + L ** 3))) < 1e-15
    np.testing.assert_allclose(b, bref, rtol=1e-12)


def test_exact_vs_scipy_ode_orientation():
    """Solve Eq. Iode I' = gamma - beta I upstream (x=0, far) to downstream
    (x=L, near) with scipy; s = L - x is the oracle's near-end coordinate."""
    from scipy.integrate import solve_ivp
    L = 1.3
    beta_s = lambda s: 0.5 + 2 * math.sin(2 * s) ** 2
    gam_s = lambda s: 1.0 + 0.8 * s
    a, b, _ = oracle.segment_exact(lambda s: (beta_s(s), gam_s(s)), L)
    f = lambda x, I: [gam_s(L - x) - beta_s(L - x) * I[0]]
    B = solve_ivp(f, (0, L), [0.0], rtol=1e-13, atol=1e-14, method="DOP853").y[0, -1]
    A = solve_ivp(lambda x, I: [-beta_s(L - x) * I[0]], (0, L), [1.0], rtol=1e-13, atol=1e-14,
                  method="DOP853").y[0, -1]
    np.testing.assert_allclose(a, A, rtol=1e-11)
    np.testing.assert_allclose(b, B, rtol=1e-11)


def test_exact_vs_paper_gauss2_composite_P13():
    """Eq. gaussAB/gaussABab with x1 = upstream end, composed
    over M panels with Eq. aggregate, converges to exact mode at order 4.
    A wrong orientation of exact mode (attenuating towards the far end) would
    not be the limit of this composite."""
    L = 0.8
    kap = lambda s: 1 + 3 * s * s
    gam = lambda s: 2 - s + math.sin(3 * s)
    a_ex, b_ex, _ = oracle.segment_exact(lambda s: (kap(s), gam(s)), L)

    def gauss2(x1, dx):
        beta = lambda x: kap(L - x)
        gamma = lambda x: gam(L - x)
        xi0, xi1 = x1 + (0.5 - math.sqrt(3) / 6) * dx, x1 + (0.5 + math.sqrt(3) / 6) * dx   # DESIGN D6
        a1 = dx * (beta(xi0) + beta(xi1)) / 4
        a2 = dx * dx * beta(xi0) * beta(xi1) / 12
        b1 = dx * (gamma(xi0) + gamma(xi1)) / 2
        b2 = dx * dx * (beta(xi0) * gamma(xi1) - beta(xi1) * gamma(xi0)) * math.sqrt(3) / 12
        return (1 - a1 + a2) / (1 + a1 + a2), (b1 + b2) / (1 + a1 + a2)

    errs = []
    for M in (8, 16, 32, 64):
        acc = (1.0, 0.0)
        dx = L / M
        for m in range(M):   # far panel first, then nearer ones on the left
            acc = oracle.combine(gauss2(m * dx, dx), acc)
        errs.append((abs(acc[0] - a_ex), abs(acc[1] - b_ex[0])))
    assert errs[-1][0] < 1e-8 and errs[-1][1] < 1e-8
    for (e0, f0), (e1, f1) in zip(errs, errs[1:]):
        assert e1 < e0 / 12 and f1 < f0 / 12    # fourth order: consistent orientation


def test_exact_self_convergence_P12():
    L = 1.1
    fn = lambda s: (2 + math.cos(7 * s), (1 + math.sin(5 * s), 0.5, 0.2 * s))
    a, b, M = oracle.segment_exact(fn, L)
    a2, b2 = oracle.segment_rule(16, fn, L)   # fp64 rule with many nodes, independent discretisation
    assert M > 0
    assert abs(a - a2) < 1e-12
    np.testing.assert_allclose(b, b2, atol=1e-11)


def test_rule_transmission_exact_for_polynomial_kappa():
    """a = exp(-L sum w kappa) is exact for deg(kappa) <= 2N-1."""
    L = 0.7
    for N in (2, 3, 4):
        c = np.arange(1, 2 * N + 1) * 0.1
        kap = lambda s: float(np.polynomial.polynomial.polyval(s, c))
        a, _ = oracle.segment_rule(N, lambda s: (kap(s), 0.0), L)
        integ = np.polynomial.polynomial.polyval(L, np.polynomial.polynomial.polyint(c))
        assert abs(a - math.exp(-integ)) < 1e-14


# ---------------------------------------------------------------------------
# Geometry and camera
# ---------------------------------------------------------------------------
def test_gll_nodes_nodality_unity():
    assert list(oracle.gll(1)) == [0.0, 1.0]          # PAPER.md:152 eta_0 = 0, eta_N = 1
    assert list(oracle.gll(2)) == [0.0, 0.5, 1.0]     # GLL(3): roots of P'_2 on [0,1] -> 1/2
    x = np.polynomial.legendre.Legendre.basis(2).deriv().roots()
    assert abs((x[0] + 1) / 2 - 0.5) < 1e-15
    for R in (1, 2):
        eta = oracle.gll(R)
        for m in range(R + 1):
            psi, _ = oracle.lagrange(R, eta, eta[m])
            np.testing.assert_allclose(psi, np.eye(R + 1)[m], atol=1e-15)   # Eq. nodal
        for t in np.linspace(-0.3, 1.3, 11):
            psi, dpsi = oracle.lagrange(R, eta, t)
            assert abs(psi.sum() - 1) < 1e-14 and abs(dpsi.sum()) < 1e-13    # Eq. tensorunity


def _affine_scene(R, M, c, level=2):
    anchor, tree, lev = sg.uniform_leaves(1, level)
    cam = sg.perspective_camera([3.0, 2.0, 1.5], [0.5, 0.5, 0.5], 40.0, 32, 32)
    fld = np.zeros((anchor.shape[0], 8), dtype=np.float32)
    return sg.Scene("affine", R, 1, sg.affine_ctrl(R, M, c), anchor, tree, lev, fld, 5.0, 1.0, 1.0, cam)


def test_tree_map_affine_invariance():
    """Eq. tensorunity => an affine control grid reproduces the affine map."""
    rng = np.random.default_rng(3)
    for R in (1, 2):
        M = rng.normal(size=(3, 3)); c = rng.normal(size=3)
        o = oracle.OracleScene(_affine_scene(R, M, c))
        for _ in range(50):
            t = rng.uniform(-0.2, 1.2, size=3)
            np.testing.assert_allclose(o.tree_map(0, t), M @ t + c, atol=1e-12)


def test_camera_transform_and_camerapoints():
    """Eq. camerageometry examples and Eq. camerapoints:
    Phi o J = J built from Phi(z)."""
    sc = sg.config2(width=64, maxlevel=4)
    o = oracle.OracleScene(sc)
    cam = sc.camera
    np.testing.assert_allclose(o.camera_transform(cam.origin), 0, atol=1e-15)
    np.testing.assert_allclose(o.camera_transform(cam.origin + cam.view), [0, 0, 1.0], atol=1e-14)
    sh = sg.shell_uniform(1, 32, 4)
    osh = oracle.OracleScene(sh)
    zc = np.array([osh.camera_transform(p) for p in sh.tree_ctrl.reshape(-1, 3)]).reshape(sh.tree_ctrl.shape)
    import dataclasses
    osc = oracle.OracleScene(dataclasses.replace(sh, tree_ctrl=zc))
    rng = np.random.default_rng(4)
    for _ in range(30):
        t = rng.uniform(size=3); k = int(rng.integers(6))
        np.testing.assert_allclose(osc.tree_map(k, t), osh.camera_transform(osh.tree_map(k, t)), atol=1e-13)


def test_ray_direction_examples():
    """Eq. ray."""
    cam = sg.perspective_camera([0, 0, 0], [1.0, 0, 0], 40.0, 5, 5)
    cam.pixel_size = 0.1
    o = oracle.OracleScene(sg.Scene("x", 1, 1, sg.identity_cube_ctrl(), np.zeros((1, 3), np.int32),
                                    np.zeros(1, np.int32), np.zeros(1, np.int8), np.zeros((1, 8), np.float32),
                                    5, 1, 1, cam))
    _, r = o.ray(2, 2)
    np.testing.assert_allclose(r, cam.view, atol=1e-15)
    _, r1 = o.ray(3, 2)
    np.testing.assert_allclose(r1 - r, 0.1 * cam.right, atol=1e-15)
    cam2 = sg.perspective_camera([0, 0, 0], [1.0, 0, 0], 40.0, 2, 2)
    cam2.pixel_size = 0.1
    o2 = oracle.OracleScene(sg.Scene("x", 1, 1, sg.identity_cube_ctrl(), np.zeros((1, 3), np.int32),
                                     np.zeros(1, np.int32), np.zeros(1, np.int8), np.zeros((1, 8), np.float32),
                                     5, 1, 1, cam2))
    _, r = o2.ray(1, 1)
    np.testing.assert_allclose(r, cam2.view + 0.05 * cam2.right + 0.05 * cam2.up, atol=1e-15)


def test_shell_aabb_contains_samples():
    """Convex-hull property of the Bernstein points:
    the camera-space AABB contains every sampled point of the element."""
    sh = sg.shell_uniform(1, 64, 4)
    o = oracle.OracleScene(sh)
    rng = np.random.default_rng(5)
    for e in range(0, sh.num_leaves, 5):
        lo, hi = o.aabb(e)
        for _ in range(60):
            X = o.camera_transform(o.element_map(e, rng.uniform(size=3))[0])
            assert np.all(X >= lo - 1e-13) and np.all(X <= hi + 1e-13)


def test_shell_aabb_is_the_bernstein_box():
    """AABB tightness: the culling box is exactly the camera-space
    min/max of the element's 27 Bernstein-Bezier points, which this test forms
    itself from the Lagrange points X_E({0,1/2,1}^3) by the per-axis
    conversion b_mid = 2 x_mid - (x_0 + x_2)/2 (degree-2 Bernstein basis,
    textbook identity).  A looser (or tighter) box fails."""
    sh = sg.shell_uniform(1, 64, 4)
    o = oracle.OracleScene(sh)
    eta = (0.0, 0.5, 1.0)
    for e in range(0, sh.num_leaves, 3):
        L = np.array([[[o.element_map(e, [eta[m1], eta[m2], eta[m3]])[0] for m1 in range(3)] for m2 in range(3)]
                      for m3 in range(3)])            # [m3][m2][m1][xyz]
        B = L.copy()
        for ax in (2, 1, 0):                          # numpy axis of m1, m2, m3
            Bm = np.moveaxis(B, ax, 0)
            Bm[1] = 2.0 * Bm[1] - 0.5 * (Bm[0] + Bm[2])
        X = np.array([o.camera_transform(p) for p in B.reshape(-1, 3)])
        lo, hi = o.aabb(e)
        assert np.allclose(lo, X.min(axis=0), rtol=0, atol=1e-12) and np.allclose(hi, X.max(axis=0), rtol=0,
                                                                                  atol=1e-12), e


def test_constant_shell_exact_sphere_chord_P14():
    """P14: f == const on the
    cubed-sphere shell: every pixel is Eq. ABconstant over the ray's chord
    through the exact spherical shell 0.55 <= |x| <= 1, up to the R=2
    geometry's deviation from the sphere (~0.8 % of the radius).
    Rays within 0.1 of tangency to either sphere are left out (the chord is
    ill-conditioned there)."""
    sc = sg.constant_field(sg.shell_uniform(2, 48, 4, gl_points=6), 0.6)
    o = oracle.OracleScene(sc)
    res = o.render(mode="exact", with_hits=False)
    ft = float(np.float32(0.6))
    kap = 5.0 * ft * ft
    q = np.array([(1 + ft) / 2, (1 - ft) / 2, 0.5])
    W = sc.camera.width
    errs = []
    for k, p in enumerate(res["pixels"]):
        ro, rd = o.ray(int(p) % W, int(p) // W)
        d = rd / np.linalg.norm(rd)
        dist = np.linalg.norm(np.cross(ro, d))        # distance of the line from the centre
        if dist > 0.9 or abs(dist - 0.55) < 0.1:
            continue
        L = 2.0 * math.sqrt(1.0 - dist * dist) - (2.0 * math.sqrt(0.55 ** 2 - dist * dist) if dist < 0.55 else 0.0)
        A = math.exp(-kap * L)
        ref = np.r_[q * (1 - A) / kap, 1 - A]
        errs.append(float(np.abs(res["rgba"][k] - ref).max()))
    errs = np.array(errs)
    assert errs.size > 500
    assert errs.max() < 0.03 and errs.mean() < 0.01, (errs.max(), errs.mean())


def test_pixel_rect_similar_triangles():
    """Centered box at depth z, axis-aligned camera: rect width from
    similar triangles p = (n/l) X/Z + (w-1)/2."""
    cam = sg.perspective_camera([0, 0, 0], [0, 0, 1.0], 40.0, 101, 101)
    # view along +z: the frame falls back to +y as the up reference (no NaN)
    assert np.all(np.isfinite(np.r_[cam.view, cam.right, cam.up]))
    assert abs(np.dot(cam.right, cam.up)) < 1e-15 and abs(np.linalg.norm(cam.up) - 1) < 1e-15
    o = oracle.OracleScene(sg.Scene("x", 1, 1, sg.identity_cube_ctrl(), np.zeros((1, 3), np.int32),
                                    np.zeros(1, np.int32), np.zeros(1, np.int8), np.zeros((1, 8), np.float32),
                                    5, 1, 1, cam))
    half = 0.1
    ok, rc = o.pixel_rect([-half, -half, 2.0], [half, half, 2.2])
    p = (1.0 / cam.pixel_size) * half / 2.0
    assert ok and rc[0] == math.ceil(50 - p) and rc[1] == math.floor(50 + p)
    ok, _ = o.pixel_rect([-1, -1, -3], [1, 1, -2])     # behind the camera
    assert not ok


def test_inverse_map_and_field():
    sh = sg.shell_uniform(1, 32, 4)
    o = oracle.OracleScene(sh)
    rng = np.random.default_rng(6)
    for e in (0, 7, 20, 40):
        for _ in range(10):
            xi = rng.uniform(size=3)
            st, xi2 = o.inverse_map(e, o.element_map(e, xi)[0])
            assert st == 0 and np.allclose(xi, xi2, atol=1e-13)
        # nodal interpolation reproduces nodal values (Eq. nodal for the field)
        f = sh.leaf_field[e].reshape(3, 3, 3)
        for k3 in range(3):
            for k2 in range(3):
                for k1 in range(3):
                    assert o.field_at(e, [k1 / 2, k2 / 2, k3 / 2]) == np.float64(f[k3, k2, k1])


# ---------------------------------------------------------------------------
# Intersection and pixels
# ---------------------------------------------------------------------------
def _dda_cells(o, d, n):
    """Amanatides-Woo 3D-DDA through an n^3 grid on [0,1]^3; (cell, length) list."""
    t0, t1 = -np.inf, np.inf
    for k in range(3):
        if d[k] == 0:
            if not 0 <= o[k] <= 1:
                return []
            continue
        a, b = (0 - o[k]) / d[k], (1 - o[k]) / d[k]
        t0, t1 = max(t0, min(a, b)), min(t1, max(a, b))
    t0 = max(t0, 0.0)
    if not t1 > t0:
        return []
    p = o + t0 * d
    cell = np.clip(np.floor(p * n).astype(int), 0, n - 1)
    step = np.sign(d).astype(int)
    tmax = np.array([((cell[k] + (step[k] > 0)) / n - o[k]) / d[k] if d[k] != 0 else np.inf for k in range(3)])
    tdel = np.array([abs(1.0 / (n * d[k])) if d[k] != 0 else np.inf for k in range(3)])
    out, t = [], t0
    while True:
        k = int(np.argmin(tmax))
        tn = min(tmax[k], t1)
        out.append((tuple(cell), (tn - t) * np.linalg.norm(d)))
        if tmax[k] >= t1:
            break
        t = tmax[k]
        cell[k] += step[k]
        tmax[k] += tdel[k]
        if not 0 <= cell[k] < n:
            break
    return out


def test_c1_hits_vs_dda_P10():
    sc = sg.config1()
    o = oracle.OracleScene(sc)
    res = o.render(mode="rule", cap=32)
    idx = {tuple((sc.leaf_anchor[e] >> 15).tolist()): e for e in range(sc.num_leaves)}
    W = sc.camera.width
    assert res["total_hits"] == 15412 and (res["nhits"] > 0).sum() == 1928
    nbad = 0
    for q, pix in enumerate(res["pixels"]):
        ro, rd = o.ray(pix % W, pix // W)
        dda = {idx[c] for c, ln in _dda_cells(ro, rd, 8) if ln > 0}
        hl = res["hits"][q]
        hl = hl[hl["elem"] >= 0]
        amb = set(hl["elem"][(hl["flags"] & oracle.AMBIGUOUS) != 0].tolist())
        hit = set(hl["elem"][(hl["flags"] & oracle.HIT) != 0].tolist())
        if (hit - amb) != (dda - amb):
            nbad += 1
    assert nbad == 0


def _chord_unit_cube(o, d, amin, amax):
    t0, t1 = amin, amax
    for k in range(3):
        if d[k] == 0:
            if not 0 <= o[k] <= 1:
                return 0.0
            continue
        a, b = (0 - o[k]) / d[k], (1 - o[k]) / d[k]
        t0, t1 = max(t0, min(a, b)), min(t1, max(a, b))
    return max(0.0, t1 - t0) * np.linalg.norm(d)


@pytest.mark.parametrize("which", ["c1", "c2", "uni4"])
def test_constant_medium_whole_domain_chord_P8_P3(which):
    """f == const: every pixel equals Eq. ABconstant with L = chord of the ray
    through [0,1]^3, whatever the mesh (refinement invariance P3)."""
    if which == "c1":
        base = sg.config1(width=32)
    elif which == "c2":
        base = sg.config2(width=32, maxlevel=5)
    else:
        anchor, tree, lev = sg.uniform_leaves(1, 4)
        base = sg.Scene("u4", 1, 1, sg.identity_cube_ctrl(), anchor, tree, lev,
                        np.zeros((anchor.shape[0], 8), np.float32), 5.0, 1.0, 1.0, sg.config1(width=32).camera)
    sc = sg.constant_field(base, 0.4)
    o = oracle.OracleScene(sc)
    res = o.render(mode="exact", cap=64, with_hits=False)
    ft = float(np.float32(0.4))
    kap = 5.0 * ft * ft
    q = np.array([(1 + ft) / 2, (1 - ft) / 2, 0.5])
    amin, amax = (0.0, 100.0) if sc.camera.projection == 1 else (1.0, 100.0)
    for q_i, pix in enumerate(res["pixels"]):
        ro, rd = o.ray(pix % sc.camera.width, pix // sc.camera.width)
        L = _chord_unit_cube(ro, rd, amin, amax)
        a = math.exp(-kap * L)
        exp_rgb = q * (1 - a) / kap
        np.testing.assert_allclose(res["rgba"][q_i, :3], exp_rgb, atol=2e-12)
        assert abs(res["rgba"][q_i, 3] - (1 - a)) < 2e-12


def test_general_path_reproduces_slab_P9():
    """The face-root intersection on identity control points (an affine lattice)
    reproduces the slab test."""
    sc = sg.config1(width=16)
    o = oracle.OracleScene(sc)
    rng = np.random.default_rng(7)
    pairs = [(int(rng.integers(512)), int(rng.integers(16)), int(rng.integers(16))) for _ in range(300)]
    try:
        ref = [o.intersect(e, i, j) for e, i, j in pairs]
        oracle.set_force_general(True)
        gen = [o.intersect(e, i, j) for e, i, j in pairs]
    finally:
        oracle.set_force_general(False)
    for (s0, f0), (s1, f1) in zip(ref, gen):
        if (f0 | f1) & oracle.AMBIGUOUS:
            continue
        assert s0.shape == s1.shape
        np.testing.assert_allclose(s0, s1, atol=1e-11)


def test_curved_intersection_residual_and_dense_sampling_P11():
    sh = sg.shell_uniform(1, 48, 4)
    o = oracle.OracleScene(sh)
    vis, amb, rects = o.cull()
    rng = np.random.default_rng(8)
    checked = 0
    for e in rng.permutation(sh.num_leaves)[:25]:
        rc = rects[e]
        for _ in range(6):
            i = int(rng.integers(rc[0], rc[1] + 1)); j = int(rng.integers(rc[2], rc[3] + 1))
            seg, fl = o.intersect(int(e), i, j)
            if fl & oracle.AMBIGUOUS:
                continue
            ro, rd = o.ray(i, j)
            for a0, a1 in seg:
                for al in (a0, a1):
                    st, xi = o.inverse_map(int(e), ro + al * rd)
                    assert st == 0
                    assert np.all(xi > -1e-9) and np.all(xi < 1 + 1e-9)
                    assert np.min(np.minimum(np.abs(xi), np.abs(1 - xi))) < 1e-9   # on the boundary
            # dense sampling of the ray near the element: inside <=> in a segment
            lo, hi = o.aabb(int(e))
            alphas = np.linspace(lo[2] * 0.999, hi[2] * 1.001, 400) / np.linalg.norm(sh.camera.view)
            for al in alphas:
                st, xi = o.inverse_map(int(e), ro + al * rd)
                inside = st == 0 and np.all(xi >= 0) and np.all(xi <= 1)
                inseg = any(a0 <= al <= a1 for a0, a1 in seg)
                near = any(min(abs(al - a0), abs(al - a1)) * np.linalg.norm(rd) < 1e-7 for a0, a1 in seg)
                if not near:
                    assert inside == inseg
            checked += 1
    assert checked > 40


def test_partition_invariance_and_any_order_fold_P4_P5():
    """Split the leaves into SFC ranges, render each range separately, merge
    the per-pixel segment lists: equals the single render.  Random tree-shaped
    (+) folds and inserted empty gaps (1,0) leave pixels unchanged."""
    sc = sg.config1(width=24)
    o = oracle.OracleScene(sc)
    full = o.render(mode="rule", cap=32)
    parts = [oracle.OracleScene(sc.subset(lo, hi)).render(mode="rule", cap=32) for lo, hi in
             ((0, 100), (100, 333), (333, 512))]
    offs = (0, 100, 333)
    rng = np.random.default_rng(9)
    for q in range(full["pixels"].shape[0]):
        segs = []
        for p, off in zip(parts, offs):
            h = p["hits"][q]
            h = h[(h["elem"] >= 0) & ((h["flags"] & oracle.HIT) != 0)].copy()
            h["elem"] += off
            segs.append(h)
        segs = np.concatenate(segs)
        rgba, ab = oracle.fold_pixel(segs[rng.permutation(len(segs))])
        np.testing.assert_allclose(rgba, full["rgba"][q], atol=1e-13)
        if len(segs) < 2:
            continue
        # any-order (random tree) fold of the alpha-sorted list
        srt = segs[np.argsort(segs["alpha_near"])]
        items = [(s["a"], s["b"][0]) for s in srt]
        while len(items) > 1:
            k = int(rng.integers(len(items) - 1))
            items[k:k + 2] = [oracle.combine(items[k], items[k + 1])]
        assert abs(items[0][0] - ab[0]) < 1e-13 and abs(items[0][1] - ab[1]) < 1e-13
        # empty gaps: shrink every segment's far end a little and insert (1,0) gaps
        gap = srt.copy()
        extra = gap.copy()
        extra["alpha_near"] = gap["alpha_far"]
        extra["alpha_far"] = gap["alpha_far"] + 1e-3
        extra["a"] = 1.0
        extra["b"] = 0.0
        shifted = gap.copy()
        shifted["alpha_near"] += np.arange(len(gap)) * 1e-3
        shifted["alpha_far"] += np.arange(len(gap)) * 1e-3
        extra["alpha_near"] += np.arange(len(gap)) * 1e-3
        extra["alpha_far"] += np.arange(len(gap)) * 1e-3
        rgba2, _ = oracle.fold_pixel(np.concatenate([shifted, extra]))
        np.testing.assert_allclose(rgba2, rgba, atol=1e-13)


def test_overlap_cut_and_average():
    """Overlapping segments [0,2] and [1,3] of constant media:
    fold equals pieces [0,1] of s1, average over [1,2], [2,3] of s2 (Eq.
    segsplit + segaverage), all written out here."""
    s1 = oracle.from_constant(0.8, 0.5, 2.0)
    s2 = oracle.from_constant(0.3, 1.2, 2.0)
    h = np.zeros(2, dtype=oracle.HIT_DTYPE)
    h["elem"] = [0, 1]
    h["alpha_near"] = [0.0, 1.0]; h["alpha_far"] = [2.0, 3.0]
    h["a"] = [s1[0], s2[0]]
    h["b"] = [[s1[1]] * 3, [s2[1]] * 3]
    rgba, ab = oracle.fold_pixel(h)
    p1 = oracle.from_constant(0.8, 0.5, 1.0)
    mid = ((math.exp(-0.8) * math.exp(-0.3)) ** 0.5, 0.5 * (0.5 / 0.8 * (1 - math.exp(-0.8)) + 1.2 / 0.3 *
                                                            (1 - math.exp(-0.3))))
    p3 = oracle.from_constant(0.3, 1.2, 1.0)
    ref = oracle.combine(oracle.combine(p1, mid), p3)
    assert abs(ab[0] - ref[0]) < 1e-14 and abs(ab[1] - ref[1]) < 1e-14
    # identical intervals -> channel-wise average
    h["alpha_near"] = [0.0, 0.0]; h["alpha_far"] = [2.0, 2.0]
    rgba, ab = oracle.fold_pixel(h)
    avg = oracle.average(s1, s2)
    assert abs(ab[0] - avg[0]) < 1e-14 and abs(ab[1] - avg[1]) < 1e-14


def load_overlap_cases():
    """tests/golden/overlap_cases.txt -> [(name, HIT_DTYPE segments, (A, B))]."""
    import os
    cases, cur = [], None
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "overlap_cases.txt")):
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        if t[0] == "case":
            cur = [t[1], [], None]
        elif t[0] == "seg":
            cur[1].append(tuple(float(x) for x in t[1:5]))
        elif t[0] == "expect":
            cur[2] = (float(t[1]), float(t[2]))
        elif t[0] == "end":
            h = np.zeros(len(cur[1]), dtype=oracle.HIT_DTYPE)
            for k, (an, af, a, b) in enumerate(cur[1]):
                h[k]["elem"] = k
                h[k]["alpha_near"], h[k]["alpha_far"], h[k]["a"] = an, af, a
                h[k]["b"] = b
                h[k]["flags"] = oracle.HIT
            cases.append((cur[0], h, cur[2]))
    return cases


@pytest.mark.parametrize("case", load_overlap_cases(), ids=lambda c: c[0])
def test_overlap_clusters_hand_evaluated(case):
    """Nested, triple, third-before-cut, A = 1, identical and touching segments
    (D14) against the hand-evaluated values of
    tests/golden/overlap_cases.txt, in every input order."""
    import itertools
    name, h, (A, B) = case
    for perm in itertools.permutations(range(len(h))):
        rgba, ab = oracle.fold_pixel(h[list(perm)])
        assert abs(ab[0] - A) < 1e-15 and np.all(np.abs(ab[1:] - B) < 1e-15), (name, ab, A, B)


def test_c1_rule_vs_exact_discretisation():
    """the N=4 rule differs from exact mode by ~5e-9 on C1 (diagnostic)."""
    o = oracle.OracleScene(sg.config1(width=32))
    r1 = o.render(mode="rule", N=4, with_hits=False)
    r2 = o.render(mode="exact", with_hits=False)
    d = np.abs(r1["rgba"] - r2["rgba"]).max()
    assert 1e-11 < d < 1e-7


def test_generator_pins():
    c2 = sg.config2(width=64)
    assert c2.num_leaves == 87088                   # SURVEY A1 (literal rule)
    k = sg.morton_key(c2.leaf_anchor).astype(np.int64)
    assert np.all(np.diff(k) > 0)
    c1 = sg.config1()
    assert c1.num_leaves == 512 and abs(1 / c1.inv_F - 1.0) < 1e-12
    sh = sg.shell_uniform(2, 32, 8)
    assert sh.num_leaves == 6 * 64
    # cubed-sphere control points lie on spheres of radius 0.55 / 0.775 / 1
    r = np.linalg.norm(sh.tree_ctrl, axis=-1)
    for m3, rr in enumerate((0.55, 0.775, 1.0)):
        np.testing.assert_allclose(r[:, m3], rr, atol=1e-15)


def test_skimming_rays_two_roots_one_face_P11():
    """Rays grazing the outer sphere face enter and exit through the SAME
    curved face (<= 8 roots per biquadratic face).  For
    every candidate pair of coarse level-1 elements near the silhouette the
    segments must equal the inside-intervals found by dense sampling of the
    inverse map (brute force), ambiguous or not, away from 1e-6 of an end."""
    sh = sg.shell_uniform(1, 48, 4)
    o = oracle.OracleScene(sh)
    vis, amb, rects = o.cull()
    W = sh.camera.width
    checked, skims = 0, 0
    for e in range(sh.num_leaves):
        if not vis[e]:
            continue
        rc = rects[e]
        for j in range(rc[2], rc[3] + 1, 2):
            for i in range(rc[0], rc[1] + 1, 2):
                ro, rd = o.ray(i, j)
                if abs(np.linalg.norm(np.cross(ro, rd)) / np.linalg.norm(rd) - 1.0) > 0.08:
                    continue          # keep rays passing near the outer silhouette only
                seg, fl = o.intersect(e, i, j)
                lo, hi = o.aabb(e)
                al = np.linspace(lo[2] * 0.999, hi[2] * 1.001, 3000)
                inside = []
                for a in al:
                    st, xi = o.inverse_map(e, ro + a * rd)
                    inside.append(st == 0 and np.all(xi >= 0) and np.all(xi <= 1))
                for a, ins in zip(al, inside):
                    inseg = any(a0 <= a <= a1 for a0, a1 in seg)
                    near = any(min(abs(a - a0), abs(a - a1)) * np.linalg.norm(rd) < 2e-6 for a0, a1 in seg)
                    if not near:
                        assert ins == inseg, (e, i, j, a, seg)
                checked += 1
                if len(seg) and np.sum(np.diff(np.r_[False, inside, False].astype(int)) == 1) >= 1:
                    st0, x0 = o.inverse_map(e, ro + seg[0][0] * rd)
                    st1, x1 = o.inverse_map(e, ro + seg[-1][1] * rd)
                    if abs(x0[2] - 1) < 1e-9 and abs(x1[2] - 1) < 1e-9:
                        skims += 1       # entry and exit on the outer face
    assert checked > 50 and skims > 3


# ---------------------------------------------------------------------------
# The paper's integrators with Alg. 1
# ---------------------------------------------------------------------------
def _amp(scheme, z):
    """Stability function R(z) of the explicit schemes for y' = lambda y (z = lambda dx)."""
    return {"euler": 1 + z, "heun2": 1 + z + z * z / 2, "heun3": 1 + z + z * z / 2 + z ** 3 / 6,
            "rk4": 1 + z + z * z / 2 + z ** 3 / 6 + z ** 4 / 24}[scheme]


@pytest.mark.parametrize("scheme", ["euler", "heun2", "heun3", "rk4"])
def test_alg1_constant_medium_closed_form(scheme):
    """Constant beta = 10, gamma = 2, dx = 1, c_RK = 0.5: Alg. 1 halves the step
    until dx beta <= c_RK, i.e. to 1/32 (depth ceil(log2(10/0.5)) = 5);
    the explicit scheme then applies its stability function R(z), z = -10/32,
    32 times: A = R^32, and B = (gamma/beta)(1 - A) because every RK method
    keeps the equilibrium gamma/beta of B' = gamma - beta B exactly."""
    a, b, depth, fl = oracle.segment_scheme(scheme, lambda s: (10.0, 2.0), 1.0, c_rk=0.5)
    A = _amp(scheme, -10.0 / 32) ** 32
    assert depth == 5 and fl == 0
    assert abs(a - A) <= 1e-13 * abs(A)
    assert np.all(np.abs(b - 0.2 * (1 - A)) <= 1e-13)


def test_alg1_empirical_orders():
    """Halving c_RK on a smooth medium: error ratios 2^M for the explicit
    M-stage schemes ("error rate of c_RK^M"), 2^4 for Gauss-2 ("rate
    c_RK^2M"), 2^2 for Simpson's B; exact mode is the
    reference (P12-pinned)."""
    fn = lambda s: (1.0 + 0.5 * math.sin(3 * s), [0.3 + 0.2 * math.cos(2 * s), 0.5, 0.1 * s])
    ae, be, _ = oracle.segment_exact(fn, 1.7)
    for scheme, order in (("euler", 1), ("heun2", 2), ("heun3", 3), ("rk4", 4), ("gauss2", 4), ("simpson", 2)):
        errs = []
        for c in (0.2, 0.1, 0.05):
            a, b, _, _ = oracle.segment_scheme(scheme, fn, 1.7, c_rk=c)
            errs.append(max(abs(a - ae), float(np.abs(b - be).max())))
        rates = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
        assert all(abs(r - order) <= 0.5 for r in rates), (scheme, rates)


def test_gauss2_and_simpson_special_cases():
    """Gauss-2 without recursion: A -> 1 for dx beta -> infinity (the unphysical
    limit the paper notes); Simpson: A exact for constant
    beta (Eq. simpson), B = gamma dx (b0 A + b1 sqrt(A) + b2) written out."""
    a, b, _, _ = oracle.segment_scheme("gauss2", lambda s: (1e7, 1.0), 1.0, c_rk=0.0)
    assert abs(a - 1.0) < 1e-5
    a, b, d, _ = oracle.segment_scheme("simpson", lambda s: (0.8, 0.3), 2.0, c_rk=0.0)
    A = math.exp(-1.6)
    assert d == 0 and abs(a - A) < 1e-15
    assert np.all(np.abs(b - 2.0 * 0.3 * (A / 6 + 4 / 6 * math.sqrt(A) + 1 / 6)) < 1e-15)
    # gauss2 with recursion: depth ceil(log2(beta L / c)) and the exact constant-medium value within c^4
    a, b, d, _ = oracle.segment_scheme("gauss2", lambda s: (4.0, 1.0), 1.0, c_rk=0.25)
    assert d == 4 and abs(a - math.exp(-4.0)) < 1e-5


def test_curved_pairs_linear_world_field_P16():
    """Per-pair (a, b) on curved R=2 elements with a NON-constant field
    (closes the "parity unpinned" gap of DESIGN §3): nodal values of
    f(x) = c.x + d at the element's GLL nodes mapped through the tree's R=2
    Lagrange map J_k (evaluated in tests/parity_util.py with a textbook
    Lagrange basis, not the oracle), so f o X_E is triquadratic and the P = 2
    interpolation is exact.  Along a ray f is linear in alpha, kappa = kappa0 f^2
    quadratic: A = exp(-int kappa ds) is a polynomial integral (numpy, exact)
    and B = int q(s) exp(-int_0^s kappa) ds (s from the near end, the
    orientation pinned by test_exact_vs_scipy_ode_orientation) a scipy
    quadrature in world coordinates.  A wrong inverse map, interpolation or
    quadrature in the oracle's per-pair path changes (a, b)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from parity_util import linear_field_segment, linear_field_shell
    cvec, d0 = np.array([0.21, 0.11, -0.17]), 0.05
    sc = linear_field_shell(sg.shell_uniform(2, 24, 4, gl_points=6), cvec, d0)
    kap0 = float(np.float32(sc.kappa0))
    o = oracle.OracleScene(sc)
    W = sc.camera.width
    pix = np.arange(0, W * sc.camera.height, 7, dtype=np.int32)
    res = o.render(pixels=pix, mode="exact", with_hits=True, cap=32)
    nchk = 0
    for q_i, p in enumerate(res["pixels"]):
        ro, rd = o.ray(int(p) % W, int(p) // W)
        for h in res["hits"][q_i][:int(res["nhits"][q_i])]:
            if h["elem"] < 0 or not (h["flags"] & oracle.HIT) or (h["flags"] & oracle.AMBIGUOUS):
                continue
            an, af = float(h["alpha_near"]), float(h["alpha_far"])
            if af - an < 1e-6:
                continue
            A, B = linear_field_segment(ro, rd, an, af, cvec, d0, kap0)
            # bound: the nodal values are fp32 (relative 6e-8), so tau is off by <= 1.2e-7 tau
            np.testing.assert_allclose(h["a"], A, rtol=5e-7, atol=1e-12)
            np.testing.assert_allclose(h["b"], B, rtol=5e-7, atol=1e-10)
            nchk += 1
    assert nchk > 200, nchk
