"""Pins of the oracle's surface path (NEXT(3); §2.8 Eq. ABphi,
PAPER.md:1473-1514 App. A.1 ray-patch intersection, PAPER.md:1296-1367 the
Mandelbrot hexagon) against closed forms, brute force and special cases.
CPU only."""
import math

import numpy as np
import pytest

import oracle
import scenegen as sg
from scenegen import Scene


# ---------------------------------------------------------------- scene data
def test_mandelbrot_values_closed_form():
    """Eq. mbiter escape counts worked by hand: c = 1 (1, 2, 5: escapes at m=3),
    c = 2 (2, 6: m=2), |c| > 2 escapes at m=1; c = 0, -1 (period 2), i
    (period 2 after i, -1+i, -i) stay bounded (value 1)."""
    mi = 30
    xs = np.array([1.0, 2.0, -2.3, 0.0, -1.0, 0.0, 1.3])
    ys = np.array([0.0, 0.0, 0.75, 0.0, 0.0, 1.0, 1.0])
    got = sg.mandelbrot_value(xs, ys, mi)
    # c = 1.3 + i: z1 = c, |c| = 1.64; z2 = c^2 + c = (1.69 - 1 + 1.3) + (2.6 + 1) i = 1.99 + 3.6 i -> m = 2
    want = np.array([3, 2, 1, mi, mi, mi, 2]) / mi
    assert np.array_equal(got, want)


def test_hexagon_corners_and_shared_edge():
    """The two trees' corners are the paper's six hexagon corners
    and the trees share the edge x = -1/4 (continuous, with and without bend)."""
    hexpts = {(-2.3, 0.75), (-0.25, 1.8), (1.3, 1.0), (-2.3, -0.75), (-0.25, -1.8), (1.3, -1.0)}
    for bend in (0.0, 0.4):
        z = sg.hexagon_ctrl(bend)
        pts = {(round(p[0], 12), round(p[1], 12)) for p in z.reshape(-1, 3)}
        assert pts == hexpts
        assert np.array_equal(z[0, :, 1], z[1, :, 0])   # tree 0's t1 = 1 edge == tree 1's t1 = 0 edge
        assert np.all(np.abs(z[..., 2]) == 0.5 * bend)


def test_mandelbrot_refinement_rule():
    """Leaves tile both trees exactly (areas sum to 1 per tree, SFC order,
    no overlap) and every leaf above maxlevel has equal corner values."""
    sc = sg.mandelbrot_hexagon(2, 7, width=32)
    h = np.ldexp(1.0, -sc.leaf_level.astype(np.int64))
    for k in range(2):
        assert abs((h[sc.leaf_tree == k] ** 2).sum() - 1.0) < 1e-12
    f = sc.leaf_field
    coarse = sc.leaf_level < 7
    assert np.all(f[coarse].max(axis=1) == f[coarse].min(axis=1))
    assert np.all(sc.leaf_anchor[:, 2] == 0)
    # corner values are the escape counts at the corner points (fp32 of k / 30)
    xy = sg._hex_corner_xy(sc.tree_ctrl, sc.leaf_tree, sc.leaf_anchor, sc.leaf_level)
    ref = sg.mandelbrot_value(xy[..., 0], xy[..., 1], 30).astype(np.float32)
    assert np.array_equal(ref, f)


# ---------------------------------------------------------- ray-patch roots
def _square(z=(0.0, 0.0, 0.0, 0.0)):
    """unit square patch, corners [m2][m1], z per corner (00, 10, 01, 11)"""
    return np.array([[[0, 0, z[0]], [1, 0, z[1]]], [[0, 1, z[2]], [1, 1, z[3]]]], dtype=np.float64)


def test_roots_flat_square_vertical_ray():
    P = _square()
    for x, y in ((0.25, 0.5), (0.0, 0.0), (0.9, 0.1)):
        s = oracle.surface_roots(P, [x, y, 3.0], [0, 0, -1])
        assert s.shape == (1, 2) and np.allclose(s[0], (x, y), atol=1e-14)


def test_roots_half_open_and_parallel():
    """s in [0,1)^2: the corner (1,1) and the edges s = 1 belong to the
    neighbours (PAPER.md: half-open leaves); a ray in the patch plane has none."""
    P = _square()
    assert oracle.surface_roots(P, [1.0, 1.0, 3.0], [0, 0, -1]).shape[0] == 0
    assert oracle.surface_roots(P, [0.5, 1.0, 3.0], [0, 0, -1]).shape[0] == 0
    assert oracle.surface_roots(P, [0.0, 0.5, 3.0], [0, 0, -1]).shape[0] == 1
    assert oracle.surface_roots(P, [-0.5, 0.5, 0.0], [1, 0, 0]).shape[0] == 0


@pytest.mark.parametrize("c,z0,m", [(2.0, 0.1, 1.5), (1.0, 0.0, 0.9), (-1.5, -0.2, -1.0), (3.0, 0.5, 1.0)])
def test_roots_saddle_two_hits(c, z0, m):
    """Patch z = c s1 s2 over the unit square, ray in the plane x = y:
    X = (t, t, z0 + m t) meets it where c t^2 - m t - z0 = 0, two roots in
    [0,1) for these cases (App. A.1: at most two intersections)."""
    P = _square((0, 0, 0, c))
    o = np.array([0.0, 0.0, z0])
    r = np.array([1.0, 1.0, m])
    s = oracle.surface_roots(P, o, r)
    disc = m * m + 4 * c * z0
    ts = sorted(t for t in ((m - math.sqrt(disc)) / (2 * c), (m + math.sqrt(disc)) / (2 * c)) if 0 <= t < 1)
    got = sorted(s[:, 0])
    assert len(got) == len(ts) and np.allclose(got, ts, atol=1e-12)
    assert np.allclose(s[:, 0], s[:, 1], atol=1e-12)


def test_roots_random_patches_brute_force():
    """Random non-planar patches and rays: every returned s lies on the ray
    (distance < 1e-10), and no root is missed (dense grid + Newton polish)."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        P = rng.uniform(-1, 1, (2, 2, 3))
        o = rng.uniform(-3, 3, 3)
        tgt = P.reshape(4, 3)[rng.integers(0, 4)] * 0.5 + P.mean(axis=(0, 1)) * 0.5 + rng.normal(0, 0.2, 3)
        r = tgt - o
        s = oracle.surface_roots(P, o, r)

        def X(s1, s2):
            return (1 - s2) * ((1 - s1) * P[0, 0] + s1 * P[0, 1]) + s2 * ((1 - s1) * P[1, 0] + s1 * P[1, 1])

        rh = r / np.linalg.norm(r)

        def dist(s1, s2):
            d = X(s1, s2) - o
            return np.linalg.norm(d - d.dot(rh) * rh)
        for s1, s2 in s:
            assert dist(s1, s2) < 1e-10
        # brute force: from every grid point near the ray, Gauss-Newton on the
        # ray distance; each converged interior solution must be a returned root
        def dX(s1, s2):
            d1 = (1 - s2) * (P[0, 1] - P[0, 0]) + s2 * (P[1, 1] - P[1, 0])
            d2 = (1 - s1) * (P[1, 0] - P[0, 0]) + s1 * (P[1, 1] - P[0, 1])
            return d1, d2
        g = np.linspace(0.0, 1.0, 101)
        S1, S2 = np.meshgrid(g, g, indexing="ij")
        D = np.linalg.norm(np.cross((X(S1[..., None], S2[..., None]) - o), rh), axis=-1)
        for a, b in np.argwhere(D < 2e-2):
            q = np.array([g[a], g[b]])
            for _ in range(30):
                d = X(*q) - o
                res = d - d.dot(rh) * rh
                J = np.stack([v - v.dot(rh) * rh for v in dX(*q)], axis=1)
                q = q - np.linalg.lstsq(J, res, rcond=None)[0]
            if dist(*q) < 1e-11 and min(q[0], q[1], 1 - q[0], 1 - q[1]) > 1e-3:
                assert any(abs(q[0] - q1) < 1e-6 and abs(q[1] - q2) < 1e-6 for q1, q2 in s), (P, o, r, q, s)


# --------------------------------------------------- Eq. ABphi through render
def _one_patch_scene(P, corners, surface, cam):
    return Scene("patch", 1, 1, np.asarray(P, dtype=np.float64)[None], np.zeros((1, 3), np.int32),
                 np.zeros(1, np.int32), np.zeros(1, np.int8), np.asarray([corners], np.float32), 0.0, 1.0, 0.0,
                 cam, dim=2, surface=surface)


def _transfer(surface, v):
    a0, a1, ii, k = surface
    As = min(1.0, max(0.0, a0 + a1 * v))
    w = math.exp(-0.5 * ((1 - v) * k) ** 2)
    return As, [ii[c][0] + ii[c][1] * v + ii[c][2] * w for c in range(3)]


SURF = (0.7, -0.4, ((0.2, 0.5, 0.3), (0.1, 0.2, 0.0), (0.6, -0.3, 0.1)), 3.0)


@pytest.mark.parametrize("theta_deg", [0.0, 30.0, 60.0, 75.0])
def test_abphi_flat_patch_tilted_view(theta_deg):
    """Flat patch z = 0, orthographic rays at angle theta to the normal:
    A = A_s^(1/cos theta), B_c = I_s,c (1 - A) (Eq. ABphi, Eq. BIrelation),
    v the bilinear corner interpolation at the hit point; background 0."""
    th = math.radians(theta_deg)
    d = np.array([math.sin(th), 0.0, -math.cos(th)])
    cam = sg.orthographic_camera([0.5, 0.5, 0.0], d, 3.0, 1.6, 16, 16)
    corners = [0.1, 0.9, 0.4, 0.6]
    sc = _one_patch_scene(_square(), corners, SURF, cam)
    o = oracle.OracleScene(sc)
    res = o.render(mode="rule", with_hits=False)
    rgba = res["rgba"].reshape(16, 16, 4)
    nhit = 0
    for j in range(16):
        for i in range(16):
            org, r = o.ray(i, j)
            t = -org[2] / r[2]
            x, y = org[0] + t * r[0], org[1] + t * r[1]
            if not (0.01 < x < 0.99 and 0.01 < y < 0.99):
                if not (-0.01 <= x <= 1.01 and -0.01 <= y <= 1.01):
                    assert np.all(rgba[j, i] == 0.0)
                continue
            v = (1 - y) * ((1 - x) * corners[0] + x * corners[1]) + y * ((1 - x) * corners[2] + x * corners[3])
            As, I = _transfer(SURF, v)
            A = As ** (1.0 / math.cos(th))
            want = [I[c] * (1 - A) for c in range(3)] + [1 - A]
            assert np.allclose(rgba[j, i], want, atol=1e-12), (i, j, rgba[j, i], want)
            nhit += 1
    assert nhit >= 10


def test_abphi_curved_patch_normal_angle():
    """Saddle patch z = c s1 s2, vertical rays: the hit is (x, y, c x y) and
    cos phi = 1 / |(-c y, -c x, 1)|, so A = A_s^|n| (closed form)."""
    c = 0.8
    cam = sg.orthographic_camera([0.5, 0.5, 0.0], [0.0, 0.0, -1.0], 3.0, 1.0, 12, 12)
    corners = [0.2, 0.5, 0.7, 1.0]
    sc = _one_patch_scene(_square((0, 0, 0, c)), corners, SURF, cam)
    o = oracle.OracleScene(sc)
    rgba = o.render(mode="rule", with_hits=False)["rgba"].reshape(12, 12, 4)
    for j in range(12):
        for i in range(12):
            org, r = o.ray(i, j)
            x, y = org[0], org[1]
            v = (1 - y) * ((1 - x) * corners[0] + x * corners[1]) + y * ((1 - x) * corners[2] + x * corners[3])
            As, I = _transfer(SURF, v)
            A = As ** math.sqrt(1.0 + (c * y) ** 2 + (c * x) ** 2)
            assert np.allclose(rgba[j, i], [I[0] * (1 - A), I[1] * (1 - A), I[2] * (1 - A), 1 - A], atol=1e-12)


def test_opaque_surface_hides_what_is_behind():
    """A_s = 0: A = 0 at any angle, B = I_s, and a surface
    behind contributes nothing; a transparent one in front composes as
    (A1 A2, B1 + A1 B2) (Eq. aggregate)."""
    cam = sg.orthographic_camera([0.5, 0.5, 0.0], [0.2, 0.1, -1.0], 4.0, 0.5, 8, 8)
    front = _square((0.5, 0.5, 0.5, 0.5))
    back = _square()
    ctrl = np.stack([front, back])
    for op_front in (True, False):
        surf = sg.SURF_OPAQUE if op_front else SURF
        sc = Scene("two", 1, 1, ctrl, np.zeros((2, 3), np.int32), np.array([0, 1], np.int32),
                   np.zeros(2, np.int8), np.array([[0.3] * 4, [0.8] * 4], np.float32), 0.0, 1.0, 0.0, cam, dim=2,
                   surface=surf)
        o = oracle.OracleScene(sc)
        res = o.render(mode="rule", with_hits=False)
        rgba = res["rgba"]
        assert np.all(res["nhits"] == 2)
        cphi = 1.0 / np.linalg.norm([0.2, 0.1, -1.0])
        A1s, I1 = _transfer(surf, 0.3)
        A2s, I2 = _transfer(surf, 0.8)
        A1, A2 = A1s ** (1 / cphi), A2s ** (1 / cphi)
        B = [I1[c] * (1 - A1) + A1 * I2[c] * (1 - A2) for c in range(3)]
        if op_front:
            assert A1 == 0.0 and B == I1
        assert np.allclose(rgba, np.array(B + [1 - A1 * A2])[None], atol=1e-12)


def test_hexagon_tiling_one_hit_per_pixel():
    """Flat hexagon forest, orthographic view along -z: every pixel centre
    inside the hexagon (off its boundary and the leaf edges by the ambiguity
    margin) hits exactly one leaf, every centre outside none: the culled
    candidate lists miss no leaf and the half-open leaves do not double count."""
    W = 96
    cam = sg.orthographic_camera([-0.5, 0.0, 0.0], [0.0, 0.0, -1.0], 3.0, 4.0, W, W)
    sc = sg.mandelbrot_hexagon(2, 6, width=W, camera=cam)
    o = oracle.OracleScene(sc)
    res = o.render(mode="rule", with_hits=False)
    hexagon = [(-2.3, 0.75), (-0.25, 1.8), (1.3, 1.0), (1.3, -1.0), (-0.25, -1.8), (-2.3, -0.75)]

    def inside(x, y):
        s = []
        for k in range(6):
            (x0, y0), (x1, y1) = hexagon[k], hexagon[(k + 1) % 6]
            s.append((x1 - x0) * (y - y0) - (y1 - y0) * (x - x0))
        return max(s) < -1e-3 or min(s) > 1e-3, min(abs(q) for q in s) < 1e-3
    nin = 0
    for p in range(W * W):
        org, _ = o.ray(p % W, p // W)
        ins, near = inside(org[0], org[1])
        if near or res["namb"][p]:
            continue
        assert res["nhits"][p] == (1 if ins else 0), (p, org)
        nin += ins
    assert nin > 0.3 * W * W


def test_cull_against_brute_force():
    """Tiny bent hexagon, perspective camera: the hit count of every pixel
    through the culled candidate lists equals brute force over all leaves
    (orc_surface_roots on every leaf's corners, alpha in the view range)."""
    W = 24
    sc = sg.mandelbrot_hexagon(1, 4, width=W, bend=0.5)
    o = oracle.OracleScene(sc)
    res = o.render(mode="rule", with_hits=False)
    P = sg._hex_corner_xy(sc.tree_ctrl, sc.leaf_tree, sc.leaf_anchor, sc.leaf_level).reshape(-1, 2, 2, 3)
    cam = sc.camera
    amin, amax = 1.0, cam.far_dist / np.linalg.norm(cam.view)   # alpha range of a perspective camera
    for p in range(0, W * W, 3):
        org, r = o.ray(p % W, p // W)
        n = 0
        for e in range(P.shape[0]):
            for s1, s2 in oracle.surface_roots(P[e], org, r):
                X = (1 - s2) * ((1 - s1) * P[e, 0, 0] + s1 * P[e, 0, 1]) + s2 * ((1 - s1) * P[e, 1, 0] + s1 * P[e, 1, 1])
                al = (X - org).dot(r) / r.dot(r)
                n += amin <= al <= amax
        if res["namb"][p] == 0:
            assert res["nhits"][p] == n, p
