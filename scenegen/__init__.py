"""Seeded synthetic scene generator shared by the CUDA path and the oracle.

This module holds NO arithmetic of the raycasting method (no Lagrange
evaluation, no intersection, no integration, no segment algebra).  It only
builds the inputs the paper's method consumes (§2.1 domain
description; §2.2 camera):

* a forest of trees given by per-tree control points on Gauss-Lobatto nodes
  (the *scene definition*: identity cube or the cubed-sphere shell of
  SURVEY.md §8(c) R21),
* SFC (Morton, x fastest) ordered leaves: anchor (units of 2^-18), tree, level,
* a per-element nodal scalar field at element-local GLL nodes.  Node positions
  are computed from the *exact* scene geometry (unit cube / exact gnomonic
  cubed sphere), never through the degree-R Lagrange map of the method, so the
  generator shares no method arithmetic with either implementation,
* the transfer constants (kappa0, 1/F, q0) of SURVEY.md §8(c) R12,
* the camera frame of SURVEY.md §8(c) R3/R4.

Seeds: numpy default_rng(seed) (PCG64); draw order sources -> centers ->
sigma -> amplitudes.  Large configs evaluate the field
with torch on the given device in fp64 and round once to fp32.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

MAXLEVEL = 18  # anchor units 2^-18 of the tree cube

PERSPECTIVE = 0
ORTHOGRAPHIC = 1


@dataclasses.dataclass
class Camera:
    projection: int
    origin: np.ndarray      # o (perspective) / image-plane centre P0 (ortho)
    view: np.ndarray        # v, |v| = n (perspective) / unit direction d (ortho)
    right: np.ndarray       # t
    up: np.ndarray          # u
    pixel_size: float       # l
    far_dist: float         # f
    width: int
    height: int
    gl_points: int = 4
    newton_tol: float = 1e-6
    newton_max_iter: int = 20


@dataclasses.dataclass
class Scene:
    name: str
    geom_degree: int                 # R
    field_degree: int                # P
    tree_ctrl: np.ndarray            # float64 [K][R+1][R+1][R+1][3], index [k][m3][m2][m1][xyz]
    leaf_anchor: np.ndarray          # int32 [n][3]
    leaf_tree: np.ndarray            # int32 [n]
    leaf_level: np.ndarray           # int8  [n]
    leaf_field: np.ndarray           # float32 [n][(P+1)^3], node order [k3][k2][k1]
    kappa0: float
    inv_F: float
    q0: float
    camera: Camera
    tiles: tuple = (1, 1)
    coarsen_cycles: int = 0
    notes: str = ""
    # surface forests (§2.8; NEXT(3)): dim = 2 means quadtree
    # leaves (anchor z = 0) on bilinear tree patches tree_ctrl [K][2][2][3]
    # ([k][m2][m1][xyz]) with 4 corner values per leaf ([k2][k1]); `surface` is
    # the transfer (a0, a1, ((i0, i1, i2) per RGB channel), k): A_s = clamp(a0 +
    # a1 v, 0, 1), I_s = i0 + i1 v + i2 exp(-((1 - v) k)^2 / 2)
    dim: int = 3
    surface: tuple = (0.0, 0.0, ((0.0, 0.0, 0.0),) * 3, 0.0)

    @property
    def num_leaves(self) -> int:
        return int(self.leaf_tree.shape[0])

    @property
    def num_trees(self) -> int:
        return int(self.tree_ctrl.shape[0])

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.tree_ctrl, self.leaf_anchor, self.leaf_tree, self.leaf_level, self.leaf_field):
            h.update(np.ascontiguousarray(_np(a)).tobytes())
        return h.hexdigest()

    def subset(self, lo: int, hi: int) -> "Scene":
        """Contiguous SFC range [lo, hi) of the leaves (same trees/camera)."""
        return dataclasses.replace(
            self, name=f"{self.name}[{lo}:{hi}]",
            leaf_anchor=self.leaf_anchor[lo:hi], leaf_tree=self.leaf_tree[lo:hi],
            leaf_level=self.leaf_level[lo:hi], leaf_field=self.leaf_field[lo:hi])


def _np(a):
    if isinstance(a, np.ndarray):
        return a
    return a.detach().cpu().numpy()


# ---------------------------------------------------------------------------
# Gauss-Lobatto nodes of the scene definition (R <= 2 only: {0,1}, {0,1/2,1}).
# PAPER.md:119-126, 151-152 (Eq. nodal).
# ---------------------------------------------------------------------------
def gll_nodes(R: int) -> np.ndarray:
    if R == 1:
        return np.array([0.0, 1.0])
    if R == 2:
        return np.array([0.0, 0.5, 1.0])
    raise ValueError("scene generator supports R in {1,2}")


# ---------------------------------------------------------------------------
# Morton keys (x fastest), 18 bits per axis.
# ---------------------------------------------------------------------------
def _spread3(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x3FFFF)
    out = np.zeros_like(v)
    for b in range(18):
        out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
    return out


def morton_key(anchor: np.ndarray) -> np.ndarray:
    a = np.asarray(anchor)
    return _spread3(a[:, 0]) | (_spread3(a[:, 1]) << np.uint64(1)) | (_spread3(a[:, 2]) << np.uint64(2))


def _compact3(k: np.ndarray, L: int) -> np.ndarray:
    out = np.zeros_like(k)
    for b in range(L):
        out |= ((k >> np.uint64(3 * b)) & np.uint64(1)) << np.uint64(b)
    return out


def uniform_leaves(num_trees: int, level: int):
    """All leaves of a uniform level-`level` forest, tree-major, Morton within a tree."""
    n1 = 8 ** level
    idx = np.arange(n1, dtype=np.uint64)
    x = _compact3(idx, level)
    y = _compact3(idx >> np.uint64(1), level)
    z = _compact3(idx >> np.uint64(2), level)
    sh = np.uint64(MAXLEVEL - level)
    anc1 = np.stack([x << sh, y << sh, z << sh], axis=1).astype(np.int32)
    anchor = np.tile(anc1, (num_trees, 1))
    tree = np.repeat(np.arange(num_trees, dtype=np.int32), n1)
    lev = np.full(num_trees * n1, level, dtype=np.int8)
    return anchor, tree, lev


def refine_leaves(num_trees: int, level0: int, maxlevel: int, rule):
    """Adaptive forest: start uniform at level0; refine leaves where
    rule(tree, anchor, level) is True, up to maxlevel.  Returns SFC order."""
    anc, tree, lev = uniform_leaves(num_trees, level0)
    done_a, done_t, done_l = [], [], []
    for L in range(level0, maxlevel + 1):
        if anc.shape[0] == 0:
            break
        if L == maxlevel:
            sel = np.zeros(anc.shape[0], dtype=bool)
        else:
            sel = np.asarray(rule(tree, anc, L), dtype=bool)
        done_a.append(anc[~sel]); done_t.append(tree[~sel]); done_l.append(lev[~sel])
        pa, pt = anc[sel], tree[sel]
        h = np.int32(1 << (MAXLEVEL - L - 1))
        kids = []
        for c in range(8):
            off = np.array([(c & 1) * h, ((c >> 1) & 1) * h, ((c >> 2) & 1) * h], dtype=np.int32)
            kids.append(pa + off)
        anc = np.concatenate(kids, axis=0) if kids else pa
        tree = np.tile(pt, 8)
        lev = np.full(anc.shape[0], L + 1, dtype=np.int8)
    A = np.concatenate(done_a); T = np.concatenate(done_t); Lv = np.concatenate(done_l)
    key = morton_key(A)
    order = np.lexsort((key, T))
    return A[order].copy(), T[order].copy(), Lv[order].copy()


# ---------------------------------------------------------------------------
# Scene geometries (the "a-priori definition of the geometry")
# ---------------------------------------------------------------------------
def identity_cube_ctrl(R: int = 1) -> np.ndarray:
    eta = gll_nodes(R)
    z = np.zeros((1, R + 1, R + 1, R + 1, 3))
    for m3 in range(R + 1):
        for m2 in range(R + 1):
            for m1 in range(R + 1):
                z[0, m3, m2, m1] = (eta[m1], eta[m2], eta[m3])
    return z


def affine_ctrl(R: int, M: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Control points of the affine map t -> M t + c (used for SURVEY P9 tests)."""
    base = identity_cube_ctrl(R)
    return (base @ np.asarray(M, dtype=np.float64).T) + np.asarray(c, dtype=np.float64)


R_IN, R_OUT = 0.55, 1.0


def _shell_point(k, t1, t2, t3, xp=np):
    """Exact (gnomonic / equidistant) cubed-sphere shell map of tree k."""
    a = k // 2
    s = 1.0 - 2.0 * (k % 2)
    b = (a + 1) % 3
    c = (a + 2) % 3
    pa = s * xp.ones_like(t1)
    pb = 2.0 * t1 - 1.0
    pc = s * (2.0 * t2 - 1.0)
    comps = [None, None, None]
    comps[a], comps[b], comps[c] = pa, pb, pc
    p = xp.stack(comps, axis=-1)
    nrm = xp.sqrt((p * p).sum(axis=-1, keepdims=True))
    r = R_IN + (R_OUT - R_IN) * t3
    return r[..., None] * p / nrm


def shell_ctrl(R: int = 2) -> np.ndarray:
    eta = gll_nodes(R)
    z = np.zeros((6, R + 1, R + 1, R + 1, 3))
    for k in range(6):
        for m3 in range(R + 1):
            for m2 in range(R + 1):
                for m1 in range(R + 1):
                    z[k, m3, m2, m1] = _shell_point(k, np.array(eta[m1]), np.array(eta[m2]), np.array(eta[m3]))
    return z


# ---------------------------------------------------------------------------
# Cameras (PAPER.md:208-236 Eq. ray)
# ---------------------------------------------------------------------------
def _frame(view_dir):
    vh = np.asarray(view_dir, dtype=np.float64)
    vh = vh / np.linalg.norm(vh)
    zhat = np.array([0.0, 0.0, 1.0])
    u = zhat - zhat.dot(vh) * vh
    if np.linalg.norm(u) < 1e-9:   # view along +-z: SURVEY R3's up vector is undefined, use +y instead
        yhat = np.array([0.0, 1.0, 0.0])
        u = yhat - yhat.dot(vh) * vh
    u /= np.linalg.norm(u)
    t = np.cross(vh, u)
    return vh, t, u


def perspective_camera(origin, target, fov_deg, w, h, n=1.0, f=100.0, gl_points=4, **kw) -> Camera:
    o = np.asarray(origin, dtype=np.float64)
    vh, t, u = _frame(np.asarray(target, dtype=np.float64) - o)
    ell = 2.0 * n * math.tan(math.radians(fov_deg) / 2.0) / w
    return Camera(PERSPECTIVE, o, n * vh, t, u, ell, f, w, h, gl_points, **kw)


def orthographic_camera(center, direction, dist, span, w, h, gl_points=4, **kw) -> Camera:
    vh, t, u = _frame(direction)
    p0 = np.asarray(center, dtype=np.float64) - dist * vh
    return Camera(ORTHOGRAPHIC, p0, vh, t, u, span / w, 100.0, w, h, gl_points, **kw)


# ---------------------------------------------------------------------------
# Fields
# ---------------------------------------------------------------------------
def _node_coords_tree(scene_kind, P, anchor, tree, level, xp=np):
    """World coordinates of element-local GLL nodes ([n][(P+1)^3][3]) via the
    exact scene geometry.  Node order [k3][k2][k1]."""
    eta = gll_nodes(P)
    K3, K2, K1 = np.meshgrid(eta, eta, eta, indexing="ij")
    xi = np.stack([K1.ravel(), K2.ravel(), K3.ravel()], axis=-1)  # [(P+1)^3][3]
    if xp is np:
        anc = anchor.astype(np.float64) / (1 << MAXLEVEL)
        hE = np.ldexp(1.0, -level.astype(np.int64))[:, None, None]
        t = anc[:, None, :] + hE * xi[None, :, :]
    else:
        import torch
        xi_t = torch.as_tensor(xi, dtype=torch.float64, device=anchor.device)
        anc = anchor.to(torch.float64) / float(1 << MAXLEVEL)
        hE = torch.pow(2.0, -level.to(torch.float64))[:, None, None]
        t = anc[:, None, :] + hE * xi_t[None, :, :]
    if scene_kind == "cube":
        return t
    # shell: per-tree exact map
    out = xp.zeros_like(t) if xp is np else t.new_zeros(t.shape)
    for k in range(6):
        m = tree == k
        if (m.sum() if xp is np else int(m.sum().item())) == 0:
            continue
        tk = t[m]
        out[m] = _shell_point(k, tk[..., 0], tk[..., 1], tk[..., 2], xp=xp)
    return out


def _bumps_eval(x, centers, sigma, amp, xp=np):
    if xp is np:
        f = np.zeros(x.shape[:-1])
        for c, s, a in zip(centers, sigma, amp):
            d2 = ((x - c) ** 2).sum(axis=-1)
            f += a * np.exp(-d2 / (2.0 * s * s))
        return f
    import torch
    C = torch.as_tensor(centers, dtype=torch.float64, device=x.device)
    S = torch.as_tensor(sigma, dtype=torch.float64, device=x.device)
    A = torch.as_tensor(amp, dtype=torch.float64, device=x.device)
    f = torch.zeros(x.shape[:-1], dtype=torch.float64, device=x.device)
    for i in range(C.shape[0]):
        d2 = ((x - C[i]) ** 2).sum(dim=-1)
        f += A[i] * torch.exp(-d2 / (2.0 * S[i] * S[i]))
    return f


def _shell_volume_points(rng, n):
    d = rng.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = (R_IN ** 3 + rng.uniform(size=n) * (R_OUT ** 3 - R_IN ** 3)) ** (1.0 / 3.0)
    return d * r[:, None]


def _field_from(scene_kind, P, anchor, tree, level, fn, device=None, chunk=1 << 22):
    """Evaluate fn(x [m][nodes][3]) per element in fp64; return fp64 values."""
    n = anchor.shape[0]
    if device is None or device == "numpy":
        vals = np.empty((n, (P + 1) ** 3))
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            x = _node_coords_tree(scene_kind, P, anchor[lo:hi], tree[lo:hi], level[lo:hi])
            vals[lo:hi] = fn(x, np)
        return vals
    import torch
    dev = torch.device(device)
    out = torch.empty((n, (P + 1) ** 3), dtype=torch.float64, device=dev)
    A = torch.as_tensor(anchor, device=dev)
    T = torch.as_tensor(tree, device=dev)
    Lv = torch.as_tensor(level, device=dev)
    ch = max(1, chunk // 8)
    for lo in range(0, n, ch):
        hi = min(n, lo + ch)
        x = _node_coords_tree(scene_kind, P, A[lo:hi], T[lo:hi], Lv[lo:hi], xp=torch)
        out[lo:hi] = fn(x, torch)
    return out


def _finish(name, R, P, ctrl, anchor, tree, level, fvals, camera, tiles=(1, 1), cycles=0, notes="",
            kappa0=5.0, q0=1.0, F=None):
    """Normalise the transfer (F = max |nodal f|, fp64) and round the field to fp32 once."""
    if isinstance(fvals, np.ndarray):
        Fm = float(np.abs(fvals).max()) if F is None else F
        field = fvals.astype(np.float32)
    else:
        Fm = float(fvals.abs().max().item()) if F is None else F
        field = fvals.to(dtype=__import__("torch").float32)
    return Scene(name, R, P, ctrl, anchor, tree, level, field, kappa0, 1.0 / Fm, q0, camera,
                 tiles, cycles, notes)


# ---------------------------------------------------------------------------
# BASELINE.json configs and small test variants
# ---------------------------------------------------------------------------
C2_EYE = np.array([2.5, 1.8, 1.2])
SHELL_EYE = 3.0 * C2_EYE / np.linalg.norm(C2_EYE)


def config1(width=64) -> Scene:
    """C1: identity cube, uniform level 3, ortho camera along (1,.3,.2), sin field."""
    anchor, tree, level = uniform_leaves(1, 3)
    cam = orthographic_camera([0.5, 0.5, 0.5], [1.0, 0.3, 0.2], 2.0, math.sqrt(3.0), width, width, gl_points=4)

    def fn(x, xp):
        return xp.sin(2 * math.pi * x[..., 0]) * xp.sin(2 * math.pi * x[..., 1]) * xp.sin(2 * math.pi * x[..., 2])

    f = _field_from("cube", 1, anchor, tree, level, fn)
    return _finish("C1", 1, 1, identity_cube_ctrl(1), anchor, tree, level, f, cam)


def _c2_rule(band=1.0):
    def rule(tree, anc, L):
        h = 1.0 / (1 << L)
        c = anc.astype(np.float64) / (1 << MAXLEVEL) + 0.5 * h
        r = np.linalg.norm(c - 0.5, axis=1)
        return np.abs(r - 0.3) < band * h
    return rule


def cube_bumps(nb, seed):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(size=(nb, 3))
    sigma = rng.uniform(0.03, 0.15, size=nb)
    amp = rng.uniform(0.5, 1.0, size=nb)
    return centers, sigma, amp


def config2(width=512, maxlevel=7, band=1.0, seed=0, fov=40.0, target=(0.5, 0.5, 0.5), name="C2",
            device=None) -> Scene:
    """C2: identity cube, adaptive levels 3..maxlevel around the r=0.3 sphere, 16 bumps."""
    anchor, tree, level = refine_leaves(1, 3, maxlevel, _c2_rule(band))
    centers, sigma, amp = cube_bumps(16, seed)
    cam = perspective_camera(C2_EYE, target, fov, width, width, gl_points=4)
    f = _field_from("cube", 1, anchor, tree, level, lambda x, xp: _bumps_eval(x, centers, sigma, amp, xp),
                    device=device)
    return _finish(name, 1, 1, identity_cube_ctrl(1), anchor, tree, level, f, cam)


def shell_bumps(nb, seed):
    rng = np.random.default_rng(seed)
    centers = _shell_volume_points(rng, nb)
    sigma = rng.uniform(0.03, 0.15, size=nb)
    amp = rng.uniform(0.5, 1.0, size=nb)
    return centers, sigma, amp


def shell_uniform(level, width, nbumps, seed=0, gl_points=6, name=None, tiles=(1, 1), device=None,
                  fov=40.0) -> Scene:
    anchor, tree, lev = uniform_leaves(6, level)
    centers, sigma, amp = shell_bumps(nbumps, seed)
    cam = perspective_camera(SHELL_EYE, [0.0, 0.0, 0.0], fov, width, width, gl_points=gl_points)
    if device is not None and device != "numpy":
        # same bump sum in fp64 by the generator's CUDA helper (scenegen/gpu.py)
        import torch
        from . import gpu
        A, T, Lv = (torch.as_tensor(x, device=device) for x in (anchor, tree, lev))
        f, F = gpu.shell_bumps_field(A, T, Lv, 2, centers, sigma, amp)
        return _finish(name or f"shell-L{level}", 2, 2, shell_ctrl(2), A, T, Lv, f, cam, tiles, F=F)
    f = _field_from("shell", 2, anchor, tree, lev, lambda x, xp: _bumps_eval(x, centers, sigma, amp, xp))
    return _finish(name or f"shell-L{level}", 2, 2, shell_ctrl(2), anchor, tree, lev, f, cam, tiles)


def config3(device=None) -> Scene:
    return shell_uniform(6, 1024, 64, name="C3", device=device)


def config4(device=None) -> Scene:
    return shell_uniform(8, 2048, 256, name="C4", tiles=(8, 8), device=device)


def config5(device=None, c=14.0, maxlevel=10, level0=4, width=4096, nsources=512) -> Scene:
    """C5: shell adaptive around 512 sources: start uniform
    at level 4, refine E (level < 10) iff its exact-shell centre is closer than
    c 2^-level to a source; field = the 512 Gaussian bumps at the sources.
    ~1.9e8 leaves: generated on the GPU (scenegen/gpu.py, fp64 inside, field
    rounded once to fp32).  Smaller variants (maxlevel, width, nsources) serve
    the tests."""
    rng = np.random.default_rng(0)
    sources = _shell_volume_points(rng, nsources)
    sigma = rng.uniform(0.03, 0.15, size=nsources)
    amp = rng.uniform(0.5, 1.0, size=nsources)
    cam = perspective_camera(SHELL_EYE, [0.0, 0.0, 0.0], 40.0, width, width, gl_points=8)
    if device is None or device == "numpy":
        def rule(tree, anc, L):
            h = 1.0 / (1 << L)
            t = anc.astype(np.float64) / (1 << MAXLEVEL) + 0.5 * h
            out = np.zeros(anc.shape[0], dtype=bool)
            for k in range(6):
                m = tree == k
                if not m.any():
                    continue
                x = _shell_point(k, t[m, 0], t[m, 1], t[m, 2])
                d = np.full(x.shape[0], np.inf)
                for s_ in sources:
                    d = np.minimum(d, np.linalg.norm(x - s_, axis=1))
                out[m] = d < c * h
            return out

        anchor, tree, lev = refine_leaves(6, level0, maxlevel, rule)
        f = _field_from("shell", 2, anchor, tree, lev, lambda x, xp: _bumps_eval(x, sources, sigma, amp, xp))
        return _finish("C5", 2, 2, shell_ctrl(2), anchor, tree, lev, f, cam, (8, 8), 3)
    from . import gpu
    anchor, tree, lev = gpu.refine_leaves_shell(level0, maxlevel, sources, c, device)
    field, F = gpu.shell_bumps_field(anchor, tree, lev, 2, sources, sigma, amp)
    return _finish("C5", 2, 2, shell_ctrl(2), anchor, tree, lev, field, cam, (8, 8), 3, F=F)


def constant_field(scene: Scene, value: float = 0.7) -> Scene:
    """Same forest/camera with f == value everywhere (SURVEY pins P3, P8, P14).
    F is kept at 1 so kappa = kappa0 * value^2."""
    fld = np.full_like(_np(scene.leaf_field), np.float32(value))
    return dataclasses.replace(scene, name=scene.name + "-const", leaf_field=fld, inv_F=1.0)


# ---------------------------------------------------------------------------
# Surface workload (NEXT(3)): the Mandelbrot hexagon of PAPER.md:1296-1367
# ---------------------------------------------------------------------------
HEX_TOP = ((-2.3, 0.75), (-0.25, 1.8), (1.3, 1.0))   # PAPER.md:1316-1320; bottom: y negated


def _spread2(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x3FFFF)
    out = np.zeros_like(v)
    for b in range(18):
        out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
    return out


def hexagon_ctrl(bend: float = 0.0) -> np.ndarray:
    """Two bilinear quadtree patches [2][2][2][3] ([k][m2][m1][xyz]) forming the
    hexagon (tree 0: x <= -1/4, tree 1: x >= -1/4; t1 along x, t2 along y).
    bend != 0 lifts the corners to +-bend/2 (saddle patches, continuous across
    the shared edge) so that the ray-patch equation is a true quadratic."""
    (t1x, t1y), (t2x, t2y), (t3x, t3y) = HEX_TOP
    T1, T2, T3 = (t1x, t1y), (t2x, t2y), (t3x, t3y)
    B1, B2, B3 = (t1x, -t1y), (t2x, -t2y), (t3x, -t3y)
    z = np.zeros((2, 2, 2, 3))
    h = 0.5 * bend
    for k, (c00, c01, c10, c11, zs) in enumerate(((B1, B2, T1, T2, (h, -h, -h, h)),
                                                   (B2, B3, T2, T3, (-h, h, h, -h)))):
        for q, c in enumerate((c00, c01, c10, c11)):
            z[k, q // 2, q % 2] = (c[0], c[1], zs[q])
    return z


def mandelbrot_value(x, y, max_iter: int):
    """Escape count of z <- z^2 + c, z0 = 0, c = x + i y (Eq. mbiter) divided by
    max_iter: the first m >= 1 with |z_m| > 2, else max_iter."""
    c = np.asarray(x, dtype=np.float64) + 1j * np.asarray(y, dtype=np.float64)
    z = np.zeros_like(c)
    n = np.full(c.shape, max_iter, dtype=np.int64)
    alive = np.ones(c.shape, dtype=bool)
    for m in range(1, max_iter + 1):
        z = np.where(alive, z * z + c, z)
        esc = alive & (np.abs(z) > 2.0)
        n[esc] = m
        alive &= ~esc
    return n / float(max_iter)


def _hex_corner_xy(ctrl, tree, anchor, level):
    """xy of the 4 corners [k2][k1] of quadtree leaves (bilinear tree map)."""
    h = np.ldexp(1.0, -level.astype(np.int64))
    out = np.zeros((tree.shape[0], 4, 3))
    for q in range(4):
        t1 = anchor[:, 0] / float(1 << MAXLEVEL) + h * (q % 2)
        t2 = anchor[:, 1] / float(1 << MAXLEVEL) + h * (q // 2)
        Z = ctrl[tree]
        out[:, q] = ((1 - t2)[:, None] * ((1 - t1)[:, None] * Z[:, 0, 0] + t1[:, None] * Z[:, 0, 1]) +
                     t2[:, None] * ((1 - t1)[:, None] * Z[:, 1, 0] + t1[:, None] * Z[:, 1, 1]))
    return out


SURF_OPAQUE = (0.0, 0.0, ((0.5, 0.5, 0.0),) * 3, 0.0)                      # grey to white, A_s = 0
SURF_TRANSPARENT = (0.8, -0.5, ((0.1, 0.2, 0.8), (0.1, 0.2, 0.8), (0.2, 0.3, 0.0)), 20.0)   # yellow near the limit


def mandelbrot_hexagon(level0=3, maxlevel=7, max_iter=30, width=256, bend=0.0, opaque=False, camera=None,
                       name="MB") -> Scene:
    """The Mandelbrot surface: two quadtrees mapped to the
    hexagon, uniform at level0, refined where an element's four corner values
    differ (up to maxlevel; D18: no 2:1 balance, corner values taken
    at every leaf corner), bilinear corner values = escape count / max_iter."""
    ctrl = hexagon_ctrl(bend)
    n1 = 4 ** level0
    idx = np.arange(n1, dtype=np.uint64)
    # Morton (x fastest) in 2D: bits alternate x, y
    xs = np.zeros(n1, dtype=np.uint64)
    ys = np.zeros(n1, dtype=np.uint64)
    for b in range(level0):
        xs |= ((idx >> np.uint64(2 * b)) & np.uint64(1)) << np.uint64(b)
        ys |= ((idx >> np.uint64(2 * b + 1)) & np.uint64(1)) << np.uint64(b)
    sh = np.uint64(MAXLEVEL - level0)
    anc = np.tile(np.stack([xs << sh, ys << sh, np.zeros_like(xs)], axis=1).astype(np.int32), (2, 1))
    tree = np.repeat(np.arange(2, dtype=np.int32), n1)
    lev = np.full(2 * n1, level0, dtype=np.int8)
    done = []
    for L in range(level0, maxlevel + 1):
        if anc.shape[0] == 0:
            break
        xy = _hex_corner_xy(ctrl, tree, anc, lev)
        v = mandelbrot_value(xy[..., 0], xy[..., 1], max_iter)
        sel = np.zeros(anc.shape[0], dtype=bool) if L == maxlevel else (v.max(axis=1) != v.min(axis=1))
        done.append((anc[~sel], tree[~sel], lev[~sel], v[~sel]))
        pa, pt = anc[sel], tree[sel]
        hh = np.int32(1 << (MAXLEVEL - L - 1))
        kids = [pa + np.array([(c & 1) * hh, ((c >> 1) & 1) * hh, 0], dtype=np.int32) for c in range(4)]
        anc = np.concatenate(kids, axis=0)
        tree = np.tile(pt, 4)
        lev = np.full(anc.shape[0], L + 1, dtype=np.int8)
    A = np.concatenate([d[0] for d in done])
    T = np.concatenate([d[1] for d in done])
    Lv = np.concatenate([d[2] for d in done])
    V = np.concatenate([d[3] for d in done])
    key = _spread2(A[:, 0]) | (_spread2(A[:, 1]) << np.uint64(1))
    order = np.lexsort((key, T))
    if camera is None:
        camera = perspective_camera([-0.5, -2.6, 3.2], [-0.5, 0.0, 0.0], 62.0, width, width)
    surf = SURF_OPAQUE if opaque else SURF_TRANSPARENT
    return Scene(name, 1, 1, ctrl, A[order].copy(), T[order].copy(), Lv[order].copy(),
                 V[order].astype(np.float32), 0.0, 1.0, 0.0, camera, dim=2, surface=surf,
                 notes=f"Mandelbrot hexagon, levels {level0}..{maxlevel}, {max_iter} iterations, bend {bend}")


def get_config(cid: int, **kw) -> Scene:
    return {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[cid](**kw)
