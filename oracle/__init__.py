"""ctypes binding of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1809_01334_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

HIT, AMBIGUOUS, NEWTON_FAIL, OVERFLOW, SPLIT_NEAR = 1, 2, 4, 8, 16
SCHEMES = {"gl": 0, "euler": 1, "heun2": 2, "heun3": 3, "rk4": 4, "gauss2": 5, "simpson": 6}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (IEEE fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


class Scene_(C.Structure):
    _fields_ = [("R", C.c_int32), ("P", C.c_int32), ("K", C.c_int32), ("tree_ctrl", C.c_void_p),
                ("n", C.c_int64), ("anchor", C.c_void_p), ("tree", C.c_void_p), ("level", C.c_void_p),
                ("field", C.c_void_p), ("kappa0", C.c_double), ("inv_F", C.c_double), ("q0", C.c_double),
                ("dim", C.c_int32), ("surf_a", C.c_double * 2), ("surf_i", C.c_double * 9), ("surf_k", C.c_double)]


class Camera_(C.Structure):
    _fields_ = [("projection", C.c_int32), ("origin", C.c_double * 3), ("view", C.c_double * 3),
                ("right", C.c_double * 3), ("up", C.c_double * 3), ("pixel_size", C.c_double),
                ("far_dist", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


HIT_DTYPE = np.dtype([("elem", np.int64), ("pixel", np.int32), ("flags", np.int32),
                      ("alpha_near", np.float64), ("alpha_far", np.float64), ("a", np.float64),
                      ("b", np.float64, (3,))])

class Pairs_(C.Structure):
    _fields_ = [("npix", C.c_int64), ("off", C.POINTER(C.c_int64)), ("elem", C.POINTER(C.c_int64)),
                ("flags", C.POINTER(C.c_int32))]


MEDIUM_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double))

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d = C.c_double
        P = C.POINTER
        _lib.orc_combine.argtypes = [d, d, d, d, P(d), P(d)]
        _lib.orc_inverse.argtypes = [d, d, P(d), P(d)]
        _lib.orc_split.argtypes = [d, d, d, d, P(d)]
        _lib.orc_average.argtypes = [d, d, d, d, P(d), P(d)]
        _lib.orc_from_constant.argtypes = [d, d, d, P(d), P(d)]
        _lib.orc_background.argtypes = [d, d, d]
        _lib.orc_background.restype = d
        _lib.orc_gauss_legendre.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_lagrange_integrals.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_segment_exact.argtypes = [MEDIUM_FN, C.c_void_p, d, P(d), C.c_void_p]
        _lib.orc_segment_rule.argtypes = [C.c_int, MEDIUM_FN, C.c_void_p, d, P(d), C.c_void_p]
        _lib.orc_gll.argtypes = [C.c_int, C.c_void_p]
        _lib.orc_lagrange.argtypes = [C.c_int, C.c_void_p, d, C.c_void_p, C.c_void_p]
        _lib.orc_tree_map.argtypes = [P(Scene_), C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_element_map.argtypes = [P(Scene_), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_camera_transform.argtypes = [P(Camera_), C.c_void_p, C.c_void_p]
        _lib.orc_ray.argtypes = [P(Camera_), C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_element_aabb.argtypes = [P(Scene_), P(Camera_), C.c_int64, C.c_void_p, C.c_void_p]
        _lib.orc_pixel_rect.argtypes = [P(Camera_), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_cull.argtypes = [P(Scene_), P(Camera_), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_field.argtypes = [P(Scene_), C.c_int64, C.c_void_p]
        _lib.orc_field.restype = d
        _lib.orc_inverse_map.argtypes = [P(Scene_), C.c_int64, C.c_void_p, C.c_void_p]
        _lib.orc_intersect.argtypes = [P(Scene_), P(Camera_), C.c_int64, C.c_int, C.c_int, C.c_int,
                                       C.c_void_p, P(C.c_int)]
        _lib.orc_render.argtypes = [P(Scene_), P(Camera_), C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_int]
        _lib.orc_render.restype = C.c_int64
        _lib.orc_render_ex.argtypes = [P(Scene_), P(Camera_), C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                       C.c_void_p, P(Pairs_), C.c_void_p]
        _lib.orc_render_ex.restype = C.c_int64
        _lib.orc_pairs_free.argtypes = [P(Pairs_)]
        _lib.orc_segment_scheme.argtypes = [C.c_int, C.c_int, d, C.c_int, MEDIUM_FN, C.c_void_p, d, P(d),
                                            C.c_void_p, P(C.c_int)]
        _lib.orc_set_scheme.argtypes = [C.c_int, d, C.c_int]
        _lib.orc_medium_evals.argtypes = [C.c_int]
        _lib.orc_medium_evals.restype = C.c_longlong
        _lib.orc_set_force_general.argtypes = [C.c_int]
        _lib.orc_surface_roots.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, d, d, C.c_void_p]
        _lib.orc_fold_pixel.argtypes = [C.c_int, C.c_void_p, d, C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleScene:
    """Holds contiguous numpy copies of a scenegen.Scene and its C structs."""

    def __init__(self, scene):
        def npy(a, dt):
            a = a if isinstance(a, np.ndarray) else a.detach().cpu().numpy()
            return np.ascontiguousarray(a, dtype=dt)

        self.scene = scene
        self.ctrl = npy(scene.tree_ctrl, np.float64)
        self.anchor = npy(scene.leaf_anchor, np.int32)
        self.tree = npy(scene.leaf_tree, np.int32)
        self.level = npy(scene.leaf_level, np.int8)
        self.field = npy(scene.leaf_field, np.float32)
        self.s = Scene_(scene.geom_degree, scene.field_degree, self.ctrl.shape[0], _ptr(self.ctrl).value,
                        self.anchor.shape[0], _ptr(self.anchor).value, _ptr(self.tree).value,
                        _ptr(self.level).value, _ptr(self.field).value, scene.kappa0, scene.inv_F, scene.q0,
                        int(getattr(scene, "dim", 3)))
        if self.s.dim == 2:
            a0, a1, ii, k = scene.surface
            self.s.surf_a[:] = [float(a0), float(a1)]
            self.s.surf_i[:] = [float(x) for row in ii for x in row]
            self.s.surf_k = float(k)
        cam = scene.camera
        self.c = Camera_(cam.projection, (C.c_double * 3)(*cam.origin), (C.c_double * 3)(*cam.view),
                         (C.c_double * 3)(*cam.right), (C.c_double * 3)(*cam.up), cam.pixel_size, cam.far_dist,
                         cam.width, cam.height)
        self.W, self.H = cam.width, cam.height

    # ---- geometry helpers
    def ray(self, i, j):
        o = np.zeros(3); r = np.zeros(3)
        lib().orc_ray(C.byref(self.c), i, j, _ptr(o), _ptr(r))
        return o, r

    def element_map(self, e, xi):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        x = np.zeros(3); J = np.zeros(9)
        lib().orc_element_map(C.byref(self.s), e, _ptr(xi), _ptr(x), _ptr(J))
        return x, J.reshape(3, 3)

    def tree_map(self, k, t):
        t = np.ascontiguousarray(t, dtype=np.float64)
        x = np.zeros(3)
        lib().orc_tree_map(C.byref(self.s), k, _ptr(t), _ptr(x))
        return x

    def camera_transform(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        X = np.zeros(3)
        lib().orc_camera_transform(C.byref(self.c), _ptr(x), _ptr(X))
        return X

    def aabb(self, e):
        lo = np.zeros(3); hi = np.zeros(3)
        lib().orc_element_aabb(C.byref(self.s), C.byref(self.c), e, _ptr(lo), _ptr(hi))
        return lo, hi

    def pixel_rect(self, lo, hi):
        lo = np.ascontiguousarray(lo, dtype=np.float64); hi = np.ascontiguousarray(hi, dtype=np.float64)
        rc = np.zeros(4, dtype=np.int32)
        ok = lib().orc_pixel_rect(C.byref(self.c), _ptr(lo), _ptr(hi), _ptr(rc))
        return bool(ok), rc

    def field_at(self, e, xi):
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        return lib().orc_field(C.byref(self.s), e, _ptr(xi))

    def inverse_map(self, e, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        xi = np.zeros(3)
        st = lib().orc_inverse_map(C.byref(self.s), e, _ptr(x), _ptr(xi))
        return st, xi

    def cull(self):
        n = self.anchor.shape[0]
        vis = np.zeros(n, dtype=np.int8); amb = np.zeros(n, dtype=np.int8)
        rects = np.zeros((n, 4), dtype=np.int32)
        lib().orc_cull(C.byref(self.s), C.byref(self.c), _ptr(vis), _ptr(amb), _ptr(rects))
        return vis.astype(bool), amb.astype(bool), rects

    def intersect(self, e, i, j, max_seg=8):
        seg = np.zeros((max_seg, 2))
        fl = C.c_int(0)
        ns = lib().orc_intersect(C.byref(self.s), C.byref(self.c), e, i, j, max_seg, _ptr(seg), C.byref(fl))
        return seg[:min(ns, max_seg)], fl.value

    def render(self, pixels=None, mode="exact", N=None, background=(0.0, 0.0, 0.0), cap=64, with_hits=True,
               nthreads=0):
        if pixels is None:
            pixels = np.arange(self.W * self.H, dtype=np.int32)
        pixels = np.ascontiguousarray(pixels, dtype=np.int32)
        npix = pixels.shape[0]
        N = N or self.scene.camera.gl_points
        bg = np.ascontiguousarray(background, dtype=np.float64)
        rgba = np.zeros((npix, 4)); nh = np.zeros(npix, dtype=np.int32); na = np.zeros(npix, dtype=np.int32)
        hits = np.zeros((npix, cap), dtype=HIT_DTYPE) if with_hits else None
        total = lib().orc_render(C.byref(self.s), C.byref(self.c), 0 if mode == "exact" else 1, N, _ptr(bg), npix,
                                 _ptr(pixels), _ptr(rgba), _ptr(nh), _ptr(na), cap,
                                 _ptr(hits) if with_hits else None, nthreads)
        return dict(pixels=pixels, rgba=rgba, nhits=nh, namb=na, hits=hits, total_hits=int(total))


    def render_pairs(self, pixels=None, mode="exact", N=None, background=(0.0, 0.0, 0.0), nthreads=0,
                     with_cull=True, rects=None):
        """orc_render_ex: pixel values plus, per pixel, the (elem, flags) of every
        hit or eps-ambiguous candidate pair (CSR: pair_off[npix+1], pair_elem,
        pair_flags) and the culled list of the same run.  mode "hits" skips the
        integration (rgba = 0)."""
        if pixels is None:
            pixels = np.arange(self.W * self.H, dtype=np.int32)
        pixels = np.ascontiguousarray(pixels, dtype=np.int32)
        npix = pixels.shape[0]
        N = N or self.scene.camera.gl_points
        bg = np.ascontiguousarray(background, dtype=np.float64)
        rgba = np.zeros((npix, 4)); nh = np.zeros(npix, dtype=np.int32); na = np.zeros(npix, dtype=np.int32)
        n = self.anchor.shape[0]
        if rects is not None:
            with_cull = False
            rects = np.ascontiguousarray(rects, dtype=np.int32)
        vis = np.zeros(n, dtype=np.int8) if with_cull else None
        amb = np.zeros(n, dtype=np.int8) if with_cull else None
        pr = Pairs_()
        m = {"exact": 0, "rule": 1, "hits": 2, "scheme": 3}[mode]
        total = lib().orc_render_ex(C.byref(self.s), C.byref(self.c), m, N, _ptr(bg), npix, _ptr(pixels),
                                    _ptr(rgba), _ptr(nh), _ptr(na), nthreads,
                                    _ptr(vis) if with_cull else None, _ptr(amb) if with_cull else None,
                                    C.byref(pr), _ptr(rects) if rects is not None else None)
        off = np.ctypeslib.as_array(pr.off, shape=(npix + 1,)).copy()
        tot = int(off[-1])
        elem = np.ctypeslib.as_array(pr.elem, shape=(max(tot, 1),))[:tot].copy()
        flags = np.ctypeslib.as_array(pr.flags, shape=(max(tot, 1),))[:tot].copy()
        lib().orc_pairs_free(C.byref(pr))
        out = dict(pixels=pixels, rgba=rgba, nhits=nh, namb=na, total_hits=int(total), pair_off=off,
                   pair_elem=elem, pair_flags=flags)
        if with_cull:
            out["visible"] = vis.astype(bool)
            out["ambiguous"] = amb.astype(bool)
        return out


# ---- algebra / quadrature wrappers --------------------------------------
def combine(near, far):
    a = C.c_double(); b = C.c_double()
    lib().orc_combine(near[0], near[1], far[0], far[1], C.byref(a), C.byref(b))
    return a.value, b.value


def inverse(s):
    a = C.c_double(); b = C.c_double()
    st = lib().orc_inverse(s[0], s[1], C.byref(a), C.byref(b))
    if st:
        raise ValueError("segment with A = 0 has no inverse")
    return a.value, b.value


def split(s, dx1, dx2):
    out = (C.c_double * 4)()
    st = lib().orc_split(s[0], s[1], dx1, dx2, out)
    if st:
        raise ValueError("invalid split lengths")
    return (out[0], out[1]), (out[2], out[3])


def average(s1, s2):
    a = C.c_double(); b = C.c_double()
    lib().orc_average(s1[0], s1[1], s2[0], s2[1], C.byref(a), C.byref(b))
    return a.value, b.value


def from_constant(beta, gamma, dx):
    a = C.c_double(); b = C.c_double()
    lib().orc_from_constant(beta, gamma, dx, C.byref(a), C.byref(b))
    return a.value, b.value


def background(s, Ib):
    return lib().orc_background(s[0], s[1], Ib)


def gauss_legendre(N):
    u = np.zeros(N); w = np.zeros(N)
    lib().orc_gauss_legendre(N, _ptr(u), _ptr(w))
    return u, w


def lagrange_integrals(N, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    S = np.zeros((N, N))
    lib().orc_lagrange_integrals(N, _ptr(u), _ptr(S))
    return S


def _medium(fn):
    def cb(ctx, s, kap, q3):
        k, q = fn(s)
        kap[0] = k
        q = np.broadcast_to(np.asarray(q, dtype=np.float64), (3,))
        for c in range(3):
            q3[c] = q[c]
    return MEDIUM_FN(cb)


def segment_exact(fn, L):
    """fn(s) -> (kappa, q or q[3]); s from the near end.  Returns (a, b[3], panels)."""
    a = C.c_double(); b = np.zeros(3)
    cb = _medium(fn)
    M = lib().orc_segment_exact(cb, None, L, C.byref(a), _ptr(b))
    return a.value, b, M


def segment_rule(N, fn, L):
    a = C.c_double(); b = np.zeros(3)
    cb = _medium(fn)
    lib().orc_segment_rule(N, cb, None, L, C.byref(a), _ptr(b))
    return a.value, b


def segment_scheme(scheme, fn, L, N=4, c_rk=0.0, max_depth=24):
    """Alg. 1 adaptive integration with scheme in SCHEMES.
    Returns (a, b[3], depth, flags)."""
    a = C.c_double(); b = np.zeros(3); fl = C.c_int(0)
    cb = _medium(fn)
    depth = lib().orc_segment_scheme(SCHEMES[scheme], N, c_rk, max_depth, cb, None, L, C.byref(a), _ptr(b),
                                     C.byref(fl))
    return a.value, b, depth, fl.value


def medium_evals(reset=False):
    """Field evaluations made by orc_render since the last reset (diagnostic)."""
    return int(lib().orc_medium_evals(1 if reset else 0))


def set_scheme(scheme, c_rk=0.0, max_depth=24):
    """Scheme of OracleScene.render_pairs(mode="scheme")."""
    lib().orc_set_scheme(SCHEMES[scheme], c_rk, max_depth)


def gll(R):
    eta = np.zeros(R + 1)
    lib().orc_gll(R, _ptr(eta))
    return eta


def lagrange(R, eta, t):
    eta = np.ascontiguousarray(eta, dtype=np.float64)
    psi = np.zeros(R + 1); dpsi = np.zeros(R + 1)
    lib().orc_lagrange(R, _ptr(eta), t, _ptr(psi), _ptr(dpsi))
    return psi, dpsi


def set_force_general(on: bool):
    lib().orc_set_force_general(1 if on else 0)


def fold_pixel(segs, tau=1e-12, background=(0.0, 0.0, 0.0)):
    """segs: structured HIT_DTYPE array (one pixel).  Returns (rgba[4], (T,B[3]))."""
    s = np.ascontiguousarray(segs, dtype=HIT_DTYPE).copy()
    rgba = np.zeros(4); ab = np.zeros(4)
    bg = np.ascontiguousarray(background, dtype=np.float64)
    lib().orc_fold_pixel(s.shape[0], _ptr(s), tau, _ptr(bg), _ptr(rgba), _ptr(ab))
    return rgba, ab


def surface_roots(P, o, r, lo=0.0, hi=1.0):
    """Parameters s = (s1, s2) in [lo, hi)^2 where the ray o + alpha r meets the
    bilinear patch with corners P [2][2][3] ([m2][m1][xyz]) (App. A.1)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    o = np.ascontiguousarray(o, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    out = np.zeros(4)
    n = lib().orc_surface_roots(_ptr(P), _ptr(o), _ptr(r), lo, hi, _ptr(out))
    return out[:2 * n].reshape(n, 2)
