"""Thin ctypes binding of librc (include/rc.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels of librc.so.  There is no
CPU fallback: a missing or unloadable librc.so raises RcError."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RC_LIB") or os.path.join(HERE, "librc.so")   # RC_LIB: an in-tree build variant

RC_OK = 0
RC_ERR_CAPACITY = -6
STATUS_NAMES = {0: "RC_OK", -1: "RC_ERR_INVALID_ARG", -2: "RC_ERR_NOT_SFC_SORTED", -3: "RC_ERR_OUT_OF_MEMORY",
                -4: "RC_ERR_CUDA", -5: "RC_ERR_NCCL", -6: "RC_ERR_CAPACITY", -7: "RC_ERR_STATE",
                -8: "RC_ERR_NUMERIC"}
RC_HOST_COPY, RC_DEVICE_COPY, RC_HOST_COPY_TRUSTED, RC_DEVICE_BORROW = 0, 1, 2, 3
RC_PERSPECTIVE, RC_ORTHOGRAPHIC = 0, 1
SCHEMES = {"gl": 0, "euler": 1, "heun2": 2, "heun3": 3, "rk4": 4, "gauss2": 5, "simpson": 6}   # RC_SCHEME_*


class RcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Transfer(C.Structure):
    _fields_ = [("kappa0", C.c_float), ("inv_F", C.c_float), ("q0", C.c_float)]


class SurfaceTransfer(C.Structure):
    _fields_ = [("a", C.c_float * 2), ("i", C.c_float * 9), ("k", C.c_float)]


class ForestDesc(C.Structure):
    _fields_ = [("num_trees", C.c_int32), ("geom_degree", C.c_int32), ("tree_ctrl", C.c_void_p),
                ("field_degree", C.c_int32), ("num_leaves", C.c_int64), ("first_global_leaf", C.c_int64),
                ("leaf_anchor", C.c_void_p), ("leaf_tree", C.c_void_p), ("leaf_level", C.c_void_p),
                ("leaf_field", C.c_void_p), ("memory", C.c_int32), ("transfer", Transfer), ("dim", C.c_int32),
                ("surface", SurfaceTransfer)]


class CameraDesc(C.Structure):
    _fields_ = [("projection", C.c_int32), ("origin", C.c_double * 3), ("view", C.c_double * 3),
                ("right", C.c_double * 3), ("up", C.c_double * 3), ("pixel_size", C.c_double),
                ("far_dist", C.c_double), ("width", C.c_int32), ("height", C.c_int32), ("gl_points", C.c_int32),
                ("newton_tol", C.c_double), ("newton_max_iter", C.c_int32), ("scheme", C.c_int32),
                ("c_rk", C.c_double), ("max_depth", C.c_int32)]


class Segments(C.Structure):
    _fields_ = [("count", C.c_int64), ("candidates", C.c_int64), ("hit_pairs", C.c_int64),
                ("newton_failures", C.c_int64), ("face_failures", C.c_int64), ("num_visible", C.c_int64),
                ("raw_segments", C.c_int64), ("level", C.c_int64), ("units", C.c_int64),
                ("unfolded_units", C.c_int64), ("face_tasks", C.c_int64), ("fallback_tasks", C.c_int64),
                ("segs", C.c_void_p),
                ("hits_per_pixel", C.c_void_p), ("depth_capped", C.c_int64)]


class PairResult(C.Structure):
    _fields_ = [("nseg", C.c_int32), ("alpha_near", C.c_float * 4), ("alpha_far", C.c_float * 4),
                ("a", C.c_float * 4), ("b", (C.c_float * 3) * 4)]


class Tiling(C.Structure):
    _fields_ = [("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("nranks", C.c_int32), ("rank", C.c_int32)]


class Marker(C.Structure):
    _fields_ = [("tree", C.c_int32), ("anchor", C.c_int32 * 3)]


SEG_BYTES = 32
EXPORTS = ["rc_last_error", "rc_version", "rc_forest_create", "rc_forest_destroy", "rc_camera_set", "rc_cull",
           "rc_cull_result", "rc_leaf_weights", "rc_cast_segments", "rc_segments_get", "rc_segments_set",
           "rc_debug_pair", "rc_aggregate", "rc_comm_unique_id", "rc_comm_create", "rc_comm_destroy",
           "rc_pack_tiles", "rc_composite_tiles", "rc_composite_records", "rc_composite", "rc_render_frame",
           "rc_launch_count", "rc_last_cast_ms", "rc_last_phase_ms", "rc_node_table", "rc_pool_trim",
           "rc_frame_capture", "rc_frame_replay", "rc_exchange_partners", "rc_comm_set_partners",
           "rc_visible_area_add", "rc_vforest_create", "rc_forest_leaves"]

_lib = None


def lib():
    """Load librc.so (built by paper_1809_01334_b200.build); raise if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RcError(-4, f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.rc_last_error.restype = C.c_char_p
    L.rc_version.restype = i32
    L.rc_forest_create.argtypes = [C.POINTER(ForestDesc), vp, C.POINTER(vp)]
    L.rc_forest_destroy.argtypes = [vp]
    L.rc_camera_set.argtypes = [vp, C.POINTER(CameraDesc), vp]
    L.rc_cull.argtypes = [vp, vp, vp]
    L.rc_cull_result.argtypes = [vp, vp, i64, C.POINTER(i64), vp]
    L.rc_leaf_weights.argtypes = [vp, vp, i64, vp]
    L.rc_segments_set.argtypes = [vp, vp, i64, i32, vp]
    L.rc_debug_pair.argtypes = [vp, i64, i32, i32, C.POINTER(PairResult), vp]
    L.rc_comm_unique_id.argtypes = [C.POINTER(C.c_uint8 * 128)]
    L.rc_comm_create.argtypes = [C.POINTER(C.c_uint8 * 128), i32, i32, vp, C.POINTER(vp)]
    L.rc_comm_destroy.argtypes = [vp]
    L.rc_cast_segments.argtypes = [vp, i32, vp]
    L.rc_node_table.argtypes = [vp, i32, vp, i64, C.POINTER(i64), vp]
    L.rc_segments_get.argtypes = [vp, C.POINTER(Segments), vp]
    L.rc_aggregate.argtypes = [vp, i32, vp]
    L.rc_pack_tiles.argtypes = [vp, C.POINTER(Tiling), vp, C.POINTER(vp), vp]
    L.rc_composite_tiles.argtypes = [vp, C.POINTER(Tiling), vp, vp, vp, i64, vp]
    L.rc_composite_records.argtypes = [vp, C.POINTER(Tiling), vp, i64, vp, vp, i64, vp]
    L.rc_composite.argtypes = [vp, vp, vp, i64, vp]
    L.rc_render_frame.argtypes = [vp, C.POINTER(CameraDesc), i32, i32, vp, vp, i64, C.POINTER(i64), vp]
    L.rc_frame_capture.argtypes = [vp, C.POINTER(CameraDesc), vp, vp, i64, vp]
    L.rc_frame_replay.argtypes = [vp, vp]
    L.rc_exchange_partners.argtypes = [vp, C.POINTER(Tiling), vp, vp, vp]
    L.rc_comm_set_partners.argtypes = [vp, vp, vp]
    L.rc_visible_area_add.argtypes = [vp, vp, i64, vp]
    L.rc_vforest_create.argtypes = [vp, vp, i64, vp, C.POINTER(vp), C.POINTER(i64), vp]
    L.rc_forest_leaves.argtypes = [vp, vp, vp, vp, vp, i64, vp]
    L.rc_launch_count.argtypes = [i32]
    L.rc_launch_count.restype = i64
    L.rc_last_cast_ms.argtypes = [vp]
    L.rc_last_cast_ms.restype = C.c_float
    L.rc_last_phase_ms.argtypes = [vp, i32]
    L.rc_last_phase_ms.restype = C.c_float
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype if name in (
            "rc_last_error", "rc_version", "rc_launch_count", "rc_last_cast_ms", "rc_last_phase_ms") else C.c_int
    _lib = L
    return L


def _check(st):
    if st != RC_OK:
        raise RcError(st, lib().rc_last_error().decode(errors="replace"))


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class _DevArray:
    """Zero-copy __cuda_array_interface__ wrapper of a library-owned buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def device_view(ptr, shape, typestr):
    import torch
    if int(ptr or 0) == 0 or int(np.prod(shape)) == 0:
        dt = {"<i4": torch.int32, "<f4": torch.float32, "<i8": torch.int64, "<u4": torch.int32}[typestr]
        return torch.empty(shape, dtype=dt, device="cuda")
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda")


def camera_desc(cam, gl_points=None, newton_tol=None, newton_max_iter=None, scheme=None, c_rk=None,
                max_depth=None) -> CameraDesc:
    """scheme / c_rk / max_depth: the segment integrator; defaults from the camera
    object's attributes when present, else the R13 GL rule without recursion."""
    d3 = C.c_double * 3
    sch = scheme if scheme is not None else getattr(cam, "scheme", "gl")
    return CameraDesc(int(cam.projection), d3(*map(float, cam.origin)), d3(*map(float, cam.view)),
                      d3(*map(float, cam.right)), d3(*map(float, cam.up)), float(cam.pixel_size),
                      float(cam.far_dist), int(cam.width), int(cam.height),
                      int(gl_points or cam.gl_points), float(newton_tol or cam.newton_tol),
                      int(newton_max_iter or cam.newton_max_iter), SCHEMES[sch] if isinstance(sch, str) else int(sch),
                      float(c_rk if c_rk is not None else getattr(cam, "c_rk", 0.0)),
                      int(max_depth if max_depth is not None else getattr(cam, "max_depth", 0)))


def unpack_segments(raw):
    """raw: int32 tensor [n, 8] of rc_seg records -> dict of column views."""
    import torch
    f = raw.view(torch.float32)
    return {"pixel": raw[:, 0], "alpha_near": f[:, 1], "alpha_far": f[:, 2], "a": f[:, 3], "b": f[:, 4:7],
            "key": raw[:, 7]}


class Forest:
    """rc_forest handle.  Leaf arrays may be numpy (host copy) or CUDA tensors
    (device copy); they are copied by rc_forest_create."""

    def __init__(self, tree_ctrl, geom_degree, field_degree, leaf_anchor, leaf_tree, leaf_level, leaf_field,
                 kappa0, inv_F, q0, first_global_leaf=0, stream=None, trusted=False, dim=3, surface=None,
                 borrow=False):
        import torch
        L = lib()
        ctrl = np.ascontiguousarray(tree_ctrl if isinstance(tree_ctrl, np.ndarray) else tree_ctrl.cpu().numpy(),
                                    dtype=np.float64)
        on_dev = isinstance(leaf_anchor, torch.Tensor) and leaf_anchor.is_cuda
        # leaf_field None: keys-only forest (aggregation / partition bookkeeping, no casting)
        if on_dev:
            keep = [leaf_anchor.contiguous().to(torch.int32), leaf_tree.contiguous().to(torch.int32),
                    leaf_level.contiguous().to(torch.int8),
                    None if leaf_field is None else leaf_field.contiguous().to(torch.float32)]
            ptrs = [0 if t is None else t.data_ptr() for t in keep]
            mem = RC_DEVICE_BORROW if borrow else RC_DEVICE_COPY
        else:
            def npy(a, dt):
                a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
                return np.ascontiguousarray(a, dtype=dt)
            keep = [npy(leaf_anchor, np.int32), npy(leaf_tree, np.int32), npy(leaf_level, np.int8),
                    None if leaf_field is None else npy(leaf_field, np.float32)]
            ptrs = [0 if k is None else k.ctypes.data for k in keep]
            mem = RC_HOST_COPY_TRUSTED if trusted else RC_HOST_COPY
        n = int(keep[1].shape[0])
        self.n = n
        self.P = int(field_degree)
        self.R = int(geom_degree)
        desc = ForestDesc(int(ctrl.shape[0]), int(geom_degree), ctrl.ctypes.data, int(field_degree), n,
                          int(first_global_leaf), ptrs[0], ptrs[1], ptrs[2], ptrs[3] or None, mem,
                          Transfer(float(kappa0), float(inv_F), float(q0)), int(dim))
        if int(dim) == 2:   # surface forest: (a0, a1, ((i0, i1, i2) x 3), k)
            a0, a1, ii, k = surface
            desc.surface.a[:] = [float(a0), float(a1)]
            desc.surface.i[:] = [float(x) for row in ii for x in row]
            desc.surface.k = float(k)
        self.surface = int(dim) == 2
        h = C.c_void_p()
        _check(L.rc_forest_create(C.byref(desc), _stream(stream), C.byref(h)))
        self.h = h
        self._borrowed = keep if (on_dev and borrow) else None   # RC_DEVICE_BORROW: alive as long as the forest
        self.cam = None

    @classmethod
    def from_scene(cls, scene, first=0, count=None, device_copy=False, stream=None, borrow=False):
        """Build from a scenegen.Scene-like object (attributes only, duck typed).
        borrow: the leaves go to the device once and the forest uses them in
        place (RC_DEVICE_BORROW)."""
        import torch
        hi = scene.num_leaves if count is None else first + count
        arrs = [scene.leaf_anchor[first:hi], scene.leaf_tree[first:hi], scene.leaf_level[first:hi],
                scene.leaf_field[first:hi]]
        if device_copy or borrow:
            arrs = [torch.as_tensor(np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a).cuda() for a in arrs]
        return cls(scene.tree_ctrl, scene.geom_degree, scene.field_degree, *arrs, scene.kappa0, scene.inv_F,
                   scene.q0, first_global_leaf=first, stream=stream, dim=getattr(scene, "dim", 3),
                   surface=getattr(scene, "surface", None), borrow=borrow)

    def close(self):
        if getattr(self, "h", None):
            lib().rc_forest_destroy(self.h)
            self.h = None
        self._borrowed = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- pipeline --------------------------------------------------------
    def camera_set(self, cam, stream=None, **kw):
        self.cam = cam
        self.W, self.H = int(cam.width), int(cam.height)
        d = camera_desc(cam, **kw)
        _check(lib().rc_camera_set(self.h, C.byref(d), _stream(stream)))

    def cull(self, stream=None, d_num_visible=None):
        """d_num_visible: optional int64 CUDA tensor receiving the visible count (async)."""
        ptr = C.c_void_p(d_num_visible.data_ptr()) if d_num_visible is not None else None
        _check(lib().rc_cull(self.h, _stream(stream), ptr))

    def leaf_weights(self, out=None, stream=None):
        """Partition weights w_E = rect area + 1 of the last cull (int64 CUDA tensor [n])."""
        import torch
        if out is None:
            out = torch.empty(self.n, dtype=torch.int64, device="cuda")
        _check(lib().rc_leaf_weights(self.h, C.c_void_p(out.data_ptr()), out.numel(), _stream(stream)))
        return out

    def segments_set(self, recs, level, stream=None):
        """Import records (int32 CUDA tensor [n, 8]) as this forest's records at node level `level`."""
        n = int(recs.shape[0])
        ptr = C.c_void_p(recs.data_ptr()) if n else None
        _check(lib().rc_segments_set(self.h, ptr, n, int(level), _stream(stream)))

    def debug_pair(self, local_leaf, i, j, stream=None):
        """One (leaf, pixel) pair evaluated by the segment kernel: list of (an, af, a, b[3])."""
        r = PairResult()
        _check(lib().rc_debug_pair(self.h, int(local_leaf), int(i), int(j), C.byref(r), _stream(stream)))
        return [(r.alpha_near[k], r.alpha_far[k], r.a[k], tuple(r.b[k])) for k in range(r.nseg)]

    def cull_result(self, stream=None):
        import torch
        cnt = C.c_int64()
        buf = torch.empty(self.n, dtype=torch.int32, device="cuda")
        _check(lib().rc_cull_result(self.h, C.c_void_p(buf.data_ptr()), self.n, C.byref(cnt), _stream(stream)))
        return buf[:cnt.value]

    def cast_segments(self, fold_levels=0, stream=None):
        """fold_levels = c: records per (node of coarsening level c, pixel) (row a6)."""
        _check(lib().rc_cast_segments(self.h, int(fold_levels), _stream(stream)))

    def node_table(self, level, stream=None):
        """Local first-leaf index of every node of coarsening level `level`."""
        import torch
        cnt = C.c_int64()
        st = lib().rc_node_table(self.h, int(level), None, 0, C.byref(cnt), _stream(stream))
        if st not in (RC_OK, RC_ERR_CAPACITY):
            _check(st)
        buf = torch.empty(max(cnt.value, 1), dtype=torch.int32, device="cuda")
        _check(lib().rc_node_table(self.h, int(level), C.c_void_p(buf.data_ptr()), buf.numel(), C.byref(cnt),
                                   _stream(stream)))
        return buf[:cnt.value]

    def segments(self, stream=None):
        s = Segments()
        _check(lib().rc_segments_get(self.h, C.byref(s), _stream(stream)))
        raw = device_view(s.segs, (s.count, 8), "<i4")
        hpp = device_view(s.hits_per_pixel, (self.H, self.W), "<i4")
        return {"count": s.count, "candidates": s.candidates, "hit_pairs": s.hit_pairs,
                "newton_failures": s.newton_failures, "face_failures": s.face_failures,
                "num_visible": s.num_visible, "raw": raw, "raw_segments": s.raw_segments, "level": s.level,
                "units": s.units, "unfolded_units": s.unfolded_units, "face_tasks": s.face_tasks,
                "fallback_tasks": s.fallback_tasks, "depth_capped": s.depth_capped,
                "hits_per_pixel": hpp}

    def aggregate(self, cycles, stream=None):
        _check(lib().rc_aggregate(self.h, int(cycles), _stream(stream)))

    def composite(self, background=(0.0, 0.0, 0.0), out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.H, self.W, 4), dtype=torch.float32, device="cuda")
        bg = (C.c_float * 3)(*background)
        _check(lib().rc_composite(self.h, bg, C.c_void_p(out.data_ptr()), out.numel(), _stream(stream)))
        return out

    def pack_tiles(self, tiles_x, tiles_y, nranks, rank, stream=None):
        t = Tiling(tiles_x, tiles_y, nranks, rank)
        counts = (C.c_int64 * nranks)()
        ptr = C.c_void_p()
        _check(lib().rc_pack_tiles(self.h, C.byref(t), counts, C.byref(ptr), _stream(stream)))
        cnt = [int(c) for c in counts]
        raw = device_view(ptr.value, (sum(cnt), 8), "<i4")
        return raw, cnt

    def composite_tiles(self, tiles_x, tiles_y, nranks, rank, recv=None, comm=None, background=(0.0, 0.0, 0.0),
                        out=None, stream=None):
        """This rank's tiles [ntiles][th][tw][4].  comm (a Comm): NCCL exchange
        inside librc (rc_composite_tiles); recv (int32 [n, 8] CUDA tensor):
        composite records moved by the caller (rc_composite_records); neither:
        this forest's own records."""
        import torch
        t = Tiling(tiles_x, tiles_y, nranks, rank)
        tw, th = self.W // tiles_x, self.H // tiles_y
        mine = [(tx, ty) for ty in range(tiles_y) for tx in range(tiles_x) if (tx + ty) % nranks == rank]
        if out is None:
            out = torch.empty((len(mine), th, tw, 4), dtype=torch.float32, device="cuda")
        bg = (C.c_float * 3)(*background)
        if comm is not None:
            _check(lib().rc_composite_tiles(self.h, C.byref(t), comm.h, bg, C.c_void_p(out.data_ptr()), out.numel(),
                                            _stream(stream)))
            return out, mine
        if recv is None:
            _check(lib().rc_composite_records(self.h, C.byref(t), None, 0, bg, C.c_void_p(out.data_ptr()),
                                              out.numel(), _stream(stream)))
            return out, mine
        n = int(recv.shape[0])
        keep = recv if n else torch.empty((1, 8), dtype=torch.int32, device="cuda")   # non-null, count 0
        _check(lib().rc_composite_records(self.h, C.byref(t), C.c_void_p(keep.data_ptr()), n, bg,
                                          C.c_void_p(out.data_ptr()), out.numel(), _stream(stream)))
        return out, mine

    def render_frame(self, cam, fold_levels=0, cycles=0, background=(0.0, 0.0, 0.0), out=None, stream=None):
        import torch
        self.cam = cam
        self.W, self.H = int(cam.width), int(cam.height)
        if out is None:
            out = torch.empty((self.H, self.W, 4), dtype=torch.float32, device="cuda")
        d = camera_desc(cam)
        hp = C.c_int64()
        bg = (C.c_float * 3)(*background)
        _check(lib().rc_render_frame(self.h, C.byref(d), int(fold_levels), int(cycles), bg,
                                     C.c_void_p(out.data_ptr()), out.numel(), C.byref(hp), _stream(stream)))
        return out, hp.value

    def frame_capture(self, cam, background=(0.0, 0.0, 0.0), out=None, stream=None):
        """CUDA-graph frame (affine forests): one ordinary frame, then the captured copy; returns the image
        tensor the graph writes."""
        import torch
        self.cam = cam
        self.W, self.H = int(cam.width), int(cam.height)
        if out is None:
            out = torch.empty((self.H, self.W, 4), dtype=torch.float32, device="cuda")
        d = camera_desc(cam)
        bg = (C.c_float * 3)(*background)
        _check(lib().rc_frame_capture(self.h, C.byref(d), bg, C.c_void_p(out.data_ptr()), out.numel(), _stream(stream)))
        self._graph_out = out
        return out

    def frame_replay(self, stream=None):
        _check(lib().rc_frame_replay(self.h, _stream(stream)))
        return self._graph_out

    def last_cast_ms(self):
        return float(lib().rc_last_cast_ms(self.h))

    # -- NEXT(4): partner discovery, image instances, vforest -------------
    def exchange_partners(self, tiles_x, tiles_y, nranks, rank, markers, send=True, recv=True):
        """rc_exchange_partners: markers = [(tree, (ax, ay, az))] * (nranks + 1).
        Returns (send_to, recv_from): lists of ranks (None when not asked)."""
        t = Tiling(tiles_x, tiles_y, nranks, rank)
        mk = (Marker * (nranks + 1))()
        for p, (tr, a) in enumerate(markers):
            mk[p].tree = int(tr)
            mk[p].anchor[:] = [int(x) for x in a]
        so = (C.c_uint8 * nranks)()
        ro = (C.c_uint8 * nranks)()
        _check(lib().rc_exchange_partners(self.h, C.byref(t), mk, so if send else None, ro if recv else None))
        return ([q for q in range(nranks) if so[q]] if send else None,
                [p for p in range(nranks) if ro[p]] if recv else None)

    def visible_area_add(self, w, stream=None):
        """w (int64 CUDA tensor [n]) += pixel-centre rectangle area of every leaf in the last cull."""
        _check(lib().rc_visible_area_add(self.h, C.c_void_p(w.data_ptr()), w.numel(), _stream(stream)))
        return w

    def leaves(self, stream=None):
        """rc_forest_leaves: (anchor [n,3] int32, tree int32, level int8, field [n,nf] f32) CUDA tensors."""
        import torch
        nf = 4 if self.surface else (self.P + 1) ** 3
        out = [torch.empty((self.n, 3), dtype=torch.int32, device="cuda"),
               torch.empty(self.n, dtype=torch.int32, device="cuda"),
               torch.empty(self.n, dtype=torch.int8, device="cuda"),
               torch.empty((self.n, nf), dtype=torch.float32, device="cuda")]
        _check(lib().rc_forest_leaves(self.h, *[C.c_void_p(t.data_ptr()) for t in out], self.n, _stream(stream)))
        return out

    def vforest(self, w, first_global_leaf=0, stream=None):
        """rc_vforest_create: (Forest of the leaves with w > 0 or None, count, their weights)."""
        import torch
        h = C.c_void_p()
        cnt = C.c_int64()
        wout = torch.zeros(self.n, dtype=torch.int64, device="cuda")
        _check(lib().rc_vforest_create(self.h, C.c_void_p(w.data_ptr()), int(first_global_leaf), _stream(stream),
                                       C.byref(h), C.byref(cnt), C.c_void_p(wout.data_ptr())))
        if cnt.value == 0:
            return None, 0, wout[:0]
        vf = Forest.__new__(Forest)
        vf.h, vf.n, vf.P, vf.R, vf.surface, vf.cam = h, int(cnt.value), self.P, self.R, self.surface, None
        return vf, int(cnt.value), wout[:cnt.value]

    def last_phase_ms(self, phase):
        return float(lib().rc_last_phase_ms(self.h, int(phase)))


class Comm:
    """rc_comm: librc's NCCL communicator.  Collective over a torch.distributed
    group: rank 0 draws the NCCL id (rc_comm_unique_id), the group broadcasts
    its 128 bytes, every rank calls rc_comm_create on its current device."""

    def __init__(self, nranks, rank, group=None, stream=None):
        import torch
        import torch.distributed as dist
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib().rc_comm_unique_id(C.byref(uid)))
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _check(lib().rc_comm_create(C.byref(uid), int(nranks), int(rank), _stream(stream), C.byref(h)))
        self.h = h
        self.nranks, self.rank = int(nranks), int(rank)

    def set_partners(self, send_to=None, recv_from=None):
        """rc_comm_set_partners: exchanges only between the listed ranks (None: all-to-all)."""
        if send_to is None:
            _check(lib().rc_comm_set_partners(self.h, None, None))
            return
        so = (C.c_uint8 * self.nranks)(*[1 if q in set(send_to) else 0 for q in range(self.nranks)])
        ro = (C.c_uint8 * self.nranks)(*[1 if p in set(recv_from) else 0 for p in range(self.nranks)])
        _check(lib().rc_comm_set_partners(self.h, so, ro))

    def close(self):
        if getattr(self, "h", None):
            lib().rc_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pool_trim() -> None:
    """Return librc's cached device blocks to the driver."""
    _check(lib().rc_pool_trim())


def launch_count(reset=False) -> int:
    return int(lib().rc_launch_count(1 if reset else 0))
