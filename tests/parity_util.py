"""Helpers of the GPU-vs-oracle parity tests (SURVEY §8(c) gates 1-3)."""
import numpy as np

import oracle


def gpu_run(scene, background=(0.0, 0.0, 0.0), device_copy=False, fold=0, cycles=0, keep_raw=True):
    import torch
    from paper_1809_01334_b200 import rc
    f = rc.Forest.from_scene(scene, device_copy=device_copy)
    f.camera_set(scene.camera)
    f.cull()
    vis = f.cull_result().cpu().numpy()
    f.cast_segments(fold)
    if cycles:
        f.aggregate(cycles)
    segs = f.segments()
    raw = segs["raw"].cpu().numpy().copy() if keep_raw else None
    hpp = segs["hits_per_pixel"].cpu().numpy().copy()
    img = f.composite(background).cpu().numpy().copy()
    torch.cuda.synchronize()
    out = dict(visible=vis, raw=raw, hits_per_pixel=hpp, rgba=img.reshape(-1, 4), count=segs["count"],
               candidates=segs["candidates"], hit_pairs=segs["hit_pairs"], newton_failures=segs["newton_failures"],
               face_failures=segs["face_failures"], raw_segments=segs["raw_segments"], level=segs["level"],
               units=segs["units"], unfolded_units=segs["unfolded_units"], forest=f)
    return out


def seg_columns(raw):
    f = raw.view(np.float32)
    return dict(pixel=raw[:, 0].astype(np.int64), alpha_near=f[:, 1], alpha_far=f[:, 2], a=f[:, 3], b=f[:, 4:7],
                key=raw[:, 7].astype(np.int64))


def compare(scene, g, ores, pixels, cull=None, tol=1e-4, by_counts=False):
    """Return a report dict with the three gates evaluated on `pixels`.
    by_counts: records are folded (node keys), so gate 2 compares the
    per-pixel hit counts (rc_segments.hits_per_pixel) with the oracle's:
    non-ambiguous hits <= count <= non-ambiguous hits + ambiguous pairs."""
    rep = {}
    # gate 1: culled list
    if cull is not None:
        vis_o, amb_o, _ = cull
        so = set(np.nonzero(vis_o & ~amb_o)[0].tolist())
        sg_ = set(g["visible"].tolist()) - set(np.nonzero(amb_o)[0].tolist())
        rep["cull_mismatch"] = len(so ^ sg_)
        rep["cull_ambiguous"] = int(amb_o.sum())
    if not by_counts:
        cols = seg_columns(g["raw"])
        order = np.argsort(cols["pixel"], kind="stable")
        pix_sorted = cols["pixel"][order]
        keys_sorted = cols["key"][order]
        lo = np.searchsorted(pix_sorted, pixels, side="left")
        hi = np.searchsorted(pix_sorted, pixels, side="right")
    hit_mismatch, amb_pairs, amb_pixels, bad_pix, bad_amb_pix = 0, 0, 0, 0, 0
    maxerr, maxerr_amb = 0.0, 0.0
    for q, p in enumerate(pixels):
        h = ores["hits"][q]
        h = h[h["elem"] >= 0]
        amb = set(h["elem"][(h["flags"] & oracle.AMBIGUOUS) != 0].tolist())
        ohit = set(h["elem"][(h["flags"] & oracle.HIT) != 0].tolist()) - amb
        if by_counts:
            c = int(g["hits_per_pixel"].reshape(-1)[p])
            if not (len(ohit) <= c <= len(ohit) + len(amb)):
                hit_mismatch += 1
        else:
            ghit = set(keys_sorted[lo[q]:hi[q]].tolist()) - amb
            if ohit != ghit:
                hit_mismatch += 1
        amb_pairs += len(amb)
        err = float(np.abs(g["rgba"][p] - ores["rgba"][q]).max())
        if amb:
            amb_pixels += 1
            maxerr_amb = max(maxerr_amb, err)
            bad_amb_pix += err > tol
        else:
            maxerr = max(maxerr, err)
            bad_pix += err > tol
    rep.update(hit_mismatch_pixels=hit_mismatch, ambiguous_pairs=amb_pairs, ambiguous_pixels=amb_pixels,
               max_err=maxerr, bad_pixels=bad_pix, max_err_ambiguous_pixels=maxerr_amb,
               bad_ambiguous_pixels=bad_amb_pix)
    return rep


# ---------------------------------------------------------------------------
# Vectorised gates (every pixel of C2/C3, 1/256 .. 1/2304 samples of C4/C5)
# ---------------------------------------------------------------------------
def stride_pixels(W, H, s, off=None):
    """Every s-th pixel row and column (stratified sample)."""
    o = s // 2 if off is None else off
    jj, ii = np.meshgrid(np.arange(o, H, s), np.arange(o, W, s), indexing="ij")
    return (jj * W + ii).ravel().astype(np.int32)


def gpu_pairs(raw, pixels, npix_image, key_offset=0):
    """Unique (pixel, leaf) pairs of fold-0 records (leaf keys) restricted to
    `pixels`, as int64 keys pixel << 32 | leaf.  raw: int32 [n, 8] tensor on
    the device (filtered there) or numpy."""
    import torch
    if isinstance(raw, torch.Tensor):
        mask = torch.zeros(npix_image, dtype=torch.bool, device=raw.device)
        mask[torch.as_tensor(pixels, dtype=torch.int64, device=raw.device)] = True
        pix = raw[:, 0].to(torch.int64)
        sel = mask[pix]
        pk = (pix[sel] << 32) | (raw[sel, 7].to(torch.int64) & 0xFFFFFFFF) + key_offset
        return torch.unique(pk).cpu().numpy()
    pix = raw[:, 0].astype(np.int64)
    sel = np.zeros(npix_image, dtype=bool)
    sel[pixels] = True
    m = sel[pix]
    return np.unique((pix[m] << 32) | ((raw[m, 7].astype(np.int64) & 0xFFFFFFFF) + key_offset))


def oracle_pairs(ores):
    """From OracleScene.render_pairs: (non-ambiguous hit pair keys, ambiguous
    pair keys), each pixel << 32 | leaf."""
    import oracle
    cnt = np.diff(ores["pair_off"])
    pix = np.repeat(ores["pixels"].astype(np.int64), cnt)
    key = (pix << 32) | ores["pair_elem"].astype(np.int64)
    fl = ores["pair_flags"]
    amb = (fl & oracle.AMBIGUOUS) != 0
    hit = ((fl & oracle.HIT) != 0) & ~amb
    return np.unique(key[hit]), np.unique(key[amb])


def gate_pairs(gkeys, okeys, akeys):
    """Gate 2: GPU hit pairs minus eps-ambiguous pairs == the oracle's
    non-ambiguous hit pairs.  Returns (mismatching pairs, mismatching pixels)."""
    g = np.setdiff1d(gkeys, akeys, assume_unique=True)
    diff = np.setxor1d(g, okeys, assume_unique=True)
    return int(diff.size), int(np.unique(diff >> 32).size)


def gate_cull(gvis_idx, ovis, oamb):
    """Gate 1: culled-list set equality after removing ambiguous leaves."""
    g = np.zeros(ovis.shape[0], dtype=bool)
    g[np.asarray(gvis_idx, dtype=np.int64)] = True
    return int(np.count_nonzero((g ^ ovis) & ~oamb))


def gate_rgba(g_rgba, pixels, ores, tol=1e-4):
    """Gate 3 on the pixels without eps-ambiguous pairs; the ambiguous ones
    are reported separately.  g_rgba: [H*W, 4] numpy."""
    err = np.abs(g_rgba[pixels] - ores["rgba"]).max(axis=1)
    clean = ores["namb"] == 0
    return dict(max_err=float(err[clean].max(initial=0.0)), bad_pixels=int(np.count_nonzero(err[clean] > tol)),
                max_err_ambiguous=float(err[~clean].max(initial=0.0)), ambiguous_pixels=int(np.count_nonzero(~clean)))


def gpu_fold0_chunked(scene, pixels, nchunks, device_copy=False):
    """Fold-0 cast of `scene` split into `nchunks` contiguous SFC ranges (one
    forest at a time, as the ranks of a multi-GPU run hold them): the visible
    leaves (global indices), the unique (pixel, leaf) hit pairs at `pixels`
    and the per-pixel hit counts of the whole image."""
    import torch
    from paper_1809_01334_b200 import rc
    n = scene.num_leaves
    W, H = scene.camera.width, scene.camera.height
    cuts = [n * k // nchunks for k in range(nchunks + 1)]
    vis, keys = [], []
    hpp = torch.zeros(H * W, dtype=torch.int64, device="cuda")
    stats = dict(hit_pairs=0, candidates=0, newton_failures=0, records=0)
    for lo, hi in zip(cuts, cuts[1:]):
        f = rc.Forest.from_scene(scene, first=lo, count=hi - lo, device_copy=device_copy)
        f.camera_set(scene.camera)
        f.cull()
        vis.append(f.cull_result().cpu().numpy().astype(np.int64) + lo)
        f.cast_segments(0)
        s = f.segments()
        keys.append(gpu_pairs(s["raw"], pixels, H * W))
        hpp += s["hits_per_pixel"].reshape(-1).to(torch.int64)
        for k in ("hit_pairs", "candidates", "newton_failures"):
            stats[k] += int(s[k])
        stats["records"] += int(s["count"])
        f.close()
        del f, s
        rc.pool_trim()
        torch.cuda.empty_cache()
    return dict(visible=np.concatenate(vis), keys=np.unique(np.concatenate(keys)),
                hits_per_pixel=hpp.cpu().numpy(), **stats)


def linear_field_shell(base, cvec, d0):
    """The scene `base` (R = 2 shell) with P = 2 nodal values of the world-linear
    field f(x) = cvec.x + d0 at every element's GLL nodes, mapped through the
    tree's R = 2 Lagrange map J_k (textbook Lagrange basis on {0, 1/2, 1}
    evaluated here, not the oracle's or the GPU's code): f o X_E is then
    triquadratic and the nodal interpolation exact (pin P16).  inv_F = 1."""
    import dataclasses
    ctrl = np.asarray(base.tree_ctrl)                 # [K][3][3][3][3], [k][m3][m2][m1][xyz]
    g = np.array([0.0, 0.5, 1.0])

    def lag(t):
        return np.array([(t - g[1]) * (t - g[2]) / ((g[0] - g[1]) * (g[0] - g[2])),
                         (t - g[0]) * (t - g[2]) / ((g[1] - g[0]) * (g[1] - g[2])),
                         (t - g[0]) * (t - g[1]) / ((g[2] - g[0]) * (g[2] - g[1]))])

    anc = np.asarray(base.leaf_anchor, np.float64) / (1 << 18)
    hE = np.ldexp(1.0, -np.asarray(base.leaf_level, np.int64))
    fld = np.zeros((base.num_leaves, 27), np.float32)
    for e in range(base.num_leaves):
        C = ctrl[int(base.leaf_tree[e])]
        for k3 in range(3):
            for k2 in range(3):
                for k1 in range(3):
                    t = anc[e] + hE[e] * g[[k1, k2, k3]]
                    x = np.einsum("a,b,c,abcx->x", lag(t[2]), lag(t[1]), lag(t[0]), C)
                    fld[e, (k3 * 3 + k2) * 3 + k1] = np.asarray(cvec) @ x + d0
    return dataclasses.replace(base, leaf_field=fld, inv_F=1.0)


def linear_field_segment(ro, rd, an, af, cvec, d0, kappa0):
    """Closed-form A and quadrature B of one segment [an, af] of the ray
    ro + alpha rd in the world-linear field (kappa = kappa0 f^2, q = ((1+f)/2,
    (1-f)/2, 1/2)); s measured from the near end (Eq. ABgeneral)."""
    import math
    from numpy.polynomial import polynomial as Pn
    from scipy.integrate import quad
    nr = float(np.linalg.norm(rd))
    fa = np.array([np.dot(cvec, ro) + d0, np.dot(cvec, rd)])
    ik = Pn.polyint(kappa0 * Pn.polymul(fa, fa) * nr)
    A = math.exp(-(Pn.polyval(af, ik) - Pn.polyval(an, ik)))
    B = []
    for c in range(3):
        def qf(a_, c=c):
            f = fa[0] + fa[1] * a_
            return ((1 + f) / 2, (1 - f) / 2, 0.5)[c] * math.exp(-(Pn.polyval(a_, ik) - Pn.polyval(an, ik))) * nr
        B.append(quad(qf, an, af, epsabs=1e-14, epsrel=1e-12)[0])
    return A, np.array(B)

