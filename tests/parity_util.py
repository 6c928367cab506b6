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
