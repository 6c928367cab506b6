"""GPU parity of the surface path (NEXT(3); PAPER.md:780-808 Eq. ABphi,
PAPER.md:1473-1514 App. A.1, PAPER.md:1296-1367 the Mandelbrot hexagon):
k_cull_surface + k_cast_surface through the C ABI against the oracle's
surface render (pinned in tests/test_oracle_surface.py).

Pixels with an eps-ambiguous candidate pair (a ray within 1e-6 of a leaf
edge, where fp32 / fp64 and the half-open convention may assign the point
to either neighbour) are excluded from the element-wise gates and counted."""
import dataclasses
import math

import numpy as np
import pytest

import oracle
import scenegen as sg

pytestmark = pytest.mark.gpu

TOL = 2e-5   # fp32 transfer (powf, expf) on fp64 geometry; |rgba| <= ~1.5


def _gpu_frame(sc, fold=0, cycles=0, bg=(0.0, 0.0, 0.0)):
    import torch
    from paper_1809_01334_b200 import rc
    f = rc.Forest.from_scene(sc)
    img, hits = f.render_frame(sc.camera, fold_levels=fold, cycles=cycles, background=bg)
    torch.cuda.synchronize()
    return f, img.cpu().numpy().reshape(-1, 4), hits


@pytest.mark.parametrize("bend", [0.0, 0.35])
@pytest.mark.parametrize("opaque", [False, True])
def test_mandelbrot_every_pixel(bend, opaque):
    sc = sg.mandelbrot_hexagon(3, 9, width=192, bend=bend, opaque=opaque)
    f, img, hits = _gpu_frame(sc, bg=(0.1, 0.2, 0.3))
    ref = oracle.OracleScene(sc).render(mode="rule", with_hits=False, background=(0.1, 0.2, 0.3))
    clean = ref["namb"] == 0
    err = np.abs(img - ref["rgba"]).max(axis=1)
    print("bend", bend, "opaque", opaque, "hits", hits, ref["total_hits"], "ambiguous pixels", int((~clean).sum()),
          "max err", err[clean].max())
    assert (~clean).sum() <= 0.01 * clean.size
    assert err[clean].max() < TOL
    assert abs(hits - ref["total_hits"]) <= int(ref["namb"].sum())
    hpp = f.segments()["hits_per_pixel"].cpu().numpy().reshape(-1)
    assert np.array_equal(hpp[clean], ref["nhits"][clean])


def test_records_match_oracle_points():
    """Every record is a zero-length point whose (alpha, A, b) equals the
    oracle's for the same (pixel, leaf)."""
    sc = sg.mandelbrot_hexagon(2, 7, width=96, bend=0.5)
    f, img, hits = _gpu_frame(sc)
    raw = f.segments()["raw"].cpu().numpy()
    rec = raw.view(np.float32)
    assert np.all(rec[:, 1] == rec[:, 2])
    o = oracle.OracleScene(sc)
    ref = o.render(mode="rule", with_hits=True, cap=8)
    hits_o = ref["hits"]
    amb = ref["namb"] > 0
    got = {}
    for r, fr in zip(raw, rec):
        got.setdefault((int(r[0]), int(r[7])), []).append((fr[1], fr[3], fr[4], fr[5], fr[6]))
    n_checked = 0
    for p in range(hits_o.shape[0]):
        if amb[p]:
            continue
        for h in hits_o[p]:
            if h["elem"] < 0:
                continue
            g = sorted(got.pop((p, int(h["elem"]))))
            want = (h["alpha_near"], h["a"], *h["b"])
            assert any(np.allclose(x, want, rtol=1e-6, atol=2e-6) for x in g), (p, h, g)
            n_checked += 1
    assert n_checked > 1000


def test_tilted_flat_patch_closed_form():
    """Orthographic rays at 60 degrees to a flat patch: A = A_s^2 exactly
    (cos phi = 1/2), B_c = I_s,c (1 - A), on the GPU."""
    th = math.radians(60.0)
    cam = sg.orthographic_camera([0.5, 0.5, 0.0], [math.sin(th), 0.0, -math.cos(th)], 3.0, 1.2, 32, 32)
    P = np.array([[[[0, 0, 0], [1, 0, 0]], [[0, 1, 0], [1, 1, 0]]]], dtype=np.float64)
    surf = (0.7, -0.4, ((0.2, 0.5, 0.3), (0.1, 0.2, 0.0), (0.6, -0.3, 0.1)), 3.0)
    corners = [0.1, 0.9, 0.4, 0.6]
    sc = sg.Scene("patch", 1, 1, P, np.zeros((1, 3), np.int32), np.zeros(1, np.int32), np.zeros(1, np.int8),
                  np.asarray([corners], np.float32), 0.0, 1.0, 0.0, cam, dim=2, surface=surf)
    _, img, hits = _gpu_frame(sc)
    o = oracle.OracleScene(sc)
    n = 0
    for p in range(32 * 32):
        org, r = o.ray(p % 32, p // 32)
        t = -org[2] / r[2]
        x, y = org[0] + t * r[0], org[1] + t * r[1]
        if not (0.01 < x < 0.99 and 0.01 < y < 0.99):
            continue
        v = (1 - y) * ((1 - x) * corners[0] + x * corners[1]) + y * ((1 - x) * corners[2] + x * corners[3])
        As = min(1.0, max(0.0, 0.7 - 0.4 * v))
        w = math.exp(-0.5 * ((1 - v) * 3.0) ** 2)
        A = As * As
        want = [(surf[2][c][0] + surf[2][c][1] * v + surf[2][c][2] * w) * (1 - A) for c in range(3)] + [1 - A]
        assert np.allclose(img[p], want, atol=3e-6), (p, img[p], want)
        n += 1
    assert n > 100 and hits >= n


@pytest.mark.parametrize("fold,cycles", [(2, 0), (1, 2), (3, 1)])
def test_aggregated_points_same_image(fold, cycles):
    """Aggregation (rows a6/a7) folds zero-length records only where they
    touch; the composite of the aggregated records equals the fold-0 image."""
    sc = sg.mandelbrot_hexagon(3, 8, width=128, bend=0.35)
    _, ref, _ = _gpu_frame(sc)
    _, img, _ = _gpu_frame(sc, fold=fold, cycles=cycles)
    assert np.abs(img - ref).max() < 1e-6


def test_surface_tiles_composite():
    """4 x 4 tiles, one rank: the tile composite assembles the same image."""
    from paper_1809_01334_b200 import dist as rdist
    from paper_1809_01334_b200 import rc
    sc = sg.mandelbrot_hexagon(3, 8, width=128, opaque=True)
    _, ref, _ = _gpu_frame(sc)
    f = rc.Forest.from_scene(sc)
    f.camera_set(sc.camera)
    f.cull()
    f.cast_segments(0)
    out, mine = f.composite_tiles(4, 4, 1, 0)
    img = rdist.assemble_image({0: (out, mine)}, 4, 4, 128, 128).numpy().reshape(-1, 4)
    assert np.array_equal(img.view(np.uint32), ref.view(np.uint32))


def test_full_size_sampled():
    """The bench workload (MB: levels 3..11, 2048^2, bent): sampled pixels
    against the oracle, and hits per pixel on every clean sampled pixel."""
    import bench
    sc = bench.make_scene(6, "cpu")
    f, img, hits = _gpu_frame(sc)
    rng = np.random.default_rng(6)
    W = sc.camera.width
    pix = np.sort(rng.choice(W * W, 20000, replace=False)).astype(np.int32)
    ref = oracle.OracleScene(sc).render_pairs(pixels=pix, mode="rule")
    cnt = np.diff(ref["pair_off"])
    flagged = np.zeros(pix.size, dtype=bool)
    flagged[np.repeat(np.arange(pix.size), cnt)[(ref["pair_flags"] & oracle.AMBIGUOUS) != 0]] = True
    clean = ~flagged
    err = np.abs(img[pix] - ref["rgba"]).max(axis=1)
    print("MB full: hits", hits, "sampled clean", int(clean.sum()), "max err", err[clean].max())
    assert err[clean].max() < TOL
    assert clean.sum() > 0.99 * pix.size
