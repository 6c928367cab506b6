"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same
seeded inputs (SURVEY §8(c) gates: culled list and per-pixel hit sets
bit-exact after removing eps-ambiguous pairs; RGBA within 1e-4 absolute)."""
import math

import numpy as np
import pytest

import oracle
import scenegen as sg
from parity_util import (compare, gate_cull, gate_pairs, gate_rgba, gpu_fold0_chunked, gpu_pairs, gpu_run,
                         oracle_pairs, seg_columns, stride_pixels)

pytestmark = pytest.mark.gpu

TOL = 1e-4   # BASELINE.json north_star: pixels within 1e-4 absolute


def _check(rep):
    assert rep.get("cull_mismatch", 0) == 0, rep
    assert rep["hit_mismatch_pixels"] == 0, rep
    assert rep["bad_pixels"] == 0, rep


def _full(scene, mode="exact"):
    o = oracle.OracleScene(scene)
    pixels = np.arange(scene.camera.width * scene.camera.height, dtype=np.int32)
    ores = o.render(pixels, mode=mode, cap=128)
    return o, pixels, ores


def test_c1_full_frame():
    sc = sg.config1()
    o, pixels, ores = _full(sc)
    g = gpu_run(sc)
    rep = compare(sc, g, ores, pixels, cull=o.cull())
    _check(rep)
    assert g["hit_pairs"] == 15412 and g["count"] == 15412
    assert g["candidates"] >= 15412
    # hits per pixel equal the oracle's non-ambiguous counts
    assert rep["ambiguous_pairs"] == 8
    # diagnostic: GPU vs oracle rule mode, implementation error only
    orule = o.render(pixels, mode="rule", cap=128, with_hits=False)
    assert np.abs(g["rgba"] - orule["rgba"]).max() < 2e-5


def test_c2_small_full_frame():
    sc = sg.config2(width=96, maxlevel=5)
    o, pixels, ores = _full(sc)
    g = gpu_run(sc)
    _check(compare(sc, g, ores, pixels, cull=o.cull()))


def _gates_full(sc, g, ores, pixels):
    """Gates 1-3 (vectorised) of a fold-0 GPU run against render_pairs."""
    W, H = sc.camera.width, sc.camera.height
    okeys, akeys = oracle_pairs(ores)
    gkeys = gpu_pairs(g["raw"], pixels, W * H)
    nbad, nbadpix = gate_pairs(gkeys, okeys, akeys)
    rep = dict(cull_mismatch=gate_cull(g["visible"], ores["visible"], ores["ambiguous"]),
               cull_ambiguous=int(ores["ambiguous"].sum()), pair_mismatch=nbad, hit_mismatch_pixels=nbadpix,
               ambiguous_pairs=int(akeys.size), pixels=int(pixels.size), oracle_hits=int(okeys.size))
    rep.update(gate_rgba(g["rgba"], pixels, ores))
    return rep


def test_c2_full_size_every_pixel():
    """BASELINE C2 at its full size (87,088 leaves, 512^2) in the bench's launch
    configuration: gates 1-3 on every pixel."""
    sc = sg.config2()
    o = oracle.OracleScene(sc)
    pixels = np.arange(sc.camera.width * sc.camera.height, dtype=np.int32)
    ores = o.render_pairs(pixels, mode="exact")
    g = gpu_run(sc)
    rep = _gates_full(sc, g, ores, pixels)
    print(rep)
    _check(rep)
    assert rep["pair_mismatch"] == 0
    # full-frame properties: alpha order, transmission range, hit counts
    cols = seg_columns(g["raw"])
    assert np.all(cols["alpha_near"] <= cols["alpha_far"])   # equal only for sub-ulp chords
    assert np.all((cols["a"] > 0) & (cols["a"] <= 1))
    assert g["hits_per_pixel"].sum() == g["hit_pairs"]


def test_constant_medium_closed_form_gpu():
    """P8 on the GPU: f == const -> every pixel is Eq. ABconstant over the
    chord of the ray through the unit cube (independent slab test here)."""
    sc = sg.constant_field(sg.config2(width=64, maxlevel=5), 0.6)
    g = gpu_run(sc)
    o = oracle.OracleScene(sc)
    ft = float(np.float32(0.6))
    kap = 5.0 * ft * ft
    q = np.array([(1 + ft) / 2, (1 - ft) / 2, 0.5])
    W = sc.camera.width
    worst = 0.0
    for p in range(W * W):
        ro, rd = o.ray(p % W, p // W)
        t0, t1 = 1.0, 100.0
        for k in range(3):
            a, b = (0 - ro[k]) / rd[k], (1 - ro[k]) / rd[k]
            t0, t1 = max(t0, min(a, b)), min(t1, max(a, b))
        L = max(0.0, t1 - t0) * np.linalg.norm(rd)
        A = math.exp(-kap * L)
        ref = np.r_[q * (1 - A) / kap, 1 - A]
        worst = max(worst, float(np.abs(g["rgba"][p] - ref).max()))
    assert worst < TOL


def test_empty_and_single_leaf():
    import dataclasses
    sc = sg.config1(width=32)
    # camera looking away from the cube: nothing visible
    cam = sg.perspective_camera([3.0, 3.0, 3.0], [6.0, 6.0, 6.0], 30.0, 32, 32)
    g = gpu_run(dataclasses.replace(sc, camera=cam))
    assert g["visible"].size == 0 and g["count"] == 0
    assert np.all(g["rgba"][:, 3] == 0)
    # a single leaf (level 0 = the whole tree)
    one = dataclasses.replace(sc, leaf_anchor=np.zeros((1, 3), np.int32), leaf_tree=np.zeros(1, np.int32),
                              leaf_level=np.zeros(1, np.int8), leaf_field=sc.leaf_field[:1].copy())
    o, pixels, ores = _full(one)
    g = gpu_run(one)
    _check(compare(one, g, ores, pixels, cull=o.cull()))


def test_device_copy_and_background():
    """RC_DEVICE_COPY input path and a non-zero background I_b."""
    sc = sg.config1(width=40)
    bg = (0.2, 0.5, 0.9)
    o = oracle.OracleScene(sc)
    pixels = np.arange(40 * 40, dtype=np.int32)
    ores = o.render(pixels, mode="exact", cap=64, background=bg)
    g = gpu_run(sc, background=bg, device_copy=True)
    _check(compare(sc, g, ores, pixels))


def test_errors_are_loud():
    from paper_1809_01334_b200 import rc
    sc = sg.config1(width=16)
    with pytest.raises(rc.RcError) as ei:
        bad = sc.leaf_anchor[::-1].copy()
        rc.Forest(sc.tree_ctrl, 1, 1, bad, sc.leaf_tree, sc.leaf_level, sc.leaf_field, 5, 1, 1)
    assert "SFC" in str(ei.value)
    f = rc.Forest.from_scene(sc)
    with pytest.raises(rc.RcError):
        f.cull()      # before camera_set -> RC_ERR_STATE


# ---------------------------------------------------------------------------
# Curved R=2 geometry (cubed-sphere shell, configs C3-C5)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("level,width,nb", [(1, 48, 8), (2, 64, 16), (3, 96, 16)])
def test_shell_full_frame(level, width, nb):
    sc = sg.shell_uniform(level, width, nb, gl_points=6)
    o, pixels, ores = _full(sc)
    g = gpu_run(sc)
    rep = compare(sc, g, ores, pixels, cull=o.cull())
    print(rep, "newton_failures", g["newton_failures"])
    _check(rep)
    assert g["newton_failures"] == 0


def test_shell_gl8_field_p2():
    """N = 8 GL points (C5's rule) on a level-2 shell."""
    sc = sg.shell_uniform(2, 56, 32, gl_points=8)
    o, pixels, ores = _full(sc)
    g = gpu_run(sc)
    _check(compare(sc, g, ores, pixels, cull=o.cull()))


def test_c3_reduced_every_pixel():
    """C3's geometry, field and rule at reduced size (level-4 shell, 24,576
    curved hexes, 256^2, 64 bumps, N = 6): gates 1-3 on every pixel."""
    sc = sg.shell_uniform(4, 256, 64, gl_points=6, name="C3-L4")
    o = oracle.OracleScene(sc)
    pixels = np.arange(256 * 256, dtype=np.int32)
    ores = o.render_pairs(pixels, mode="exact")
    g = gpu_run(sc)
    rep = _gates_full(sc, g, ores, pixels)
    print(rep, "newton_failures", g["newton_failures"])
    _check(rep)
    assert rep["pair_mismatch"] == 0 and g["newton_failures"] == 0


def test_c3_full_size_sampled():
    """BASELINE C3 at full size (1,572,864 curved hexes, 1024^2, N=6): gates 1-3
    on every 4th pixel row and column (65,536 pixels; the oracle intersects
    ~3e4 pairs/s per core, every pixel would take ~1 h on the box), all leaves
    culled by the oracle; then the bench's configuration (fold level 2) against
    the same oracle values and the fold-0 run."""
    sc = sg.config3(device="cuda")
    W = sc.camera.width
    pixels = stride_pixels(W, W, 4, off=1)
    g = gpu_run(sc, device_copy=True)
    g2 = gpu_run(sc, device_copy=True, fold=2, keep_raw=False)    # bench.py's launch configuration
    import bench
    o = oracle.OracleScene(bench.scene_to_host(sc))
    ores = o.render_pairs(pixels, mode="exact")
    rep = _gates_full(sc, g, ores, pixels)
    print(rep, "hit_pairs", g["hit_pairs"], "newton_failures", g["newton_failures"])
    _check(rep)
    assert rep["pair_mismatch"] == 0 and g["newton_failures"] == 0
    rep2 = gate_rgba(g2["rgba"], pixels, ores)
    print(rep2, "records", g2["count"], "raw", g2["raw_segments"], "units", g2["units"])
    assert rep2["bad_pixels"] == 0, rep2
    assert np.array_equal(g2["hits_per_pixel"], g["hits_per_pixel"])
    assert g2["raw_segments"] == g["count"] and g2["count"] < g["count"] // 2
    assert np.abs(g2["rgba"] - g["rgba"]).max() < 1e-5


def test_affine_r2_matches_r1_P9():
    """R=2 tree with affine (identity) control points goes through the same
    slab path and reproduces the R=1 result."""
    import dataclasses
    sc1 = sg.config2(width=64, maxlevel=5)
    sc2 = dataclasses.replace(sc1, geom_degree=2, tree_ctrl=sg.identity_cube_ctrl(2))
    g1, g2 = gpu_run(sc1), gpu_run(sc2)
    assert g1["count"] == g2["count"]
    assert np.abs(g1["rgba"] - g2["rgba"]).max() < 1e-6


@pytest.mark.parametrize("which,nranks", [("c2", 2), ("c2", 3), ("shell", 4)])
def test_virtual_ranks_tile_exchange(which, nranks):
    """Multi-GPU path on one GPU: P forests over contiguous SFC
    ranges, rc_pack_tiles by tile owner, the per-owner concatenation stands in
    for the NCCL all-to-all, rc_composite_tiles per owner.  Equals the
    single-forest image (partition invariance)."""
    import torch
    from paper_1809_01334_b200 import dist as rdist
    from paper_1809_01334_b200 import rc
    sc = sg.config2(width=96, maxlevel=5) if which == "c2" else sg.shell_uniform(3, 96, 16, gl_points=6)
    tiles = (4, 4)
    full = gpu_run(sc)["rgba"].reshape(96, 96, 4)
    ranges = rdist.weighted_ranges(torch.ones(sc.num_leaves), nranks)
    forests, packed = [], []
    for lo, hi in ranges:
        f = rc.Forest.from_scene(sc, first=lo, count=hi - lo)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments()
        raw, counts = f.pack_tiles(*tiles, nranks, 0)
        offs = np.r_[0, np.cumsum(counts)]
        packed.append([raw[offs[d]:offs[d + 1]].clone() for d in range(nranks)])
        forests.append(f)
    out = {}
    for d in range(nranks):
        recv = torch.cat([packed[s][d] for s in range(nranks)])
        img, mine = forests[d].composite_tiles(*tiles, nranks, d, recv=recv)
        out[d] = (img, mine)
    merged = rdist.assemble_image(out, *tiles, 96, 96).numpy()
    assert np.abs(merged - full).max() < 1e-6


@pytest.mark.parametrize("nranks", [2, 4])
def test_virtual_ranks_fold_aggregate_aligned(nranks):
    """The bench's multi-GPU configuration on one GPU: family-aligned SFC
    ranges (dist.node_starts / aligned_ranges at fold + cycles levels), the
    on-chip fold at level 2 and one aggregation cycle per rank, records packed
    by tile owner and composited by the owner; equals the single-forest image
    up to the fp32 records (lossless folds)."""
    import torch
    from paper_1809_01334_b200 import dist as rdist
    from paper_1809_01334_b200 import rc
    sc = sg.shell_uniform(3, 96, 16, gl_points=6)
    tiles = (4, 4)
    full = gpu_run(sc)["rgba"].reshape(96, 96, 4)
    A, T, L = (torch.as_tensor(x) for x in (sc.leaf_anchor, sc.leaf_tree, sc.leaf_level))
    allowed = rdist.node_starts(A, T, L, 3)
    ranges = rdist.aligned_ranges(torch.ones(sc.num_leaves, dtype=torch.float64), nranks, allowed)
    assert all(lo == 0 or bool(allowed[lo]) for lo, hi in ranges if lo < sc.num_leaves)
    forests, packed = [], []
    for lo, hi in ranges:
        f = rc.Forest.from_scene(sc, first=lo, count=hi - lo)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(2)
        f.aggregate(1)
        raw, counts = f.pack_tiles(*tiles, nranks, 0)
        offs = np.r_[0, np.cumsum(counts)]
        packed.append([raw[offs[d]:offs[d + 1]].clone() for d in range(nranks)])
        forests.append(f)
    out = {}
    for d in range(nranks):
        recv = torch.cat([packed[s][d] for s in range(nranks)])
        img, mine = forests[d].composite_tiles(*tiles, nranks, d, recv=recv)
        out[d] = (img, mine)
    merged = rdist.assemble_image(out, *tiles, 96, 96).numpy()
    assert np.abs(merged - full).max() < 1e-5


def _big_config_gates(sc, pixels, nchunks, fold, cycles):
    """Full-size C4 / C5: fold-0 casts of SFC chunks (gate 1 on the full culled
    list, gate 2 on the hit pairs of the sampled pixels), then the bench's
    launch configuration for gate 3 and the per-pixel hit counts."""
    import torch
    import bench
    from paper_1809_01334_b200 import rc
    W, H = sc.camera.width, sc.camera.height
    ch = gpu_fold0_chunked(sc, pixels, nchunks, device_copy=isinstance(sc.leaf_anchor, torch.Tensor))
    assert ch["newton_failures"] == 0
    g = gpu_run(sc, device_copy=isinstance(sc.leaf_anchor, torch.Tensor), fold=fold, cycles=cycles, keep_raw=False)
    assert g["newton_failures"] == 0
    # the SFC chunks and the single forest see the same hits per pixel
    assert np.array_equal(ch["hits_per_pixel"], g["hits_per_pixel"].reshape(-1).astype(np.int64))
    assert ch["hit_pairs"] == g["hit_pairs"]
    host = bench.scene_to_host(sc)
    del sc
    g.pop("forest").close()
    rc.pool_trim()
    torch.cuda.empty_cache()
    o = oracle.OracleScene(host)
    ores = o.render_pairs(pixels, mode="exact")
    okeys, akeys = oracle_pairs(ores)
    nbad, nbadpix = gate_pairs(ch["keys"], okeys, akeys)
    rep = dict(cull_mismatch=gate_cull(ch["visible"], ores["visible"], ores["ambiguous"]),
               cull_ambiguous=int(ores["ambiguous"].sum()), pair_mismatch=nbad, hit_mismatch_pixels=nbadpix,
               ambiguous_pairs=int(akeys.size), pixels=int(pixels.size), oracle_hit_pairs=int(okeys.size),
               leaves=int(host.num_leaves), hit_pairs=g["hit_pairs"], records=g["count"])
    rep.update(gate_rgba(g["rgba"], pixels, ores))
    return rep


def test_c4_full_size_sampled():
    """BASELINE C4 at full size on one GPU (100,663,296 curved hexes, 2048^2,
    N = 6): culled list in full; hit pairs and pixels on every 16th pixel row
    and column (16,384 pixels, SURVEY §8(d)'s 1/256 sample); pixel values in
    the bench's launch configuration (fold level 2)."""
    from paper_1809_01334_b200 import rc
    rc.pool_trim()
    sc = sg.config4(device="cuda")
    pixels = stride_pixels(sc.camera.width, sc.camera.height, 16, off=5)
    rep = _big_config_gates(sc, pixels, nchunks=4, fold=2, cycles=0)
    print(rep)
    _check(rep)
    assert rep["pair_mismatch"] == 0


def test_c5_full_size_sampled():
    """BASELINE C5 at full size on one GPU (~1.97e8 curved hexes on levels
    6..10, 4096^2, N = 8): culled list in full; hit pairs and pixels on every
    48th pixel row and column (7,225 pixels); pixel values in the bench's
    launch configuration (fold 2 + 3 aggregation cycles)."""
    import torch
    import bench
    from paper_1809_01334_b200 import rc
    rc.pool_trim()   # earlier tests' cached blocks back to the driver (the generator needs them)
    sc = bench.scene_to_host(sg.config5(device="cuda"))   # generated on the GPU, kept on the host
    torch.cuda.empty_cache()
    pixels = stride_pixels(sc.camera.width, sc.camera.height, 48, off=13)
    rep = _big_config_gates(sc, pixels, nchunks=8, fold=2, cycles=3)
    print(rep)
    _check(rep)
    assert rep["pair_mismatch"] == 0


@pytest.mark.gpu
def test_composite_tilings_on_one_forest():
    """rc_composite_tiles keeps the owner's tile list on the device across calls
    (re-uploaded when the tiling changes): composites of one forest's own records
    under several tilings / ranks, in sequence, each equal the full composite."""
    import torch
    from paper_1809_01334_b200 import dist as rdist
    from paper_1809_01334_b200 import rc
    sc = sg.shell_uniform(3, 96, 16, gl_points=6)
    f = rc.Forest.from_scene(sc)
    f.camera_set(sc.camera)
    f.cull()
    f.cast_segments(2)
    full = f.composite().cpu().numpy()
    for tiles, nranks in (((4, 4), 2), ((2, 3), 3), ((4, 4), 2), ((1, 1), 1)):
        out = {}
        for d in range(nranks):
            img, mine = f.composite_tiles(*tiles, nranks, d)
            out[d] = (img.clone(), mine)
        merged = rdist.assemble_image(out, *tiles, 96, 96).numpy()
        assert np.abs(merged - full).max() < 1e-6, (tiles, nranks)


def test_curved_linear_field_pairs_closed_form():
    """The GPU's per-pair (a, b) on curved R=2 elements with a non-constant
    field against the closed form of pin P16 (independent of the oracle):
    f linear in world coordinates is exactly triquadratic on every element, so
    along a ray A = exp(-int kappa) is a polynomial integral and B a scipy
    quadrature; the N = 6 GL rule is exact for the quadratic kappa.  Every
    fold-0 record of the frame, on the ray of Eq. ray written out here.
    Tolerance 2e-5: fp32 arithmetic and the 1e-6 inverse-map tolerance."""
    from parity_util import linear_field_segment, linear_field_shell
    cvec, d0 = np.array([0.21, 0.11, -0.17]), 0.05
    sc = linear_field_shell(sg.shell_uniform(2, 48, 4, gl_points=6), cvec, d0)
    g = gpu_run(sc)
    cam = sc.camera
    assert cam.projection == 0
    rec = seg_columns(g["raw"])
    kap0 = float(np.float32(sc.kappa0))
    W, H = cam.width, cam.height
    n = rec["pixel"].size
    assert n > 1000
    idx = np.random.default_rng(0).choice(n, size=min(n, 3000), replace=False)
    worst_a = worst_b = 0.0
    for k in idx:
        p = int(rec["pixel"][k])
        i, j = p % W, p // W
        rd = np.asarray(cam.view) + cam.pixel_size * ((i - (W - 1) / 2) * np.asarray(cam.right) +
                                                      (j - (H - 1) / 2) * np.asarray(cam.up))
        an, af = float(rec["alpha_near"][k]), float(rec["alpha_far"][k])
        A, B = linear_field_segment(np.asarray(cam.origin, np.float64), rd, an, af, cvec, d0, kap0)
        worst_a = max(worst_a, abs(float(rec["a"][k]) - A))
        worst_b = max(worst_b, float(np.abs(rec["b"][k] - B).max()))
    print("records", n, "max |a - A|", worst_a, "max |b - B|", worst_b)
    assert worst_a < 2e-5 and worst_b < 2e-5, (worst_a, worst_b)
