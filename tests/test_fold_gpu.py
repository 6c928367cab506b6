"""GPU tests of rows a6 (on-chip fold in the segment kernel) and a7
(rc_aggregate coarsening cycles): PAPER.md:956-994, SURVEY §8(c) R22.

The fold and the aggregation reorganise the segments only: the pixels must
equal the unfolded result up to roundoff ("lossless"; SURVEY
R22: <= 1e-6 in fp64 folds, 1e-5 with fp32 records) and the oracle within
the 1e-4 gate, the per-pixel hit counts must not change, and the record
count must fall with every level.  The node tables are checked against an
independent host implementation of the coarsening rule."""
import numpy as np
import pytest

import oracle
import scenegen as sg
from oracle import coarsen
from parity_util import compare, gpu_run

pytestmark = pytest.mark.gpu

LOSSLESS = 1e-5


nodes_reference = coarsen.node_tables


def _record_counts(g, npix):
    return np.bincount(g["raw"][:, 0].astype(np.int64), minlength=npix)


def _oracle_runs(ores, table):
    """Per pixel: oracle run count at the table's level, or -1 for pixels
    with eps-ambiguous pairs (excluded from the exact comparison)."""
    out = np.zeros(len(ores["pixels"]), dtype=np.int64)
    for q in range(len(ores["pixels"])):
        h = ores["hits"][q]
        h = h[h["elem"] >= 0]
        if ((h["flags"] & oracle.AMBIGUOUS) != 0).any():
            out[q] = -1
        else:
            out[q] = coarsen.run_counts(h, table)
    return out


@pytest.mark.parametrize("which", ["c2", "shell"])
def test_node_tables_match_reference(which):
    from paper_1809_01334_b200 import rc
    sc = sg.config2(width=64, maxlevel=5) if which == "c2" else sg.shell_uniform(2, 48, 8, gl_points=6)
    f = rc.Forest.from_scene(sc)
    ref = nodes_reference(sc.leaf_anchor, sc.leaf_tree, sc.leaf_level, 4)
    for c in range(1, 5):
        got = f.node_table(c).cpu().numpy()
        assert np.array_equal(got, ref[c]), (c, got[:20], ref[c][:20])
    # a range that splits families: only complete local families coarsen
    lo, hi = 3, sc.num_leaves - 5
    f2 = rc.Forest.from_scene(sc, first=lo, count=hi - lo)
    ref2 = nodes_reference(sc.leaf_anchor[lo:hi], sc.leaf_tree[lo:hi], sc.leaf_level[lo:hi], 2)
    for c in (1, 2):
        assert np.array_equal(f2.node_table(c).cpu().numpy(), ref2[c])


@pytest.mark.parametrize("level,width", [(2, 64), (3, 96)])
def test_fold_levels_curved(level, width):
    """Fused fold (a6) at levels 1-3 on the curved path."""
    sc = sg.shell_uniform(level, width, 16, gl_points=6)
    g0 = gpu_run(sc, fold=0)
    assert g0["level"] == 0 and g0["raw_segments"] == g0["count"]
    o = oracle.OracleScene(sc)
    pixels = np.arange(width * width, dtype=np.int32)
    ores = o.render(pixels, mode="exact", cap=256)
    prev = g0["count"]
    for c in (1, 2, 3):
        g = gpu_run(sc, fold=c)
        assert g["level"] == c
        assert g["raw_segments"] == g0["count"]
        assert np.array_equal(g["hits_per_pixel"], g0["hits_per_pixel"])
        assert g["hit_pairs"] == g0["hit_pairs"]
        # fewer records while the nodes grow (fold units hold <= 64 leaves, so
        # beyond level 2 the fused fold cannot merge more; rc_aggregate can)
        if c <= min(level, 2):
            assert g["count"] < prev, (c, g["count"], prev)
        prev = g["count"]
        assert np.abs(g["rgba"] - g0["rgba"]).max() < LOSSLESS
        rep = compare(sc, g, ores, pixels, by_counts=True)
        assert rep["hit_mismatch_pixels"] == 0 and rep["bad_pixels"] == 0, rep
        # per pixel the fused fold leaves at least the maximal runs of the
        # plain coarsening (units may cut big nodes), exactly those when every
        # unit is a whole node
        table = coarsen.node_tables(sc.leaf_anchor, sc.leaf_tree, sc.leaf_level, c)[c]
        ref = _oracle_runs(ores, table)
        clean = ref >= 0
        got = _record_counts(g, width * width)
        assert (got[clean] >= ref[clean]).all()
        vis_nodes = np.unique(np.searchsorted(table, g["visible"], side="right") - 1).size
        if g["units"] == vis_nodes:
            assert np.array_equal(got[clean], ref[clean]), (c, int((got[clean] != ref[clean]).sum()))
        # records are keyed by nodes of level c
        keys = np.unique(g["raw"][:, 7].astype(np.int64))
        table = g["forest"].node_table(c).cpu().numpy()
        assert np.isin(keys, table).all()


@pytest.mark.parametrize("which", ["c2", "shell"])
def test_aggregate_cycles_lossless(which):
    """rc_aggregate (a7): each cycle lowers the record count, pixels unchanged."""
    sc = sg.config2(width=96, maxlevel=5) if which == "c2" else sg.shell_uniform(3, 96, 16, gl_points=6)
    g0 = gpu_run(sc, fold=0)
    W = sc.camera.width
    ores = oracle.OracleScene(sc).render(np.arange(W * W, dtype=np.int32), mode="rule", cap=256)
    tables = coarsen.node_tables(sc.leaf_anchor, sc.leaf_tree, sc.leaf_level, 3)
    clean = None
    prev = g0["count"]
    for cyc in (1, 2, 3):
        g = gpu_run(sc, fold=0, cycles=cyc)
        assert g["level"] == cyc
        assert g["count"] < prev, (cyc, g["count"], prev)
        prev = g["count"]
        assert np.abs(g["rgba"] - g0["rgba"]).max() < LOSSLESS
        assert np.array_equal(g["hits_per_pixel"], g0["hits_per_pixel"])
        # exact record counts per pixel vs the plain coarsening of the oracle's segments
        ref = _oracle_runs(ores, tables[cyc])
        clean = ref >= 0
        got = _record_counts(g, W * W)
        assert np.array_equal(got[clean], ref[clean]), (cyc, int((got[clean] != ref[clean]).sum()))
    # on-chip fold then aggregation reaches the same level with the same pixels
    g2 = gpu_run(sc, fold=1, cycles=2)
    assert g2["level"] == 3
    assert np.abs(g2["rgba"] - g0["rgba"]).max() < LOSSLESS
    # aggregation merges only touching records of one node: per (node, pixel)
    # runs are maximal, so aggregating fold-1 records to level 3 gives at most
    # as many records as the fused fold to level 3 (which splits big nodes
    # into units)
    g3 = gpu_run(sc, fold=3) if which == "shell" else None
    if g3 is not None:
        assert g2["count"] <= g3["count"]


def test_affine_fold_matches():
    """fold_levels > 0 on the affine path (cast per leaf + one aggregation pass)."""
    sc = sg.config2(width=96, maxlevel=5)
    g0 = gpu_run(sc, fold=0)
    g2 = gpu_run(sc, fold=2)
    assert g2["level"] == 2 and g2["raw_segments"] == g0["count"]
    assert g2["count"] < g0["count"]
    assert np.abs(g2["rgba"] - g0["rgba"]).max() < LOSSLESS


def test_aggregate_errors():
    from paper_1809_01334_b200 import rc
    sc = sg.shell_uniform(1, 32, 4, gl_points=4)
    f = rc.Forest.from_scene(sc)
    f.camera_set(sc.camera)
    f.cull()
    with pytest.raises(rc.RcError):
        f.aggregate(1)           # before the cast -> RC_ERR_STATE
    with pytest.raises(rc.RcError):
        f.cast_segments(9)       # fold level out of range
    f.cast_segments(6)
    with pytest.raises(rc.RcError):
        f.aggregate(3)           # beyond the 8 node levels


def test_c5_generator_gpu_matches_host():
    """The GPU generator of C5 (scenegen/gpu.py) builds the same forest as the
    host generator on a reduced variant, and the same field up to the final
    fp32 rounding."""
    host = sg.config5(device=None, maxlevel=6, level0=3, width=64, nsources=24)
    dev = sg.config5(device="cuda", maxlevel=6, level0=3, width=64, nsources=24)
    assert np.array_equal(host.leaf_anchor, dev.leaf_anchor.cpu().numpy())
    assert np.array_equal(host.leaf_tree, dev.leaf_tree.cpu().numpy())
    assert np.array_equal(host.leaf_level, dev.leaf_level.cpu().numpy())
    fd = dev.leaf_field.cpu().numpy()
    assert np.abs(fd - host.leaf_field).max() <= 2e-7 * max(1.0, np.abs(host.leaf_field).max())
    assert abs(dev.inv_F / host.inv_F - 1.0) < 1e-12


def test_c5_reduced_fold_and_cycles():
    """C5's pipeline (fold 2 on chip + 3 aggregation cycles, N = 8) on a reduced
    adaptive shell vs the oracle on every pixel."""
    import dataclasses
    sc = sg.config5(device="cuda", maxlevel=6, level0=3, width=96, nsources=24)
    import bench
    sc = bench.scene_to_host(sc)
    o = oracle.OracleScene(sc)
    pixels = np.arange(96 * 96, dtype=np.int32)
    ores = o.render(pixels, mode="exact", cap=512)
    g0 = gpu_run(sc, fold=0)
    rep0 = compare(sc, g0, ores, pixels, cull=o.cull())
    assert rep0["hit_mismatch_pixels"] == 0 and rep0["bad_pixels"] == 0, rep0
    g = gpu_run(sc, fold=2, cycles=3)
    assert g["level"] == 5
    rep = compare(sc, g, ores, pixels, by_counts=True)
    assert rep["hit_mismatch_pixels"] == 0 and rep["bad_pixels"] == 0, rep
    assert g["count"] < g0["count"] // 2
    assert np.abs(g["rgba"] - g0["rgba"]).max() < LOSSLESS


def test_shell_generator_gpu_matches_host():
    """shell_uniform(device=cuda) (generator CUDA helper) vs the host generator."""
    host = sg.shell_uniform(3, 64, 16)
    dev = sg.shell_uniform(3, 64, 16, device="cuda")
    assert np.array_equal(host.leaf_anchor, dev.leaf_anchor.cpu().numpy())
    fd = dev.leaf_field.cpu().numpy()
    assert np.abs(fd - host.leaf_field).max() <= 2e-7 * max(1.0, np.abs(host.leaf_field).max())
    assert abs(dev.inv_F / host.inv_F - 1.0) < 1e-12
