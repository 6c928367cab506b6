"""Pins of oracle/partition.py (NEXT(4): partition-marker partner discovery and
the vforest of several image instances).
CPU only.  The traversal is checked against brute force over the leaves (every
pair that can carry a record must be found), against cases where the paper's
recursion must stop exactly at the leaves or at whole trees (then it equals
brute force / the trees' own rectangles), and the markers against the ranks'
own leaves."""
import dataclasses

import numpy as np
import pytest

import oracle
import scenegen as sg
from oracle import partition as op


def owner_latin(P):
    return lambda tx, ty: (tx + ty) % P


def _with_leaves(scene, anchor, tree, level):
    P = scene.field_degree
    nf = 4 if getattr(scene, "dim", 3) == 2 else (P + 1) ** 3
    return dataclasses.replace(scene, leaf_anchor=np.asarray(anchor, np.int32), leaf_tree=np.asarray(tree, np.int32),
                               leaf_level=np.asarray(level, np.int8),
                               leaf_field=np.zeros((len(tree), nf), np.float32))


def _random_cuts(n, P, rng, empty=False):
    c = np.sort(rng.choice(np.arange(1, n), size=P - 1, replace=empty))
    if empty and P > 2:
        c[0] = c[1]   # one empty rank
    return [0] + [int(x) for x in c] + [n]


def test_markers_own_the_ranks_leaves():
    """m_p <= key(leaf) < m_{p+1} exactly for the leaves of rank p (brute
    force over every leaf), including empty ranks and SFC order of the keys."""
    sc = sg.shell_uniform(2, 16, 4)
    n = sc.num_leaves
    keys = [op.sfc_key(sc.leaf_tree[e], sc.leaf_anchor[e]) for e in range(n)]
    assert all(a < b for a, b in zip(keys, keys[1:]))
    rng = np.random.default_rng(3)
    for P, empty in ((2, False), (5, False), (6, True)):
        cuts = _random_cuts(n, P, rng, empty)
        m = op.markers(sc, cuts)
        assert m[0] == 0 and m[-1] == sc.num_trees * op.SPAN
        for p in range(P):
            for e in range(cuts[p], cuts[p + 1]):
                assert op.owner_of(m, keys[e]) == p
            if cuts[p] == cuts[p + 1]:
                assert m[p] == m[p + 1]


@pytest.mark.parametrize("which", ["c1", "shell"])
def test_discovery_superset_of_brute_force(which):
    """Every (sender, writer) pair some visible leaf links is found, for
    random SFC cuts ("discovers all processes that will be
    sending at least one ray segment")."""
    sc = sg.config1(width=32) if which == "c1" else sg.shell_uniform(2, 24, 4)
    rng = np.random.default_rng(11)
    for P, tiles in ((2, (2, 2)), (3, (4, 4)), (5, (4, 2))):
        cuts = _random_cuts(sc.num_leaves, P, rng)
        m = op.markers(sc, cuts)
        brute = op.brute_force_pairs(sc, cuts, tiles[0], tiles[1], owner_latin(P))
        found = op.partner_relation(sc, m, tiles[0], tiles[1], owner_latin(P), eps=1e-6)
        assert brute <= found, (P, tiles, brute - found)
        assert brute, "degenerate case: no pairs"


def test_discovery_one_leaf_per_rank_is_brute_force():
    """With exactly one leaf per rank the recursion stops at the leaves, so the
    relation is the brute-force one."""
    base = sg.config1(width=32)
    anc, tree, lev = sg.uniform_leaves(1, 1)
    sc = _with_leaves(base, anc, tree, lev)
    cuts = list(range(9))
    m = op.markers(sc, cuts)
    for tiles in ((2, 2), (4, 4), (8, 1)):
        brute = op.brute_force_pairs(sc, cuts, tiles[0], tiles[1], owner_latin(8))
        found = op.partner_relation(sc, m, tiles[0], tiles[1], owner_latin(8), eps=1e-6)
        assert found == brute, tiles


def test_discovery_whole_trees_are_the_root_rectangles():
    """Ranks owning whole trees: the recursion stops at the roots, so the
    relation is {(p, q): root rectangle of p's trees meets q's tiles}, with the
    roots' rectangles taken as the cull rectangles of a level-0 forest."""
    base = sg.shell_uniform(2, 24, 4)
    roots = _with_leaves(base, np.zeros((6, 3)), np.arange(6), np.zeros(6))
    vis, amb, rects = oracle.OracleScene(roots).cull()
    # 3 ranks x 2 trees of the level-2 shell (64 leaves per tree)
    cuts = [0, 128, 256, 384]
    m = op.markers(base, cuts)
    W, H = base.camera.width, base.camera.height
    for tiles in ((2, 2), (3, 3)):
        own = owner_latin(3)
        expect = set()
        for k in range(6):
            if not (vis[k] or amb[k]):
                continue
            for q in range(3):
                if op._meets(rects[k], op.tile_rects(W, H, tiles[0], tiles[1], own, q)):
                    expect.add((k // 2, q))
        assert op.partner_relation(base, m, tiles[0], tiles[1], own, eps=1e-6) == expect


def test_discovery_single_rank_and_empty_ranks():
    sc = sg.config1(width=32)
    m = op.markers(sc, [0, sc.num_leaves])
    assert op.partner_relation(sc, m, 2, 2, owner_latin(1), eps=1e-6) == {(0, 0)}
    # empty ranks (first, middle, last) never send
    cuts = [0, 0, 100, 100, 512, 512]
    m = op.markers(sc, cuts)
    rel = op.partner_relation(sc, m, 4, 4, owner_latin(5), eps=1e-6)
    assert {p for p, _ in rel} <= {1, 3}
    assert op.brute_force_pairs(sc, cuts, 4, 4, owner_latin(5)) <= rel


def test_discovery_sure_within_possible():
    """Deflating the boxes (eps < 0) can only lose pairs (the band the product
    must fall in, DESIGN D19)."""
    sc = sg.shell_uniform(2, 24, 4)
    cuts = _random_cuts(sc.num_leaves, 4, np.random.default_rng(5))
    m = op.markers(sc, cuts)
    sure = op.partner_relation(sc, m, 4, 4, owner_latin(4), eps=-1e-6)
    poss = op.partner_relation(sc, m, 4, 4, owner_latin(4), eps=1e-6)
    assert sure <= poss and sure


def test_discovery_quadtree_surface():
    sc = sg.mandelbrot_hexagon(level0=2, maxlevel=4, max_iter=12, width=48)
    rng = np.random.default_rng(2)
    for P in (2, 4):
        cuts = _random_cuts(sc.num_leaves, P, rng)
        m = op.markers(sc, cuts)
        brute = op.brute_force_pairs(sc, cuts, 4, 4, owner_latin(P))
        found = op.partner_relation(sc, m, 4, 4, owner_latin(P), eps=1e-6)
        assert brute <= found and brute


def test_vforest_union_of_instances():
    """vforest leaves = leaves visible in at least one instance; weight = the
    pixel count summed over the instances, pinned against
    the oracle's own cull flags per instance."""
    sc = sg.config2(width=64, maxlevel=5)
    cams = [sg.perspective_camera((0.5, 0.5, 2.2), (0.5, 0.5, 0.5), 12.0, 48, 40),
            sg.orthographic_camera((0.2, 0.3, 0.5), (1.0, 0.1, 0.05), 3.0, 0.35, 32, 32)]
    keep, w, amb = op.vforest_leaves(sc, cams)
    union = np.zeros(sc.num_leaves, bool)
    tot = np.zeros(sc.num_leaves, np.int64)
    for cam in cams:
        vis, a, rects = oracle.OracleScene(dataclasses.replace(sc, camera=cam)).cull()
        union |= vis
        area, am = op.visible_area(sc, cam)
        clean = ~am
        assert np.array_equal(area[clean] > 0, vis[clean])
        # the weight is the cull rectangle's pixel count (clean leaves: inflated rect == rect)
        ra = np.where(vis, (rects[:, 1] - rects[:, 0] + 1) * (rects[:, 3] - rects[:, 2] + 1), 0)
        assert np.array_equal(area[clean], ra[clean])
        tot += area
    ks = set(keep.tolist())
    assert set(np.nonzero(union & ~amb)[0].tolist()) <= ks <= set(np.nonzero(union | amb)[0].tolist())
    assert np.array_equal(w, tot[keep]) and (w > 0).all()
    assert 0 < len(keep) < sc.num_leaves   # the narrow instances do not see everything
