"""Pins of the plain coarsening reference (oracle/coarsen.py) that the GPU
fold (row a6) and rc_aggregate (row a7) are checked against
(SURVEY §8(c) R22)."""
import numpy as np

import oracle
import scenegen as sg
from oracle import coarsen


def test_uniform_forest_tables_closed_form():
    """Uniform level-L forest of K trees: level c has K 8^(L-c) nodes, node k
    starting at leaf 8^c k, until the tree roots (level 0) stop coarsening."""
    for K, L in ((1, 3), (6, 2)):
        anchor, tree, level = sg.uniform_leaves(K, L)
        t = coarsen.node_tables(anchor, tree, level, L + 2)
        for c in range(1, L + 3):
            cc = min(c, L)
            assert np.array_equal(t[c], np.arange(K * 8 ** (L - cc)) * 8 ** cc)


def test_adaptive_nodes_tile_octants():
    """Every node of every level is either an unchanged leaf or a complete
    octant: its leaves are contiguous and their volumes sum to the octant's."""
    sc = sg.config2(width=32, maxlevel=5)
    anchor, tree, level = sc.leaf_anchor, sc.leaf_tree, sc.leaf_level
    n = len(tree)
    t = coarsen.node_tables(anchor, tree, level, 4)
    vol = 8.0 ** (-level.astype(np.float64))
    for c in range(1, 5):
        first = np.r_[t[c], n]
        assert first[0] == 0 and np.all(np.diff(first) >= 1)
        for k in range(len(first) - 1):
            a, b = first[k], first[k + 1]
            if b - a == 1:
                continue
            assert len(set(tree[a:b].tolist())) == 1
            v = vol[a:b].sum()
            lvl = -np.log(v) / np.log(8.0)
            assert abs(lvl - round(lvl)) < 1e-9           # a whole octant
            sh = 18 - int(round(lvl))
            assert np.all((anchor[a:b] >> sh) == (anchor[a] >> sh))   # inside it
        # the number of nodes never grows and levels nest
        if c > 1:
            assert np.isin(t[c], t[c - 1]).all()


def _rows(segs):
    h = np.zeros(len(segs), dtype=oracle.HIT_DTYPE)
    for q, (e, an, af) in enumerate(segs):
        h[q]["elem"], h[q]["alpha_near"], h[q]["alpha_far"], h[q]["flags"] = e, an, af, oracle.HIT
    return h


def test_run_counts_examples():
    h = _rows([(2, 3.5, 4.0), (0, 1.0, 2.0), (1, 2.0, 3.0)])   # unsorted on purpose
    assert coarsen.run_counts(h, None) == 3                    # leaves: one record each
    assert coarsen.run_counts(h, np.array([0])) == 2           # one node: [1,3] + gap + [3.5,4]
    assert coarsen.run_counts(h, np.array([0, 1])) == 3        # node boundary between e0 and e1
    assert coarsen.run_counts(h, np.array([0, 2])) == 2        # e0,e1 touch in node 0; e2 alone
    # touching within the tolerance, separated beyond it
    h2 = _rows([(0, 1.0, 2.0), (1, 2.0 + 5e-7, 3.0), (2, 3.0 + 5e-6, 4.0)])
    assert coarsen.run_counts(h2, np.array([0])) == 2
