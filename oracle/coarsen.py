"""Plain reference of the paper's coarsening cycles.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): used by tests/ to check
the node tables of rc_forest_create and the record counts of the on-chip fold
(row a6) and of rc_aggregate (row a7).  Shares no code with the CUDA path.

* node_tables: "coarsening ... replaces a complete local family by its
  parent": level c+1 is level c with every run of 8
  consecutive same-level siblings (child ids 0..7 of one parent, SFC order)
  replaced by the parent.  Plain loops (small forests only).
* run_counts: per pixel, the number of records after merging, in alpha order,
  consecutive segments that touch (|gap| <= tau max(1, alpha))
  and lie in the same node (only touching segments combine, so a
  ray that leaves and re-enters a node keeps two records).
"""
from __future__ import annotations

import numpy as np

MAXLEVEL = 18


def node_tables(anchor, tree, level, levels):
    """{c: first-leaf index of every node of level c} for c = 1..levels."""
    nodes = [(int(tree[k]), tuple(int(x) for x in anchor[k]), int(level[k]), k) for k in range(len(tree))]
    out = {}
    for c in range(1, levels + 1):
        new, k = [], 0
        while k < len(nodes):
            t, a, l, first = nodes[k]
            family = False
            if l >= 1 and k + 7 < len(nodes):
                sh = MAXLEVEL - l
                parent = tuple(x >> (sh + 1) for x in a)
                family = True
                for j in range(8):
                    t2, a2, l2, _ = nodes[k + j]
                    child = ((a2[0] >> sh) & 1) | (((a2[1] >> sh) & 1) << 1) | (((a2[2] >> sh) & 1) << 2)
                    family = family and t2 == t and l2 == l and tuple(x >> (sh + 1) for x in a2) == parent \
                        and child == j
            if family:
                new.append((t, a, l - 1, first))
                k += 8
            else:
                new.append(nodes[k])
                k += 1
        nodes = new
        out[c] = np.array([nd[3] for nd in nodes], dtype=np.int64)
    return out


def run_counts(hit_rows, node_first, tau=1e-6, hit_flag=1):
    """hit_rows: the oracle's per-pixel hit records (oracle.HIT_DTYPE rows with
    elem >= 0); node_first: first-leaf table of the target level (None = the
    leaves themselves).  Returns the number of merged records."""
    h = hit_rows[(hit_rows["elem"] >= 0) & ((hit_rows["flags"] & hit_flag) != 0)]
    if h.size == 0:
        return 0
    order = np.lexsort((h["elem"], h["alpha_near"]))
    h = h[order]
    elem = h["elem"].astype(np.int64)
    node = elem if node_first is None else np.searchsorted(node_first, elem, side="right") - 1
    runs = 1
    for k in range(1, h.size):
        an, afp = float(h["alpha_near"][k]), float(h["alpha_far"][k - 1])
        if abs(an - afp) > tau * max(1.0, abs(an)) or node[k] != node[k - 1]:
            runs += 1
    return runs
