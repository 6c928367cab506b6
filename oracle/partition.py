"""Plain reference of the paper's exchange-partner discovery and of the vforest
(NEXT(4)).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): used by tests/ to check
librc's rc_exchange_partners and rc_vforest_create.  Shares no code with the
CUDA path; node bounding boxes and pixel rectangles come from oracle.c
(orc_element_aabb / orc_pixel_rect) through OracleScene.

* sfc_key / markers: "the metadata on partition markers ... encodes the
  location of each process' first leaf in the space-forest, more precisely,
  the number of the tree and the lower left front coordinates of each
  process' first element".  A position is the pair
  (tree, Morton key of the anchor at level 18), written as one integer
  tree * 8^18 + morton; rank p owns the positions [m_p, m_{p+1}).
* senders_of: "Beginning with the root of each tree, we run a binary search
  over the markers to identify the range of processes that own this tree's
  leaves.  We then descend into the recursion, where we stop if the bounding
  box of the current node does not intersect the writer's tile.  Otherwise we
  check if the range contains just a single process.  In this case, we add it
  to the list of senders and stop the recursion.  On the other hand, if the
  range is non-trivial ... we proceed with the recursion into each child,
  where we split the range of partition markers further using a nested binary
  search".  The node's bounding box is tested as the
  R6 pixel-centre rectangle of its camera-space Bernstein AABB (the cull's
  predicate applied to a virtual node); `eps` inflates (+) or deflates (-)
  the AABB by that many world units (DESIGN D19: sure / possible relations).
* receivers_of: the same relation read from the sender's side
  (DESIGN D19).
* vforest_leaves: "Whenever we reach a leaf, it is visible to at least one
  instance and we add it to the vforest ... weight proportional to its
  visible pixel count summed over all instances".
"""
from __future__ import annotations

import dataclasses
from bisect import bisect_left, bisect_right

import numpy as np

from . import OracleScene

MAXLEVEL = 18
SPAN = 8 ** MAXLEVEL          # SFC positions per tree


def _spread(v: int) -> int:
    r = 0
    for b in range(MAXLEVEL):
        r |= ((v >> b) & 1) << (3 * b)
    return r


def sfc_key(tree: int, anchor) -> int:
    """Global SFC position of a leaf / node anchor: tree-major, Morton within
    the tree (x the lowest bit of each triple)."""
    return int(tree) * SPAN + (_spread(int(anchor[0])) | (_spread(int(anchor[1])) << 1) | (_spread(int(anchor[2])) << 2))


def markers(scene, cuts):
    """Partition markers of contiguous SFC ranges: cuts = [c_0 = 0, c_1, ...,
    c_P = n] leaf indices; m_p = position of rank p's first leaf (an empty
    rank takes the next rank's marker), m_P = K * 8^18."""
    n = scene.num_leaves
    K = scene.num_trees
    P = len(cuts) - 1
    m = [0] * (P + 1)
    m[P] = K * SPAN
    for p in range(P - 1, -1, -1):
        c = int(cuts[p])
        m[p] = m[p + 1] if c >= int(cuts[p + 1]) or c >= n else sfc_key(scene.leaf_tree[c], scene.leaf_anchor[c])
    # the first non-empty rank also owns the positions before its first leaf
    first = next((p for p in range(P) if int(cuts[p]) < int(cuts[p + 1])), P)
    for p in range(min(first + 1, P)):
        m[p] = 0
    return m


def owner_of(m, key):
    """Rank owning SFC position `key` (the last p with m_p <= key)."""
    return bisect_right(m, key) - 1


@dataclasses.dataclass
class _NodeRects:
    """Pixel-centre rectangles of virtual nodes under the scene's camera."""
    scene: object
    eps: float

    def rect(self, tree, anchor, level):
        sc = self.scene
        P = sc.field_degree
        nf = 4 if getattr(sc, "dim", 3) == 2 else (P + 1) ** 3
        one = dataclasses.replace(sc, leaf_anchor=np.array([anchor], dtype=np.int32),
                                  leaf_tree=np.array([tree], dtype=np.int32),
                                  leaf_level=np.array([level], dtype=np.int8),
                                  leaf_field=np.zeros((1, nf), dtype=np.float32))
        o = OracleScene(one)
        lo, hi = o.aabb(0)
        ok, r = o.pixel_rect(np.asarray(lo) - self.eps, np.asarray(hi) + self.eps)
        return r if ok else None


def tile_rects(W, H, tiles_x, tiles_y, owner, q):
    """Pixel rectangles (i0, i1, j0, j1) of the tiles owned by writer q."""
    tw, th = W // tiles_x, H // tiles_y
    return [(tx * tw, tx * tw + tw - 1, ty * th, ty * th + th - 1)
            for ty in range(tiles_y) for tx in range(tiles_x) if owner(tx, ty) == q]


def _meets(r, tiles):
    return any(not (r[1] < t[0] or r[0] > t[1] or r[3] < t[2] or r[2] > t[3]) for t in tiles)


def senders_of(scene, m, tiles, eps=0.0):
    """The paper's receiver-side traversal for a writer
    owning the pixel rectangles `tiles`: the set of vforest ranks that hold
    leaves whose nodes' boxes meet the tiles.  m: partition markers."""
    P = len(m) - 1
    nodes = _NodeRects(scene, eps)
    quad = getattr(scene, "dim", 3) == 2
    out = set()

    def nonempty(lo, hi):
        return [p for p in range(lo, hi + 1) if m[p] < m[p + 1]]

    def recurse(tree, anchor, level, lo, hi):
        r = nodes.rect(tree, anchor, level)
        if r is None or not _meets(r, tiles):
            return
        ranks = nonempty(lo, hi)
        if not ranks:
            return
        if len(ranks) == 1:
            out.add(ranks[0])
            return
        h = 1 << (MAXLEVEL - level - 1)
        for c in range(4 if quad else 8):
            a = (anchor[0] + h * (c & 1), anchor[1] + h * ((c >> 1) & 1), anchor[2] + h * ((c >> 2) & 1))
            s = sfc_key(tree, a)
            e = s + 8 ** (MAXLEVEL - level - 1)
            # nested binary search inside [lo, hi]: ranks whose range meets [s, e)
            clo = max(lo, bisect_right(m, s, lo, hi + 1) - 1)
            chi = min(hi, bisect_left(m, e, lo, hi + 2) - 1)
            recurse(tree, a, level + 1, clo, chi)

    for k in range(scene.num_trees):
        s, e = k * SPAN, (k + 1) * SPAN
        lo = bisect_right(m, s) - 1
        hi = bisect_left(m, e) - 1
        recurse(k, (0, 0, 0), 0, max(lo, 0), min(hi, P - 1))
    return out


def partner_relation(scene, m, tiles_x, tiles_y, owner, eps=0.0):
    """{(p, q)}: vforest rank p sends to writer q (every writer's traversal)."""
    W, H = scene.camera.width, scene.camera.height
    P = len(m) - 1
    rel = set()
    for q in range(P):
        for p in senders_of(scene, m, tile_rects(W, H, tiles_x, tiles_y, owner, q), eps):
            rel.add((p, q))
    return rel


def brute_force_pairs(scene, cuts, tiles_x, tiles_y, owner):
    """{(p, q)}: some visible leaf of rank p has a (EPS-inflated) pixel-centre
    rectangle meeting a tile of q -- every pair that can carry a record."""
    o = OracleScene(scene)
    vis, amb, rects = o.cull()
    W, H = scene.camera.width, scene.camera.height
    P = len(cuts) - 1
    tiles = [tile_rects(W, H, tiles_x, tiles_y, owner, q) for q in range(P)]
    rel = set()
    for p in range(P):
        for e in range(int(cuts[p]), int(cuts[p + 1])):
            if not (vis[e] or amb[e]):
                continue
            r = rects[e]
            if r[1] < r[0]:
                continue
            for q in range(P):
                if _meets(r, tiles[q]):
                    rel.add((p, q))
    return rel


def visible_area(scene, camera):
    """Pixel-centre rectangle area of every leaf under one image instance
    (0 when culled): the oracle's cull rect, not inflated."""
    o = OracleScene(dataclasses.replace(scene, camera=camera))
    n = scene.num_leaves
    area = np.zeros(n, dtype=np.int64)
    amb = np.zeros(n, dtype=bool)
    for e in range(n):
        lo, hi = o.aabb(e)
        ok, r = o.pixel_rect(lo, hi)
        if ok:
            area[e] = (r[1] - r[0] + 1) * (r[3] - r[2] + 1)
        okp, rp = o.pixel_rect(np.asarray(lo) - 1e-6, np.asarray(hi) + 1e-6)
        okm, rm = o.pixel_rect(np.asarray(lo) + 1e-6, np.asarray(hi) - 1e-6)
        amb[e] = okp != okm or (okp and okm and tuple(rp) != tuple(rm))
    return area, amb


def vforest_leaves(scene, cameras):
    """Leaves of the vforest of several image instances:
    indices of the leaves visible in at least one instance, and their weight =
    visible pixel count summed over the instances.  Also returns the
    ambiguous mask (a leaf whose area is eps-ambiguous in some instance)."""
    tot = np.zeros(scene.num_leaves, dtype=np.int64)
    amb = np.zeros(scene.num_leaves, dtype=bool)
    for cam in cameras:
        a, m = visible_area(scene, cam)
        tot += a
        amb |= m
    keep = np.nonzero(tot > 0)[0]
    return keep, tot[keep], amb


def receivers_of(scene, m, tiles_x, tiles_y, owner, p, eps=0.0):
    """Writers that vforest rank p sends to: every writer q whose traversal
    lists p (the sender side reads the same relation, DESIGN D19)."""
    return {q for (pp, q) in partner_relation(scene, m, tiles_x, tiles_y, owner, eps) if pp == p}
