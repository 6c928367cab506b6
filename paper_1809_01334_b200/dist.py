"""Multi-GPU plumbing of the hot path.

One process per GPU.  Every rank owns a contiguous SFC range of leaves
(PAPER.md:92-96).  What moves between ranks, and how:

* pre-partition: after the first cull every rank knows
  the weights w_E = visible pixel-centre rectangle area + 1 of its leaves
  (rc_leaf_weights, "weight proportional to its visible pixel count",
  PAPER.md:895-896); the SFC cuts move to equal prefix sums of the weights,
  aligned to node starts of the coarsest level the fold and the coarsening
  cycles reach, and the leaves move to their new owners (contiguous ranges:
  only SFC neighbours exchange);
* coarsening cycles: after each cycle but the last the
  cuts move to equal prefix sums of the record counts of the final-level
  nodes, and the records plus the leaf keys of the moved nodes go to their
  new owners, where a keys-only forest continues the aggregation
  (rc_segments_set + rc_aggregate);
* tile exchange: every record goes to the owner of its
  image tile -- inside librc over NCCL (rc_comm / rc_composite_tiles) when
  the process group is NCCL, host-staged through the group otherwise (gloo,
  used by the tests: two ranks on one GPU, no kernel waits on another).

The partition arithmetic here is host / torch bookkeeping (prefix sums,
searches, splits); no step of the method runs here.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist

SEG_WORDS = 8   # rc_seg = 8 x 32-bit words
MAXLEVEL = 18


def tile_owner(tx: int, ty: int, nranks: int) -> int:
    """Latin-square tile -> rank map of SURVEY §8(e)."""
    return (tx + ty) % nranks


def my_tiles(tiles_x: int, tiles_y: int, nranks: int, rank: int) -> List[Tuple[int, int]]:
    return [(tx, ty) for ty in range(tiles_y) for tx in range(tiles_x) if tile_owner(tx, ty, nranks) == rank]


# ---------------------------------------------------------------------------
# transport: torch.distributed, device tensors for NCCL, host-staged otherwise
# ---------------------------------------------------------------------------
class Transport:
    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host = dist.get_backend(group) != "nccl"

    def _to(self, t):
        if self.host:
            return t.cpu()
        return t if t.is_cuda else t.cuda()

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[world, *t.shape]."""
        src = self._to(t.contiguous())
        out = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(out, src, group=self.group)
        return torch.stack(out).to(t.device)

    def all_to_all_rows(self, send: torch.Tensor, send_counts: Sequence[int], recv_counts: Sequence[int]):
        """Rows of `send` split by send_counts to the ranks in order; returns the
        rows received, in rank order."""
        dev = send.device
        src = self._to(send.contiguous())
        out = torch.empty((int(sum(recv_counts)),) + tuple(send.shape[1:]), dtype=send.dtype, device=src.device)
        if self.host and dist.get_backend(self.group) == "gloo":
            # gloo has no all_to_all: pairwise send / recv (contiguous ranges talk to neighbours mostly)
            soff = [0]
            for c in send_counts:
                soff.append(soff[-1] + int(c))
            roff = [0]
            for c in recv_counts:
                roff.append(roff[-1] + int(c))
            out[roff[self.rank]:roff[self.rank + 1]] = src[soff[self.rank]:soff[self.rank + 1]]
            ops = []
            for p in range(self.world):
                if p == self.rank:
                    continue
                if send_counts[p]:
                    ops.append(dist.P2POp(dist.isend, src[soff[p]:soff[p + 1]].contiguous(), p, self.group))
                if recv_counts[p]:
                    ops.append(dist.P2POp(dist.irecv, out[roff[p]:roff[p + 1]], p, self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
        else:
            dist.all_to_all_single(out, src, output_split_sizes=[int(c) for c in recv_counts],
                                   input_split_sizes=[int(c) for c in send_counts], group=self.group)
        return out.to(dev)

    def counts_all_to_all(self, counts: Sequence[int]) -> List[int]:
        c = torch.tensor([int(x) for x in counts], dtype=torch.int64)
        allc = self.all_gather(c)                      # [world(src), world(dst)]
        return [int(x) for x in allc[:, self.rank].tolist()]

    def max(self, x: float) -> float:
        t = torch.tensor([float(x)], dtype=torch.float64)
        return float(self.all_gather(t).max())


# ---------------------------------------------------------------------------
# partition arithmetic
# ---------------------------------------------------------------------------
def weighted_ranges(weights: torch.Tensor, nranks: int) -> List[Tuple[int, int]]:
    """Contiguous SFC ranges with (nearly) equal prefix sums of the per-leaf
    weights.  Cut r is placed after the
    first leaf whose inclusive prefix sum reaches r/P of the total."""
    w = weights.to(torch.float64).flatten()
    n = w.numel()
    if n == 0:
        return [(0, 0)] * nranks
    c = torch.cumsum(w, 0)
    total = float(c[-1])
    cuts = [0]
    for r in range(1, nranks):
        target = torch.tensor(total * r / nranks, dtype=torch.float64, device=c.device)
        k = int(torch.searchsorted(c, target, right=False)) + 1
        cuts.append(min(max(k, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def node_starts(anchor: torch.Tensor, tree: torch.Tensor, level: torch.Tensor, levels: int) -> torch.Tensor:
    """Bool mask over the SFC-ordered leaves: True where a node of coarsening
    level `levels` starts (level c+1 replaces every family of 8 consecutive
    same-level siblings of level c by the parent).  Cutting
    the SFC ranges only at these leaves keeps every family of the first
    `levels` coarsening cycles on one rank ("cuts are aligned to
    family boundaries").  Vectorised torch (any device); bookkeeping only."""
    a = anchor.to(torch.int64)
    t = tree.to(torch.int64)
    lv = level.to(torch.int64)
    first = torch.arange(t.numel(), device=t.device)
    for _ in range(levels):
        n = t.numel()
        if n < 8:
            break
        m = n - 7
        sh = (MAXLEVEL - lv[:m]).clamp(min=0)
        cid = lambda aa, s: ((aa[:, 0] >> s) & 1) | (((aa[:, 1] >> s) & 1) << 1) | (((aa[:, 2] >> s) & 1) << 2)
        ok = (lv[:m] >= 1) & (cid(a[:m], sh) == 0)
        par = a[:m] >> (sh + 1)[:, None]
        for j in range(1, 8):
            aj = a[j:j + m]
            ok &= (t[j:j + m] == t[:m]) & (lv[j:j + m] == lv[:m]) & (cid(aj, sh) == j)
            ok &= ((aj >> (sh + 1)[:, None]) == par).all(dim=1)
        start = torch.zeros(n, dtype=torch.bool, device=t.device)
        start[:m] = ok
        inside = torch.zeros(n, dtype=torch.bool, device=t.device)
        for j in range(1, 8):
            inside[j:] |= start[:n - j]
        keep = ~inside
        lv = torch.where(start, lv - 1, lv)[keep]
        a, t, first = a[keep], t[keep], first[keep]
    mask = torch.zeros(anchor.shape[0], dtype=torch.bool, device=anchor.device)
    mask[first] = True
    return mask


def aligned_ranges(weights: torch.Tensor, nranks: int, allowed: torch.Tensor) -> List[Tuple[int, int]]:
    """weighted_ranges with every cut moved to the next allowed leaf (node start)."""
    rng = weighted_ranges(weights, nranks)
    idx = torch.nonzero(allowed.to(torch.bool).cpu()).flatten()
    n = int(weights.numel())
    cuts = [0]
    for r in range(1, nranks):
        c = rng[r][0]
        k = int(torch.searchsorted(idx, torch.tensor(c)))
        cut = int(idx[k]) if k < idx.numel() else n
        cuts.append(max(cut, cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def distributed_aligned_cuts(local_w: torch.Tensor, local_allowed: torch.Tensor, lo: int, n_total: int,
                             tp: Transport) -> List[Tuple[int, int]]:
    """aligned_ranges computed collectively: every rank holds only the weights
    of its own range [lo, lo + len(local_w)) and the allowed cut positions in
    it; the ranks exchange their totals and their candidate cuts (two small
    all-gathers).  Same result as aligned_ranges on the concatenated weights
    when every current cut is itself an allowed position."""
    P = tp.world
    w = local_w.to(torch.float64).flatten()
    tot = torch.tensor([float(w.sum()) if w.numel() else 0.0], dtype=torch.float64)
    tots = tp.all_gather(tot).flatten()
    off = float(tots[:tp.rank].sum())
    total = float(tots.sum())
    big = torch.iinfo(torch.int64).max
    cand = torch.full((max(P - 1, 1),), big, dtype=torch.int64)
    if w.numel():
        c = torch.cumsum(w, 0) + off
        allowed_idx = torch.nonzero(local_allowed.to(torch.bool)).flatten().cpu()
        hi = lo + w.numel()
        for r in range(1, P):
            target = total * r / P
            if not (off < target <= float(c[-1])):   # exactly one rank holds the leaf reaching the target
                continue
            k = int(torch.searchsorted(c, torch.tensor(target, dtype=torch.float64, device=c.device))) + 1
            raw = k   # local position of the raw cut (leaf k-1 is the first reaching the target)
            j = int(torch.searchsorted(allowed_idx, torch.tensor(raw)))
            cand[r - 1] = lo + int(allowed_idx[j]) if j < allowed_idx.numel() else hi
    allc = tp.all_gather(cand)
    cuts = [0]
    for r in range(1, P):
        v = int(allc[:, r - 1].min())
        cuts.append(max(min(v if v != big else n_total, n_total), cuts[-1]))
    cuts.append(n_total)
    return [(cuts[r], cuts[r + 1]) for r in range(P)]


def move_plan(old: Sequence[Tuple[int, int]], new: Sequence[Tuple[int, int]], rank: int):
    """Rows this rank sends to / receives from every rank when contiguous
    ranges change from `old` to `new` (only overlapping ranges talk)."""
    lo, hi = old[rank]
    nlo, nhi = new[rank]
    send = [max(0, min(hi, b) - max(lo, a)) for a, b in new]
    recv = [max(0, min(nhi, b) - max(nlo, a)) for a, b in old]
    return send, recv


def redistribute_rows(tensors, old, new, tp: Transport):
    """Move the leaf rows of contiguous SFC ranges from `old` to `new`
    ownership (PAPER.md:897-899 partition transfer)."""
    send, recv = move_plan(old, new, tp.rank)
    return [None if t is None else tp.all_to_all_rows(t, send, recv) for t in tensors]


# ---------------------------------------------------------------------------
# tile exchange
# ---------------------------------------------------------------------------
def partner_counts(counts: Sequence[int], partners, tp: Transport) -> List[int]:
    """Record counts between discovered pairs only: one
    int64 to every listed receiver, one from every listed sender, instead of
    the count all-to-all.  partners = (send_to, recv_from) rank lists."""
    send_to, recv_from = partners
    me = tp.rank
    missed = [q for q in range(tp.world) if q != me and counts[q] and q not in send_to]
    if missed:
        raise RuntimeError(f"records for ranks {missed}, which the partner discovery did not list")
    out = [0] * tp.world
    out[me] = int(counts[me])
    bufs, ops = {}, []
    for q in send_to:
        if q != me:
            bufs[("s", q)] = torch.tensor([int(counts[q])], dtype=torch.int64)
            ops.append(dist.P2POp(dist.isend, bufs[("s", q)], q, tp.group))
    for p in recv_from:
        if p != me:
            bufs[("r", p)] = torch.zeros(1, dtype=torch.int64)
            ops.append(dist.P2POp(dist.irecv, bufs[("r", p)], p, tp.group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for p in recv_from:
        if p != me:
            out[p] = int(bufs[("r", p)][0])
    return out


def exchange_records(send: torch.Tensor, counts: Sequence[int], tp: Transport, partners=None) -> torch.Tensor:
    """All-to-all(v) of rc_seg records ([sum(counts), 8] int32, grouped by
    destination rank); returns the records every rank sent to this one.
    partners (send_to, recv_from): counts move between those pairs only."""
    rl = tp.counts_all_to_all(counts) if partners is None else partner_counts(counts, partners, tp)
    return tp.all_to_all_rows(send, counts, rl)


def exchange_and_composite(forest, tiles, world: int, rank: int, comm=None, tp: Transport = None,
                           background=(0.0, 0.0, 0.0), partners=None):
    """rc_composite_tiles over librc's NCCL communicator (comm; partners set on
    it with Comm.set_partners), else rc_pack_tiles -> host-staged exchange ->
    rc_composite_records.  Returns this rank's tiles [ntiles][th][tw][4]."""
    tiles_x, tiles_y = tiles
    if comm is not None:
        out, _ = forest.composite_tiles(tiles_x, tiles_y, world, rank, comm=comm, background=background)
        return out
    tp = tp or Transport()
    send, counts = forest.pack_tiles(tiles_x, tiles_y, world, rank)
    recv = exchange_records(send, counts, tp, partners)
    out, _ = forest.composite_tiles(tiles_x, tiles_y, world, rank, recv=recv, background=background)
    return out


# ---------------------------------------------------------------------------
# NEXT(4): partition markers, partner discovery, vforest of several instances
# ---------------------------------------------------------------------------
def partition_markers(keys, num_trees: int, tp: Transport):
    """Partition markers: the tree and anchor of every
    rank's first leaf, all-gathered once per partition (the metadata every
    rank keeps).  keys = this rank's (anchor, tree, level) tensors.  Returns
    the rc_marker list of rc_exchange_partners: an empty rank repeats the next
    rank's marker, marker 0 = (0, (0,0,0)), marker P = (K, (0,0,0))."""
    anchor, tree = keys[0], keys[1]
    has = int(tree.numel() > 0)
    row = torch.tensor([has, int(tree[0]) if has else 0] + ([int(x) for x in anchor[0]] if has else [0, 0, 0]),
                       dtype=torch.int64)
    allm = tp.all_gather(row).cpu().tolist()
    P = tp.world
    out = [None] * (P + 1)
    out[P] = (num_trees, (0, 0, 0))
    for p in range(P - 1, -1, -1):
        out[p] = (allm[p][1], tuple(allm[p][2:5])) if allm[p][0] else out[p + 1]
    first = next((p for p in range(P) if allm[p][0]), P)
    for p in range(min(first + 1, P)):
        out[p] = (0, (0, 0, 0))
    return out


def discover_partners(forest, tiles, markers, tp: Transport):
    """rc_exchange_partners: (send_to, recv_from) of this rank, no communication."""
    return forest.exchange_partners(tiles[0], tiles[1], tp.world, tp.rank, markers)


def vforest_prepartition(forest, cameras, tp: Transport, align_levels: int, consts):
    """The paper's culling and pre-partition for one or
    more image instances: per instance camera_set + cull +
    rc_visible_area_add, then rc_vforest_create (only the leaves some
    instance sees, weights = visible pixel counts summed over the instances),
    the weighted SFC cut aligned to node starts and the move of the vforest's
    leaf rows to their new owners.  Returns (vforest, keys, ranges, stats);
    the input forest is left as it was (rendering is non-destructive)."""
    from . import rc
    w = torch.zeros(forest.n, dtype=torch.int64, device="cuda")
    for cam in cameras:
        forest.camera_set(cam)
        forest.cull()
        forest.visible_area_add(w)
    cnt = tp.all_gather(torch.tensor([int((w > 0).sum())], dtype=torch.int64)).flatten().tolist()
    first = int(sum(cnt[:tp.rank]))
    n_total = int(sum(cnt))
    vf, m, wv = forest.vforest(w, first_global_leaf=first)
    if vf is not None:
        rows = vf.leaves()
        vf.close()
    else:
        P = forest.P
        rows = [torch.zeros((0, 3), dtype=torch.int32, device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"),
                torch.zeros(0, dtype=torch.int8, device="cuda"),
                torch.zeros((0, 4 if forest.surface else (P + 1) ** 3), dtype=torch.float32, device="cuda")]
    old = [(int(sum(cnt[:p])), int(sum(cnt[:p + 1]))) for p in range(tp.world)]
    allowed = node_starts(rows[0], rows[1], rows[2], align_levels) if m else torch.zeros(0, dtype=torch.bool)
    ranges = distributed_aligned_cuts(wv, allowed, first, n_total, tp)
    rows = redistribute_rows(rows, old, ranges, tp)
    ctrl, R, P, kappa0, inv_F, q0 = consts[:6]
    extra = consts[6] if len(consts) > 6 else {}
    lo, hi = ranges[tp.rank]
    if hi <= lo:
        raise RuntimeError("empty vforest range on a rank (too few visible leaves for the ranks)")
    vf = rc.Forest(ctrl, R, P, *rows, kappa0, inv_F, q0, first_global_leaf=lo, **extra)
    stats = {"vforest_leaves": n_total, "visible_weight_local": int(wv.sum()) if m else 0, "vforest_ranges": ranges}
    return vf, rows[:3], ranges, stats


def assemble_image(tiles_out: dict, tiles_x: int, tiles_y: int, W: int, H: int) -> torch.Tensor:
    """Host-side helper: {rank: (tensor[ntiles][th][tw][4], [(tx,ty),...])} -> [H][W][4]."""
    tw, th = W // tiles_x, H // tiles_y
    img = torch.zeros((H, W, 4), dtype=torch.float32)
    for rank, (t, mine) in tiles_out.items():
        t = t.cpu()
        for k, (tx, ty) in enumerate(mine):
            img[ty * th:(ty + 1) * th, tx * tw:(tx + 1) * tw] = t[k]
    return img


def gather_image(out: torch.Tensor, tiles, W: int, H: int, tp: Transport):
    """Every rank's tiles to rank 0 (all-gather of padded tile stacks);
    returns the [H][W][4] image on rank 0 (host), None elsewhere."""
    tiles_x, tiles_y = tiles
    tw, th = W // tiles_x, H // tiles_y
    maxt = max(len(my_tiles(tiles_x, tiles_y, tp.world, r)) for r in range(tp.world))
    pad = torch.zeros((maxt, th, tw, 4), dtype=torch.float32, device=out.device)
    pad[:out.shape[0]] = out
    allt = tp.all_gather(pad).cpu()
    if tp.rank != 0:
        return None
    res = {r: (allt[r, :len(my_tiles(tiles_x, tiles_y, tp.world, r))], my_tiles(tiles_x, tiles_y, tp.world, r))
           for r in range(tp.world)}
    return assemble_image(res, tiles_x, tiles_y, W, H)


# ---------------------------------------------------------------------------
# coarsening cycles with repartition between them
# ---------------------------------------------------------------------------
def aggregate_with_repartition(forest, keys, rng, ranges, cycles, final_level, tp: Transport, scene_consts):
    """`cycles` aggregation cycles (rc_aggregate, one level each); between two
    cycles the SFC cuts move to equal prefix sums of the record counts of the
    final-level nodes and every moved node travels with its records and its
    leaf keys (anchor, tree, level) to its new owner, which continues on a
    keys-only forest ("repartition the elements, again
    weighted by their (updated) ray count ... marshal/send and receive").
    keys: this rank's (anchor, tree, level) device tensors of range `rng`;
    ranges: every rank's current range.  Returns (forest, keys, rng, ranges,
    moved_records); the returned forest is the caller's own (nothing moved)
    or a keys-only forest made here (the caller closes it)."""
    from . import rc
    moved = 0
    own = False   # the caller's forest is never closed here; keys-only forests made here are
    for c in range(cycles):
        forest.aggregate(1)
        if c == cycles - 1 or tp.world == 1:
            continue
        lo, hi = rng
        segs = forest.segments()
        recs = segs["raw"].clone()
        level = int(segs["level"])
        # record count of every final-level node of this range (the new weights)
        first = forest.node_table(final_level).to(torch.int64)     # local first leaves of the final nodes
        nodes = torch.searchsorted(first, (recs[:, 7].to(torch.int64) & 0xFFFFFFFF) - lo, right=True) - 1
        wnode = torch.bincount(nodes, minlength=first.numel()).to(torch.int64)
        w = torch.zeros(hi - lo, dtype=torch.int64, device=recs.device)
        w[first] = wnode + 1
        allowed = torch.zeros(hi - lo, dtype=torch.bool, device=recs.device)
        allowed[first] = True
        n_total = ranges[-1][1]
        new = distributed_aligned_cuts(w, allowed, lo, n_total, tp)
        if new == ranges:
            continue
        # records to the owner of their node's first leaf
        key = recs[:, 7].to(torch.int64) & 0xFFFFFFFF
        cuts = torch.tensor([b for _, b in new[:-1]], dtype=torch.int64, device=recs.device)
        dest = torch.searchsorted(cuts, key, right=True)
        order = torch.argsort(dest, stable=True)
        recs = recs[order]
        counts = torch.bincount(dest, minlength=tp.world).tolist()
        recv = exchange_records(recs, counts, tp)
        moved += sum(counts) - counts[tp.rank]
        keys = redistribute_rows(keys, ranges, new, tp)
        if own:
            forest.close()
        own = True
        ranges, rng = new, new[tp.rank]
        ctrl, R, P, kappa0, inv_F, q0, cam = scene_consts
        forest = rc.Forest(ctrl, R, P, keys[0], keys[1], keys[2], None, kappa0, inv_F, q0, first_global_leaf=rng[0])
        forest.camera_set(cam)
        forest.segments_set(recv, level)
    return forest, keys, rng, ranges, moved
