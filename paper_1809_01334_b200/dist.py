"""Multi-GPU plumbing of the tile exchange.

One process per GPU.  Each rank owns a contiguous SFC range of leaves
(weights proportional to the visible pixel count),
casts its segments, packs them by tile owner (tile (tx,ty) -> rank
(tx+ty) mod P) with librc's rc_pack_tiles, and the records travel with two
torch.distributed all_to_all_single calls (counts, then 32-byte records) —
the path's only data-path collective.  The owner composites its tiles with
rc_composite_tiles.  Nothing here computes any part of the method.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist

SEG_WORDS = 8   # rc_seg = 8 x 32-bit words


def tile_owner(tx: int, ty: int, nranks: int) -> int:
    """Latin-square tile -> rank map of SURVEY §8(e)."""
    return (tx + ty) % nranks


def my_tiles(tiles_x: int, tiles_y: int, nranks: int, rank: int) -> List[Tuple[int, int]]:
    return [(tx, ty) for ty in range(tiles_y) for tx in range(tiles_x) if tile_owner(tx, ty, nranks) == rank]


def weighted_ranges(weights: torch.Tensor, nranks: int) -> List[Tuple[int, int]]:
    """Contiguous SFC ranges with (nearly) equal prefix sums of the per-leaf
    weights (w_E = rect area + 1).  Cut r is
    the first leaf whose inclusive prefix sum reaches r/P of the total."""
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


MAXLEVEL = 18


def node_starts(anchor: torch.Tensor, tree: torch.Tensor, level: torch.Tensor, levels: int) -> torch.Tensor:
    """Bool mask over the SFC-ordered leaves: True where a node of coarsening
    level `levels` starts (level c+1 replaces every family of 8 consecutive
    same-level siblings of level c by the parent).  Cutting
    the SFC ranges only at these leaves keeps every family of the first
    `levels` coarsening cycles on one rank ("cuts are aligned to
    family boundaries"), so fold and aggregation never need a neighbour's
    leaves.  Vectorised torch (any device); host logic, no method arithmetic."""
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


def exchange_records(send: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """All-to-all(v) of rc_seg records: `send` is [sum(counts), 8] int32 with
    the records for rank d in rows [sum(counts[:d]), sum(counts[:d+1])).
    Returns the records every rank sent to this one."""
    world = dist.get_world_size(group)
    dev = send.device
    cnt = torch.tensor(list(counts), dtype=torch.int64, device=dev)
    assert cnt.numel() == world
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt, group=group)
    rl = [int(x) for x in rcnt.tolist()]
    recv = torch.empty((sum(rl), SEG_WORDS), dtype=torch.int32, device=dev)
    dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=rl, input_split_sizes=list(counts),
                           group=group)
    return recv


def exchange_and_composite(forest, tiles, world: int, rank: int, background=(0.0, 0.0, 0.0), group=None):
    """rc_pack_tiles -> all_to_all -> rc_composite_tiles; returns this rank's
    tiles [ntiles][th][tw][4]."""
    tiles_x, tiles_y = tiles
    send, counts = forest.pack_tiles(tiles_x, tiles_y, world, rank)
    recv = exchange_records(send, counts, group=group)
    out, _ = forest.composite_tiles(tiles_x, tiles_y, world, rank, recv=recv, background=background)
    return out


def assemble_image(tiles_out: dict, tiles_x: int, tiles_y: int, W: int, H: int) -> torch.Tensor:
    """Host-side helper: {rank: (tensor[ntiles][th][tw][4], [(tx,ty),...])} -> [H][W][4]."""
    tw, th = W // tiles_x, H // tiles_y
    img = torch.zeros((H, W, 4), dtype=torch.float32)
    for rank, (t, mine) in tiles_out.items():
        t = t.cpu()
        for k, (tx, ty) in enumerate(mine):
            img[ty * th:(ty + 1) * th, tx * tw:(tx + 1) * tw] = t[k]
    return img
