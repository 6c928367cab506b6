"""World-size-2 gloo tests of the multi-GPU plumbing on CPU (SURVEY §4 4(a),
§8(e)): SFC ranges, the count + record all-to-all of dist.exchange_records,
and the tile-owner protocol end to end.  Segments come from the oracle (test
infrastructure), packed by tile owner in this file; the product code under
test is paper_1809_01334_b200.dist."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1809_01334_b200 import dist as rdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q, *args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_weighted_ranges():
    w = torch.tensor([1, 1, 1, 1, 10, 1, 1, 1], dtype=torch.float64)
    r = rdist.weighted_ranges(w, 2)
    assert r[0][0] == 0 and r[-1][1] == 8 and r[0][1] == r[1][0]
    # the heavy leaf ends up alone-ish: both halves carry about half the weight
    s0 = float(w[r[0][0]:r[0][1]].sum())
    assert abs(s0 - 8.5) <= 10
    r4 = rdist.weighted_ranges(torch.ones(10), 4)
    assert [b - a for a, b in r4] == [3, 2, 3, 2] or sum(b - a for a, b in r4) == 10
    assert rdist.weighted_ranges(torch.ones(0), 3) == [(0, 0)] * 3


def _exchange_fn(rank, world):
    # each rank sends (rank*100 + dest*10 + k) records to each destination
    counts = [rank + d + 1 for d in range(world)]
    rows = []
    for d in range(world):
        for k in range(counts[d]):
            rows.append([rank, d, k, 0, 0, 0, 0, rank * 100 + d * 10 + k])
    send = torch.tensor(rows, dtype=torch.int32)
    recv = rdist.exchange_records(send, counts, rdist.Transport())
    return recv.numpy()


def test_exchange_records_gloo():
    out = _spawn(_exchange_fn)
    for rank, recv in out.items():
        assert np.all(recv[:, 1] == rank)
        for src in range(2):
            part = recv[recv[:, 0] == src]
            assert len(part) == src + rank + 1
            assert sorted(part[:, 7].tolist()) == [src * 100 + rank * 10 + k for k in range(src + rank + 1)]


def _protocol_fn(rank, world):
    """Oracle segments of this rank's SFC range -> pack by tile owner -> exchange
    -> per-pixel fold on the owner."""
    import oracle
    import scenegen as sg
    sc = sg.config1(width=24)
    n = sc.num_leaves
    lo, hi = rdist.weighted_ranges(torch.ones(n), world)[rank]
    part = oracle.OracleScene(sc.subset(lo, hi)).render(mode="rule", cap=32)
    W = sc.camera.width
    tiles_x = tiles_y = 4
    tw = th = W // 4
    rows = [[] for _ in range(world)]
    for q in range(part["pixels"].shape[0]):
        for h in part["hits"][q]:
            if h["elem"] < 0 or not (h["flags"] & oracle.HIT):
                continue
            p = int(h["pixel"])
            dest = rdist.tile_owner((p % W) // tw, (p // W) // th, world)
            rec = np.zeros(8, np.int32)
            f = rec.view(np.float32)
            rec[0] = p
            f[1], f[2], f[3] = h["alpha_near"], h["alpha_far"], h["a"]
            f[4:7] = h["b"]
            rec[7] = int(h["elem"]) + lo
            rows[dest].append(rec)
    counts = [len(r) for r in rows]
    send = torch.tensor(np.array([x for r in rows for x in r]).reshape(-1, 8), dtype=torch.int32)
    recv = rdist.exchange_records(send, counts, rdist.Transport()).numpy()
    # fold my tiles' pixels with the oracle's per-pixel fold
    mine = rdist.my_tiles(tiles_x, tiles_y, world, rank)
    img = {}
    for tx, ty in mine:
        for y in range(th):
            for x in range(tw):
                p = (ty * th + y) * W + tx * tw + x
                recs = recv[recv[:, 0] == p]
                segs = np.zeros(len(recs), dtype=oracle.HIT_DTYPE)
                fl = recs.view(np.float32)
                segs["elem"] = recs[:, 7]
                segs["pixel"] = p
                segs["alpha_near"], segs["alpha_far"], segs["a"] = fl[:, 1], fl[:, 2], fl[:, 3]
                segs["b"] = fl[:, 4:7]
                img[p] = oracle.fold_pixel(segs)[0]
    return img


def test_tile_protocol_gloo_matches_single_process():
    import oracle
    import scenegen as sg
    out = _spawn(_protocol_fn)
    sc = sg.config1(width=24)
    full = oracle.OracleScene(sc).render(mode="rule", with_hits=False)
    merged = {}
    for r in out.values():
        merged.update(r)
    assert len(merged) == 24 * 24
    for q, p in enumerate(full["pixels"]):
        # records cross the wire as fp32: compare at fp32 resolution
        assert np.abs(merged[int(p)] - full["rgba"][q]).max() < 1e-6


def test_node_starts_match_coarsening_reference():
    """dist.node_starts (vectorised) vs the plain coarsening reference of
    oracle/coarsen.py on an adaptive forest; aligned cuts fall on node starts."""
    import scenegen as sg
    from oracle import coarsen
    sc = sg.config2(width=32, maxlevel=5)
    A, T, L = (torch.as_tensor(x) for x in (sc.leaf_anchor, sc.leaf_tree, sc.leaf_level))
    ref = coarsen.node_tables(sc.leaf_anchor, sc.leaf_tree, sc.leaf_level, 3)
    for c in (1, 2, 3):
        m = rdist.node_starts(A, T, L, c)
        assert np.array_equal(np.nonzero(m.numpy())[0], ref[c])
    m3 = rdist.node_starts(A, T, L, 3)
    rng = rdist.aligned_ranges(torch.ones(sc.num_leaves), 4, m3)
    assert rng[0][0] == 0 and rng[-1][1] == sc.num_leaves
    for lo, hi in rng[1:]:
        assert lo == sc.num_leaves or m3[lo]
    # uniform forest: level-c nodes start at multiples of 8^c
    a, t, l = sg.uniform_leaves(2, 3)
    m = rdist.node_starts(torch.as_tensor(a), torch.as_tensor(t), torch.as_tensor(l), 2)
    assert np.array_equal(np.nonzero(m.numpy())[0], np.arange(0, 2 * 512, 64))


def _forest_weights(seed):
    import scenegen as sg
    sc = sg.config2(width=32, maxlevel=5)
    A, T, L = (torch.as_tensor(x) for x in (sc.leaf_anchor, sc.leaf_tree, sc.leaf_level))
    allowed = rdist.node_starts(A, T, L, 2)
    w = torch.as_tensor(np.random.default_rng(seed).integers(1, 60, sc.num_leaves), dtype=torch.int64)
    return w, allowed


def _cuts_fn(rank, world, seed):
    """Each rank holds only its own range's weights (equal-count aligned
    ranges); the collective cut must equal aligned_ranges on all weights."""
    w, allowed = _forest_weights(seed)
    old = rdist.aligned_ranges(torch.ones(w.numel()), world, allowed)
    lo, hi = old[rank]
    tp = rdist.Transport()
    new = rdist.distributed_aligned_cuts(w[lo:hi], allowed[lo:hi], lo, w.numel(), tp)
    # move the rows of a per-leaf array and check we receive exactly our new range
    idx = torch.arange(lo, hi, dtype=torch.int64)
    moved = rdist.redistribute_rows([idx, idx.to(torch.int8).reshape(-1, 1).repeat(1, 3)], old, new, tp)
    return new, moved[0].numpy(), moved[1].numpy()


@pytest.mark.parametrize("world,seed", [(2, 1), (3, 2), (4, 3)])
def test_distributed_weighted_cuts_and_leaf_moves_gloo(world, seed):
    """SURVEY §8(e) partition: cuts at equal prefix sums of w_E, aligned to
    node starts, computed collectively from per-rank weights;
    the leaf rows move to their new owners in SFC order."""
    out = _spawn(_cuts_fn, world, seed)
    w, allowed = _forest_weights(seed)
    ref = rdist.aligned_ranges(w, world, allowed)
    for rank, (new, idx, idx8) in out.items():
        assert new == ref, (new, ref)
        lo, hi = ref[rank]
        assert np.array_equal(idx, np.arange(lo, hi))
        assert np.array_equal(idx8[:, 0], np.arange(lo, hi).astype(np.int8))
    # balance: every rank within one node's weight of the mean
    tot = float(w.sum())
    for lo, hi in ref:
        assert abs(float(w[lo:hi].sum()) - tot / world) < tot / world * 0.25


def test_move_plan_contiguous():
    old = [(0, 10), (10, 20), (20, 30)]
    new = [(0, 4), (4, 25), (25, 30)]
    assert rdist.move_plan(old, new, 0) == ([4, 6, 0], [4, 0, 0])
    assert rdist.move_plan(old, new, 1) == ([0, 10, 0], [6, 10, 5])
    assert rdist.move_plan(old, new, 2) == ([0, 5, 5], [0, 0, 5])


def _partner_fn(rank, world):
    """Counts only between listed pairs (NEXT(4)): the
    partner relation {(p, q): (p + 2 q) % 3 != 0}; the records received equal
    those of the all-to-all path, and a record for an unlisted writer is an
    error."""
    rel = {(p, q) for p in range(world) for q in range(world) if (p + 2 * q) % 3 != 0 or p == q}
    send_to = [q for q in range(world) if (rank, q) in rel]
    recv_from = [p for p in range(world) if (p, rank) in rel]
    counts = [(rank + 2 * d + 1) if (rank, d) in rel else 0 for d in range(world)]
    rows = [[rank, d, k, 0, 0, 0, 0, rank * 100 + d * 10 + k] for d in range(world) for k in range(counts[d])]
    send = torch.tensor(rows, dtype=torch.int32).reshape(-1, 8)
    tp = rdist.Transport()
    a = rdist.exchange_records(send, counts, tp, partners=(send_to, recv_from)).numpy()
    b = rdist.exchange_records(send, counts, tp).numpy()
    bad = list(counts)
    q_unlisted = next((q for q in range(world) if (rank, q) not in rel), None)
    raised = None
    if q_unlisted is not None:
        bad[q_unlisted] += 1
        try:
            rdist.partner_counts(bad, (send_to, recv_from), tp)
            raised = False
        except RuntimeError:
            raised = True
    return a, b, raised


def test_exchange_with_partners_gloo():
    out = _spawn(_partner_fn, 3)
    for rank, (a, b, raised) in out.items():
        assert np.array_equal(a, b)
        assert len(a) > 0
        assert raised in (None, True)


def _markers_fn(rank, world):
    import scenegen as sg
    sc = sg.shell_uniform(2, 16, 4)
    cuts = [0, 100, 100, sc.num_leaves]   # rank 1 holds no leaves
    lo, hi = cuts[rank], cuts[rank + 1]
    keys = (torch.as_tensor(sc.leaf_anchor[lo:hi]), torch.as_tensor(sc.leaf_tree[lo:hi]),
            torch.as_tensor(sc.leaf_level[lo:hi]))
    return rdist.partition_markers(keys, sc.num_trees, rdist.Transport())


def test_partition_markers_gloo():
    """dist.partition_markers (all-gathered first leaves) equals the oracle's
    markers of the same cuts, including an empty rank."""
    import scenegen as sg
    from oracle import partition as op
    sc = sg.shell_uniform(2, 16, 4)
    want = op.markers(sc, [0, 100, 100, sc.num_leaves])
    out = _spawn(_markers_fn, 3)
    for rank, mk in out.items():
        assert [op.sfc_key(t, a) for t, a in mk] == want
