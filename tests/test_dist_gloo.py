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


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
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
    recv = rdist.exchange_records(send, counts)
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
    recv = rdist.exchange_records(send, counts).numpy()
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
