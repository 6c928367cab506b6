"""NEXT(4) on the GPU:
librc's partner discovery from the partition markers (rc_exchange_partners)
against the oracle's traversal (oracle/partition.py), the records the ranks
actually exchange, and the vforest of several image instances
(rc_visible_area_add + rc_vforest_create) against the oracle's culls and
renders.  Index work is compared exactly (sets), within the eps-ambiguity
band of SURVEY R6 where a box edge lies within 1e-6 of a pixel centre."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import scenegen as sg
from oracle import partition as op
from paper_1809_01334_b200 import rc

pytestmark = pytest.mark.gpu


def _markers_api(scene, cuts):
    """rc_marker list of the cuts, from the leaves (the definition of)."""
    P = len(cuts) - 1
    out = [None] * (P + 1)
    out[P] = (scene.num_trees, (0, 0, 0))
    for p in range(P - 1, -1, -1):
        c = cuts[p]
        out[p] = (int(scene.leaf_tree[c]), tuple(int(x) for x in scene.leaf_anchor[c])) if c < cuts[p + 1] else out[p + 1]
    first = next((p for p in range(P) if cuts[p] < cuts[p + 1]), P)
    for p in range(min(first + 1, P)):
        out[p] = (0, (0, 0, 0))
    return out


def _cuts(n, P, seed):
    rng = np.random.default_rng(seed)
    c = np.sort(rng.choice(np.arange(1, n), size=P - 1, replace=False))
    return [0] + [int(x) for x in c] + [n]


SCENES = {
    "c1": lambda: sg.config1(width=32),
    "shell": lambda: sg.shell_uniform(2, 24, 4),
    "c2": lambda: sg.config2(width=64, maxlevel=5),
    "surface": lambda: sg.mandelbrot_hexagon(level0=2, maxlevel=4, max_iter=12, width=48),
}


@pytest.mark.parametrize("which", list(SCENES))
def test_partners_match_oracle_and_cover_records(which):
    sc = SCENES[which]()
    f = rc.Forest.from_scene(sc)
    f.camera_set(sc.camera)
    for P, tiles, seed in ((2, (2, 2), 1), (3, (4, 4), 2), (5, (4, 2), 3)):
        cuts = _cuts(sc.num_leaves, P, seed)
        mk = _markers_api(sc, cuts)
        m = op.markers(sc, cuts)
        own = lambda tx, ty: (tx + ty) % P
        sure = op.partner_relation(sc, m, tiles[0], tiles[1], own, eps=-1e-6)
        poss = op.partner_relation(sc, m, tiles[0], tiles[1], own, eps=1e-6)
        got, sent = set(), set()
        for r in range(P):
            send_to, recv_from = f.exchange_partners(tiles[0], tiles[1], P, r, mk)
            got |= {(p, r) for p in recv_from}
            sent |= {(r, q) for q in send_to}
        assert got == sent   # the sender side lists the same relation (DESIGN D19)
        assert sure <= got <= poss, (P, tiles, sure - got, got - poss)
        # every record a rank's leaves produce goes to a listed writer
        for r in range(P):
            lo, hi = cuts[r], cuts[r + 1]
            fr = rc.Forest.from_scene(sc, first=lo, count=hi - lo)
            fr.camera_set(sc.camera)
            fr.cull()
            fr.cast_segments(0)
            _, counts = fr.pack_tiles(tiles[0], tiles[1], P, r)
            send_to, _ = f.exchange_partners(tiles[0], tiles[1], P, r, mk, recv=False)
            assert {q for q in range(P) if counts[q]} <= set(send_to), (r, counts, send_to)
            fr.close()
    f.close()


def test_partners_markers_validated():
    sc = sg.config1(width=32)
    f = rc.Forest.from_scene(sc)
    with pytest.raises(rc.RcError):           # before rc_camera_set
        f.exchange_partners(2, 2, 2, 0, _markers_api(sc, [0, 100, sc.num_leaves]))
    f.camera_set(sc.camera)
    bad = _markers_api(sc, [0, 100, sc.num_leaves])
    bad[1], bad[0] = bad[0], bad[1]           # out of SFC order
    with pytest.raises(rc.RcError):
        f.exchange_partners(2, 2, 2, 0, bad)
    # single rank: it is its own only partner
    s, r = f.exchange_partners(2, 2, 1, 0, _markers_api(sc, [0, sc.num_leaves]))
    assert s == [0] and r == [0]
    f.close()


def _instances(sc):
    return [sg.perspective_camera((0.5, 0.5, 2.2), (0.5, 0.5, 0.5), 12.0, 48, 40, gl_points=4),
            sg.orthographic_camera((0.2, 0.3, 0.5), (1.0, 0.1, 0.05), 3.0, 0.35, 32, 32, gl_points=4)]


def test_vforest_of_instances_matches_oracle():
    """vforest leaves and weights against the oracle's
    per-instance culls; every instance rendered from the vforest equals the
    render of the whole forest (hits exactly, pixels to 1e-6) and the
    oracle's render (1e-4, the parity gate of the affine path)."""
    sc = sg.config2(width=64, maxlevel=5)
    cams = _instances(sc)
    f = rc.Forest.from_scene(sc)
    w = torch.zeros(f.n, dtype=torch.int64, device="cuda")
    for cam in cams:
        f.camera_set(cam)
        f.cull()
        f.visible_area_add(w)
    vf, m, wv = f.vforest(w, first_global_leaf=0)
    keep, wk, amb = op.vforest_leaves(sc, cams)
    got = torch.nonzero(w > 0).flatten().cpu().numpy()
    assert set(keep[~amb[keep]].tolist()) <= set(got.tolist()) <= set(keep.tolist()) | set(np.nonzero(amb)[0].tolist())
    assert m == got.size and 0 < m < sc.num_leaves
    wg = w.cpu().numpy()
    clean = np.array([not amb[e] for e in keep])
    assert np.array_equal(wg[keep[clean]], wk[clean])
    assert np.array_equal(wv.cpu().numpy(), wg[got])
    # the vforest's leaves are the kept rows in SFC order
    rows = vf.leaves()
    assert np.array_equal(rows[1].cpu().numpy(), sc.leaf_tree[got])
    assert np.array_equal(rows[0].cpu().numpy(), sc.leaf_anchor[got])
    assert np.array_equal(rows[3].cpu().numpy(), sc.leaf_field[got])
    for cam in cams:
        img_v, hits_v = vf.render_frame(cam)
        img_f, hits_f = f.render_frame(cam)
        assert hits_v == hits_f
        assert np.array_equal(vf.segments()["hits_per_pixel"].cpu().numpy(), f.segments()["hits_per_pixel"].cpu().numpy())
        assert float((img_v - img_f).abs().max()) < 1e-6
        ref = oracle.OracleScene(dataclasses.replace(sc, camera=cam)).render(mode="rule", with_hits=False)
        assert float(np.abs(img_v.cpu().numpy().reshape(-1, 4) - ref["rgba"]).max()) < 1e-4
    vf.close()
    # nothing visible: no vforest
    z = torch.zeros(f.n, dtype=torch.int64, device="cuda")
    vf0, m0, _ = f.vforest(z)
    assert vf0 is None and m0 == 0
    f.close()


def test_comm_partners_single_rank_nccl():
    """rc_comm_set_partners on a one-rank NCCL communicator: the composite
    runs the partner count exchange and equals rc_composite bit for bit."""
    import socket
    import torch.distributed as dist
    from paper_1809_01334_b200 import dist as rdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sc = sg.shell_uniform(2, 32, 4)
        f = rc.Forest.from_scene(sc)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(1)
        ref = f.composite().cpu().numpy()
        comm = rc.Comm(1, 0)
        snd, rcv = f.exchange_partners(2, 2, 1, 0, _markers_api(sc, [0, sc.num_leaves]))
        assert snd == [0] and rcv == [0]
        comm.set_partners(snd, rcv)
        out, mine = f.composite_tiles(2, 2, 1, 0, comm=comm)
        torch.cuda.synchronize()
        img = rdist.assemble_image({0: (out, mine)}, 2, 2, 32, 32).numpy()
        assert np.array_equal(img.view(np.uint32), ref.view(np.uint32))
        comm.set_partners()
        comm.close()
        f.close()
    finally:
        dist.destroy_process_group()
