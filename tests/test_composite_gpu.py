"""GPU tests of row a9 (tile composite) on hand-built records, and of the
determinism of the folds (rows a6, a7, a9).

* Overlap clusters (Eq. segsplit / segaverage; DESIGN.md
  D14): the hand-evaluated cases of tests/golden/overlap_cases.txt, and random
  records with overlapping, nested, identical, touching, A = 1 and opaque
  segments, go through rc_composite_tiles(d_recv = ...) and are compared with
  the oracle's orc_fold_pixel on the same fp32 records.  Interval end points
  are multiples of 1/64 (exact in fp32), so the GPU's 1e-6 and the oracle's
  tolerance classify every pair the same way.
* Determinism: two casts of one forest (and of a fresh forest) give the same
  records (as a multiset, bit for bit) and bit-identical RGBA."""
import math
import os
import sys

import numpy as np
import pytest

import oracle
import scenegen as sg

sys.path.insert(0, os.path.dirname(__file__))
from test_oracle_pins import load_overlap_cases  # noqa: E402

pytestmark = pytest.mark.gpu


def _records(rows):
    """rows: [(pixel, an, af, a, b0, b1, b2, key)] -> int32 tensor [n, 8] (rc_seg)."""
    import torch
    arr = np.zeros((len(rows), 8), dtype=np.float32)
    raw = arr.view(np.int32)
    for k, (p, an, af, a, b0, b1, b2, key) in enumerate(rows):
        arr[k, 1:7] = (an, af, a, b0, b1, b2)
        raw[k, 0] = p
        raw[k, 7] = key
    return torch.from_numpy(raw.copy()).cuda()


def _composite(recs, W=32, H=32):
    from paper_1809_01334_b200 import rc
    sc = sg.config1(width=W)
    f = rc.Forest.from_scene(sc)
    f.camera_set(sc.camera)
    img, _ = f.composite_tiles(1, 1, 1, 0, recv=recs)
    return img.cpu().numpy().reshape(-1, 4)


def _oracle_pixel(rows, tau):
    h = np.zeros(len(rows), dtype=oracle.HIT_DTYPE)
    for k, (p, an, af, a, b0, b1, b2, key) in enumerate(rows):
        h[k]["elem"] = key
        h[k]["pixel"] = p
        h[k]["flags"] = oracle.HIT
        # the fp32 values the GPU sees
        h[k]["alpha_near"], h[k]["alpha_far"], h[k]["a"] = np.float32(an), np.float32(af), np.float32(a)
        h[k]["b"] = np.float32([b0, b1, b2])
    rgba, _ = oracle.fold_pixel(h, tau=tau)
    return rgba


@pytest.mark.parametrize("case", load_overlap_cases(), ids=lambda c: c[0])
def test_overlap_golden_cases_gpu(case):
    name, h, (A, B) = case
    rows = [(5, float(s["alpha_near"]), float(s["alpha_far"]), float(s["a"]), float(s["b"][0]),
             float(s["b"][1]), float(s["b"][2]), k) for k, s in enumerate(h)]
    img = _composite(_records(rows[::-1]))
    # rgba = (B, B, B, 1 - A) with I_b = 0
    assert np.abs(img[5, :3] - B).max() < 2e-6 and abs(img[5, 3] - (1 - A)) < 2e-6, (name, img[5], A, B)
    assert np.all(img[np.arange(img.shape[0]) != 5] == np.array([0, 0, 0, 0], np.float32))


@pytest.mark.parametrize("nmax", [12, 200, 700])
def test_overlap_random_clusters_vs_oracle(nmax):
    """Random pixels with up to nmax records each: register path (<= 512
    records) and list path (> 512), with and without overlaps."""
    rng = np.random.default_rng(nmax)
    W = 32
    rows, per_pix = [], {}
    for p in range(W * W):
        kind = p % 4
        n = int(rng.integers(0, nmax + 1))
        recs = []
        x = 1.0 + rng.integers(0, 64) / 64.0
        for k in range(n):
            if kind == 0:        # disjoint or touching chain (no overlap)
                an = x + (rng.integers(0, 2) / 64.0)
                af = an + rng.integers(1, 8) / 64.0
                x = af
            else:                # overlapping clusters, nested and identical intervals
                an = 1.0 + rng.integers(0, 8 * max(n, 8)) / 64.0
                af = an + rng.integers(0 if kind == 3 else 1, 40) / 64.0
                if kind == 2 and k > 0 and rng.random() < 0.3:
                    an, af = recs[-1][1], recs[-1][2]          # identical interval
            a = 1.0 if rng.random() < 0.1 else float(rng.uniform(0.05, 1.0))
            if rng.random() < 0.02:
                a = 0.0                                          # opaque
            b = rng.uniform(0.0, 0.5, 3)
            recs.append((p, an, af, a, float(b[0]), float(b[1]), float(b[2]), 1000 * p + k))
        per_pix[p] = recs
        rows.extend(recs)
    rng.shuffle(rows)
    img = _composite(_records(rows), W=W, H=W)
    worst = 0.0
    for p in range(W * W):
        ref = _oracle_pixel(per_pix[p], tau=1e-6) if per_pix[p] else np.zeros(4)
        worst = max(worst, float(np.abs(img[p] - ref).max()))
    assert worst < 5e-6, worst


def _sorted_records(raw):
    r = raw.cpu().numpy()
    keys = np.lexsort(tuple(r[:, c] for c in range(7, -1, -1)))
    return r[keys]


@pytest.mark.parametrize("fold,cycles", [(0, 0), (2, 0), (2, 1), (1, 3)])
def test_fold_and_composite_deterministic(fold, cycles):
    """Records (as a multiset) and RGBA are bit-identical across casts of the
    same forest and across forests (the atomics that schedule the work do not
    reach the results)."""
    from paper_1809_01334_b200 import rc
    sc = sg.shell_uniform(3, 96, 16, gl_points=6)
    out = []
    for rep in range(3):
        f = rc.Forest.from_scene(sc) if rep != 1 else f
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(fold)
        if cycles:
            f.aggregate(cycles)
        s = f.segments()
        img = f.composite().cpu().numpy().copy()
        out.append((s["count"], _sorted_records(s["raw"]), img))
    for cnt, recs, img in out[1:]:
        assert cnt == out[0][0]
        assert np.array_equal(recs, out[0][1])
        assert np.array_equal(img.view(np.uint32), out[0][2].view(np.uint32))


def test_comm_single_rank_nccl_exchange():
    """rc_comm over NCCL with one rank: rc_composite_tiles(comm) packs on the
    device, exchanges the counts and the records through NCCL (the self block
    is a device copy) and composites; equals the local composite bit for bit."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1809_01334_b200 import rc
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sc = sg.shell_uniform(3, 96, 16, gl_points=6)
        f = rc.Forest.from_scene(sc)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(2)
        ref = f.composite().cpu().numpy()
        comm = rc.Comm(1, 0)
        out, mine = f.composite_tiles(4, 4, 1, 0, comm=comm)
        torch.cuda.synchronize()
        from paper_1809_01334_b200 import dist as rdist
        img = rdist.assemble_image({0: (out, mine)}, 4, 4, 96, 96).numpy()
        assert np.array_equal(img.view(np.uint32), ref.view(np.uint32))
        with pytest.raises(rc.RcError):
            f.composite_tiles(4, 4, 2, 1, comm=comm)      # tiling ranks != communicator
        comm.close()
    finally:
        dist.destroy_process_group()


def test_debug_pair_matches_cast():
    """rc_debug_pair evaluates one (leaf, pixel) pair with the frame's segment
    kernel: equals the fold-0 records of that pair, and misses give none."""
    from paper_1809_01334_b200 import rc
    for sc in (sg.config2(width=64, maxlevel=5), sg.shell_uniform(2, 48, 8, gl_points=6)):
        f = rc.Forest.from_scene(sc)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(0)
        raw = f.segments()["raw"].cpu().numpy()
        W = sc.camera.width
        rng = np.random.default_rng(0)
        for k in rng.choice(raw.shape[0], 40, replace=False):
            p, e = int(raw[k, 0]), int(raw[k, 7])
            mine = raw[(raw[:, 0] == p) & (raw[:, 7] == e)].view(np.float32)
            mine = mine[np.argsort(mine[:, 1])]
            got = f.debug_pair(e, p % W, p // W)
            assert len(got) == mine.shape[0]
            for (an, af, a, b), r in zip(got, mine):
                assert (an, af, a) == (r[1], r[2], r[3]) and tuple(b) == tuple(r[4:7])
        # a pixel no ray hits anything at: no segment
        hpp = f.segments()["hits_per_pixel"].cpu().numpy().reshape(-1)
        empty = int(np.nonzero(hpp == 0)[0][0])
        assert f.debug_pair(int(raw[0, 7]), empty % W, empty // W) == []


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_graph_frame_replay_equals_frame(which):
    """rc_frame_capture / rc_frame_replay (CUDA-graph frames of affine forests,
    SURVEY §8(d)): every replay writes the same image as the ordinary frame,
    bit for bit, and the oracle's within the gate."""
    import torch
    from paper_1809_01334_b200 import rc
    sc = sg.config1() if which == "c1" else sg.config2(width=96, maxlevel=5)
    f = rc.Forest.from_scene(sc)
    ref, hits = f.render_frame(sc.camera)
    ref = ref.cpu().numpy().copy()
    img = f.frame_capture(sc.camera)
    torch.cuda.synchronize()
    for _ in range(3):
        img.zero_()
        f.frame_replay()
        torch.cuda.synchronize()
        assert np.array_equal(img.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert f.segments()["hit_pairs"] == hits
    o = oracle.OracleScene(sc)
    ores = o.render(mode="exact", with_hits=False)
    clean = ores["namb"] == 0
    assert np.abs(img.cpu().numpy().reshape(-1, 4)[clean] - ores["rgba"][clean]).max() < 1e-4


def test_device_borrow_equals_copy():
    """RC_DEVICE_BORROW: the forest renders from the caller's
    device arrays in place (levels copied) and gives the copy forest's image
    and records bit for bit; the binding keeps the arrays alive."""
    import gc
    import torch
    from paper_1809_01334_b200 import rc
    for sc, fold in ((sg.config2(width=64, maxlevel=5), 0), (sg.shell_uniform(2, 48, 8, gl_points=6), 2)):
        fb = rc.Forest.from_scene(sc, borrow=True)
        gc.collect()
        fc = rc.Forest.from_scene(sc, device_copy=True)
        ib, hb = fb.render_frame(sc.camera, fold_levels=fold)
        ic, hc = fc.render_frame(sc.camera, fold_levels=fold)
        torch.cuda.synchronize()
        assert hb == hc and torch.equal(ib, ic)
        rb, rcp = fb.segments()["raw"], fc.segments()["raw"]
        assert torch.equal(rb[:, 0].sort().values, rcp[:, 0].sort().values)
        fb.close()
        fc.close()
