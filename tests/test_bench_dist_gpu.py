"""bench.py's multi-GPU code path with two ranks on the one
GPU of the test box: torchrun with --dist-backend gloo (host-staged
exchanges; no kernel waits on another rank's).  Covers the pre-partition
(rc_leaf_weights, the collective weighted cut aligned to node starts, the
leaf move), the coarsening cycles with repartition between them
(rc_segments_set on keys-only forests), the tile exchange and the composite
of the owners, the max-over-ranks timing and the e2e leg.  The assembled
image and the per-pixel hit counts must equal the one-rank run."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(tmp, world, extra):
    dump = os.path.join(tmp, f"img{world}.npz")
    args = ["bench.py", "--gpus", str(world), "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
            "--dump", dump] + extra
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args + ["--dist-backend", "gloo"]
    else:
        cmd = [sys.executable] + args
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    return line, np.load(dump)


@pytest.mark.parametrize("extra", [["--config", "33", "--fold", "1"], ["--config", "33", "--fold", "0"],
                                   ["--config", "33", "--fold", "1", "--instances", "2"],
                                   ["--config", "33", "--fold", "0", "--prepartition", "leaves", "--all-to-all"]])
def test_bench_two_ranks_equal_one_rank(tmp_path, extra):
    """Default N > 1 path: vforest pre-partition of every instance's visible
    leaves and partners from the partition markers (NEXT(4)); --prepartition
    leaves --all-to-all: round 1's path (every leaf weighted, count all-to-all)."""
    l1, d1 = _bench(str(tmp_path), 1, extra)
    l2, d2 = _bench(str(tmp_path), 2, extra)
    assert l2["n_gpus"] == 2 and l2["config"]["dist_backend"] == "gloo"
    assert l2["config"]["hit_pairs"] == l1["config"]["hit_pairs"] == int(d1["hit_pairs"])
    ni = int(d1["instances"])
    assert ni == l2["config"]["instances"] == (2 if "--instances" in extra else 1)
    for k in range(ni):
        sfx = "" if k == 0 else f"_{k}"
        assert np.array_equal(d1["hits_per_pixel" + sfx], d2["hits_per_pixel" + sfx]), k
        # lossless folds / aggregation: equal up to the fp32 records
        assert np.abs(d1["image" + sfx] - d2["image" + sfx]).max() < 1e-5, k
    ranges = d2["ranges"]
    part = l2["partition"]
    n_part = part["vforest_leaves"]
    assert ranges[0][0] == 0 and ranges[-1][1] == n_part and ranges[0][1] == ranges[1][0]
    if "--prepartition" in extra:
        assert part["prepartition"] == "leaves" and n_part == l1["config"]["leaves"]
    else:
        assert part["prepartition"] == "vforest" and 0 < n_part <= l1["config"]["leaves"]
    if "--all-to-all" in extra:
        assert part["partners_rank0"] is None
    else:
        send_to, recv_from = part["partners_rank0"][0]
        assert 0 in recv_from or 0 in send_to or send_to or recv_from
    assert l2["e2e"]["value"] > 0 and l2["gpu_launches"] > 0
