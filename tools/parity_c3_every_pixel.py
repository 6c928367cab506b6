"""Parity evidence run (not part of the default GPU suite: ~1 h of oracle time on
the box's 16 host cores): BASELINE C3 at full size (1,572,864 curved hexes,
1024^2, N = 6) with gates 1-3 on EVERY pixel, in pixel blocks so the oracle's
pair lists stay small.  Gate 1: the full culled list; gate 2: the hit-element
set of every pixel (fold 0, exact within the eps-ambiguous pairs); gate 3:
RGBA of the fold-0 run and of the bench's configuration (fold level 2)
against the oracle's exact-mode pixels at 1e-4.  Prints one JSON line.

  python tools/parity_c3_every_pixel.py [--blocks 16]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=16)
    a = ap.parse_args()
    import bench
    import oracle
    import scenegen as sg
    from parity_util import gate_cull, gate_pairs, gate_rgba, gpu_pairs, gpu_run, oracle_pairs
    sc = sg.config3(device="cuda")
    W, H = sc.camera.width, sc.camera.height
    t0 = time.time()
    g = gpu_run(sc, device_copy=True)
    g2 = gpu_run(sc, device_copy=True, fold=2, keep_raw=False)
    o = oracle.OracleScene(bench.scene_to_host(sc))
    allpix = np.arange(W * H, dtype=np.int32)
    tot = dict(pair_mismatch=0, hit_mismatch_pixels=0, bad_pixels=0, bad_pixels_fold2=0, ambiguous_pairs=0,
               oracle_hits=0, max_abs=0.0, max_abs_fold2=0.0, cull_mismatch=None)
    vis, amb, rects = o.cull()   # the full culled list, once (gate 1)
    tot["cull_mismatch"] = gate_cull(g["visible"], vis, amb)
    tot["cull_ambiguous"] = int(amb.sum())
    for k, pixels in enumerate(np.array_split(allpix, a.blocks)):
        ores = o.render_pairs(pixels, mode="exact", rects=rects)
        okeys, akeys = oracle_pairs(ores)
        gkeys = gpu_pairs(g["raw"], pixels, W * H)
        nbad, nbadpix = gate_pairs(gkeys, okeys, akeys)
        r0 = gate_rgba(g["rgba"], pixels, ores)
        r2 = gate_rgba(g2["rgba"], pixels, ores)
        tot["pair_mismatch"] += nbad
        tot["hit_mismatch_pixels"] += nbadpix
        tot["ambiguous_pairs"] += int(akeys.size)
        tot["oracle_hits"] += int(okeys.size)
        tot["bad_pixels"] += r0["bad_pixels"]
        tot["bad_pixels_fold2"] += r2["bad_pixels"]
        tot["max_abs"] = max(tot["max_abs"], r0["max_err"])
        tot["max_abs_fold2"] = max(tot["max_abs_fold2"], r2["max_err"])
        print(f"block {k}: {pixels.size} pixels, {okeys.size} oracle hits, pair mismatches {nbad}, "
              f"bad pixels {r0['bad_pixels']} / {r2['bad_pixels']}, {time.time() - t0:.0f} s", flush=True)
    tot.update(pixels=int(allpix.size), gpu_hit_pairs=int(g["hit_pairs"]), newton_failures=int(g["newton_failures"]),
               fold2_records=int(g2["count"]), seconds=time.time() - t0,
               hits_per_pixel_equal=bool(np.array_equal(g2["hits_per_pixel"], g["hits_per_pixel"])))
    print(json.dumps(tot), flush=True)
    ok = (tot["cull_mismatch"] == 0 and tot["hit_mismatch_pixels"] == 0 and tot["bad_pixels"] == 0
          and tot["bad_pixels_fold2"] == 0 and tot["newton_failures"] == 0 and tot["hits_per_pixel_equal"])
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
