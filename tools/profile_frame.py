"""Minimal frame driver for ncu: build the scene, run `--frames` frames."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--frames", type=int, default=2)
    a = ap.parse_args()
    import torch
    import bench
    from paper_1809_01334_b200 import rc
    sc = bench.make_scene(a.config, torch.device("cuda"))
    f = rc.Forest.from_scene(sc, device_copy=True)
    sc = bench.scene_to_host(sc)
    torch.cuda.empty_cache()
    for _ in range(a.frames):
        img, hits = f.render_frame(sc.camera, fold_levels=(0 if a.config <= 2 else 2), cycles=sc.coarsen_cycles)
    if a.config == 55:   # the aggregation pass alone, for ncu -k k_coarsen (records of the last cast)
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(2)
        f.aggregate(sc.coarsen_cycles)
    torch.cuda.synchronize()
    s = f.segments()
    print("hit_pairs", hits, "candidates", s["candidates"], "records", s["count"], "raw", s["raw_segments"],
          "newton_failures", s["newton_failures"], "face_failures", s["face_failures"], "fallback_tasks",
          s["fallback_tasks"], "unfolded_units", s["unfolded_units"], "cast_ms", f.last_cast_ms())
