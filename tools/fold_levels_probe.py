"""Records after the on-chip fold at several fold levels, and the aggregation
time to the same final level (C5 / C5s).  python tools/fold_levels_probe.py CONFIG FINAL_LEVEL"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch

    import bench
    from paper_1809_01334_b200 import rc
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 55
    final = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    sc = bench.make_scene(cfg, torch.device("cuda"))
    f = rc.Forest.from_scene(sc, device_copy=True)
    sc = bench.scene_to_host(sc)
    torch.cuda.empty_cache()
    for fold in (2, 3, 4):
        for rep in range(2):
            f.camera_set(sc.camera)
            f.cull()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f.cast_segments(fold)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            n0 = f.segments()["count"]
            f.aggregate(final - fold)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
        s = f.segments()
        print(f"fold {fold}: cast {1e3 * (t1 - t0):.1f} ms, records {n0}, aggregate to level {final}: "
              f"{1e3 * (t2 - t1):.1f} ms, records {s['count']}, raw {s['raw_segments']}, units {s['units']}",
              flush=True)
