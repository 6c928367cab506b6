"""C5 memory / count probe: generate C5 on the GPU, cast with fold 2, report
record counts and device memory before and after each step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch
    import bench
    from paper_1809_01334_b200 import rc
    gb = lambda: "free %.1f GB" % (torch.cuda.mem_get_info()[0] / 1e9)
    t0 = time.time()
    sc = bench.make_scene(5, torch.device("cuda"))
    print("scene", sc.num_leaves, "leaves", "%.1fs" % (time.time() - t0), gb(), flush=True)
    f = rc.Forest.from_scene(sc, device_copy=True)
    sc = bench.scene_to_host(sc)
    torch.cuda.empty_cache()
    print("forest", gb(), flush=True)
    f.camera_set(sc.camera)
    f.cull()
    f.cast_segments(2)
    s = f.segments()
    print("cast fold2: records", s["count"], "raw", s["raw_segments"], "hits", s["hit_pairs"], "cand", s["candidates"],
          "units", s["units"], "unfolded", s["unfolded_units"], "ms", f.last_cast_ms(), gb(), flush=True)
    f.aggregate(3)
    s = f.segments()
    print("aggregate 3: records", s["count"], "level", s["level"], gb(), flush=True)
    img = f.composite()
    torch.cuda.synchronize()
    print("composite ok", gb(), flush=True)
