"""Where does the composite phase's time go?  Per frame: device times of the
phase (bench events), of the bucketing and fold kernels (library events), and
host times of the composite call, at C4."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch
    import bench
    from paper_1809_01334_b200 import rc
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    sc = bench.make_scene(cfg, torch.device("cuda"))
    f = rc.Forest.from_scene(sc, device_copy=True)
    sc = bench.scene_to_host(sc)
    torch.cuda.empty_cache()
    img = torch.empty((sc.camera.height, sc.camera.width, 4), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for it in range(8):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        f.camera_set(sc.camera)
        f.cull()
        f.cast_segments(2)
        ev[0].record(st)
        t0 = time.perf_counter()
        f.composite(out=img)
        t1 = time.perf_counter()
        ev[1].record(st)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"frame {it}: composite device {ev[0].elapsed_time(ev[1]):.2f} ms, bucket {f.last_phase_ms(4):.2f}, "
              f"fold {f.last_phase_ms(5):.2f}, host call {1e3 * (t1 - t0):.2f} ms, host to idle {1e3 * (t2 - t0):.2f} ms",
              flush=True)
