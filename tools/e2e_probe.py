"""Where does the e2e time go (forest creation from pinned host buffers vs the frame)?"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1809_01334_b200 import rc
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
sc = bench.make_scene(cfg, dev)
sc = bench.scene_to_host(sc)
torch.cuda.empty_cache()
host = [np.ascontiguousarray(a) for a in (sc.leaf_anchor, sc.leaf_tree, sc.leaf_level, sc.leaf_field)]
pinned = [torch.from_numpy(a).pin_memory().numpy() for a in host]
fold = 2
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = rc.Forest(sc.tree_ctrl, sc.geom_degree, sc.field_degree, *pinned, sc.kappa0, sc.inv_F, sc.q0, trusted=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    img, hits = f.render_frame(sc.camera, fold_levels=fold, cycles=sc.coarsen_cycles)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    img2, hits = f.render_frame(sc.camera, fold_levels=fold, cycles=sc.coarsen_cycles)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out = img2.cpu()
    t4 = time.perf_counter()
    f.close()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"it {it}: create {1e3*(t1-t0):.0f} ms, frame1 {1e3*(t2-t1):.0f} ms, frame2 {1e3*(t3-t2):.0f} ms, d2h {1e3*(t4-t3):.0f} ms, close {1e3*(t5-t4):.0f} ms", flush=True)
