"""Small frames through every kernel of librc, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): C1 64x64, C2 at 96x96
(levels 3..5), a level-2 cubed-sphere shell (curved R=2 path) with the on-chip
fold, one aggregation cycle, the tile pack and a two-rank tiled composite."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch

    import scenegen as sg
    from paper_1809_01334_b200 import rc
    for name, sc, fold, cycles in (("C1", sg.config1(), 0, 0),
                                   ("C2-96", sg.config2(width=96, maxlevel=5), 1, 1),
                                   ("shell-L2", sg.shell_uniform(2, 64, 16, gl_points=6), 2, 1)):
        f = rc.Forest.from_scene(sc)
        img, hits = f.render_frame(sc.camera, fold_levels=fold, cycles=cycles)
        raw, counts = f.pack_tiles(4, 4, 2, 0)
        offs = [0, counts[0], counts[0] + counts[1]]
        for r in range(2):
            f.composite_tiles(4, 4, 2, r, recv=raw[offs[r]:offs[r + 1]].clone())
        torch.cuda.synchronize()
        print(name, "hit pairs", hits, "records", f.segments()["count"], flush=True)
        f.close()
    print("sanitize frames done")
