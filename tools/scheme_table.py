"""Cost / accuracy table of the paper's segment integrators on the GPU
(PAPER.md:660-778): for every scheme and c_RK, the
segment kernel's device time on a full-size config, the max |RGBA - oracle
exact| on a stratified pixel sample, and the oracle's field evaluations per
segment in the same scheme (the cost unit the paper's schemes trade).
Usage on the GPU box: python tools/scheme_table.py [CONFIG] [KAPPA_SCALE] [out.json]"""
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ROWS = [("gl", 0.0, 2), ("gl", 0.0, 4), ("gl", 0.0, 6), ("gl", 0.25, 4), ("gl", 0.1, 4),
        ("euler", 0.1, 0), ("euler", 0.05, 0), ("heun2", 0.25, 0), ("heun2", 0.1, 0), ("heun3", 0.25, 0),
        ("rk4", 0.5, 0), ("rk4", 0.25, 0), ("gauss2", 0.5, 0), ("gauss2", 0.25, 0), ("simpson", 0.5, 0),
        ("simpson", 0.25, 0)]

if __name__ == "__main__":
    import numpy as np
    import torch

    import bench
    import oracle
    from paper_1809_01334_b200 import rc
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    ks = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    out_path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"scheme_table_c{cfg}.json")
    sc = bench.make_scene(cfg, torch.device("cuda"))
    sc = dataclasses.replace(sc, kappa0=sc.kappa0 * ks)
    f = rc.Forest.from_scene(sc, device_copy=True)
    host = bench.scene_to_host(sc)
    W, H = sc.camera.width, sc.camera.height
    stride = {1: 2, 2: 8, 3: 32, 45: 32}.get(cfg, 16)
    jj, ii = np.meshgrid(np.arange(stride // 2, H, stride), np.arange(stride // 2, W, stride), indexing="ij")
    pix = (jj * W + ii).ravel().astype(np.int32)
    o = oracle.OracleScene(host)
    _, _, rects = o.cull()
    ref = o.render_pairs(pix, mode="exact", rects=rects)
    fold = 0 if cfg <= 2 else 2
    rows = []
    for scheme, c_rk, N in ROWS:
        cam = dataclasses.replace(sc.camera, gl_points=N or sc.camera.gl_points)
        times = []
        for rep in range(3):
            f.camera_set(cam, scheme=scheme, c_rk=c_rk)
            f.cull()
            f.cast_segments(fold)
            times.append(f.last_cast_ms())
        s = f.segments()
        img = f.composite().cpu().numpy().reshape(-1, 4)
        err = float(np.abs(img[pix] - ref["rgba"]).max())
        oracle.set_scheme(scheme, c_rk)
        oracle.medium_evals(reset=True)
        osub = o.render_pairs(pix[::8], mode="scheme", N=N or sc.camera.gl_points, rects=rects)
        evals = oracle.medium_evals()
        oracle.set_scheme("gl", 0.0)
        nseg = max(1, int(osub["total_hits"]))
        row = dict(scheme=scheme, c_rk=c_rk, gl_points=N or None, kernel_ms=sorted(times)[1],
                   max_err_vs_exact=err, field_evals_per_hit_pair=evals / nseg, depth_capped=int(s["depth_capped"]),
                   hit_pairs=int(s["hit_pairs"]))
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"config": bench.WORKLOAD.get(cfg, str(cfg)), "kappa_scale": ks, "sample_stride": stride,
               "rows": rows}, open(out_path, "w"), indent=1)
