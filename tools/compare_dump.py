"""Compare a gpu_dump npz with the oracle pair by pair; print mismatches."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import oracle
from gpu_dump import SCENES

name = sys.argv[1]
d = np.load(f"gpurun_out/dump_{name}.npz")
sc = SCENES[name]()
o = oracle.OracleScene(sc)
W = sc.camera.width
raw = d["raw"]; f = raw.view(np.float32)
pix = raw[:, 0].astype(np.int64); key = raw[:, 7].astype(np.int64)
res = o.render(mode="exact", cap=256)
gsets = {}
for p, k, an, af in zip(pix, key, f[:, 1], f[:, 2]):
    gsets.setdefault(int(p), []).append((int(k), float(an), float(af)))
miss, extra = [], []
for q in range(W * W):
    h = res["hits"][q]; h = h[h["elem"] >= 0]
    amb = set(h["elem"][(h["flags"] & 2) != 0].tolist())
    oh = {int(r["elem"]): (r["alpha_near"], r["alpha_far"]) for r in h if r["flags"] & 1}
    gh = {k: (a, b) for k, a, b in gsets.get(q, [])}
    for e in set(oh) - set(gh) - amb:
        miss.append((q % W, q // W, e, oh[e]))
    for e in set(gh) - set(oh) - amb:
        extra.append((q % W, q // W, e, gh[e]))
print("missed", len(miss), "extra", len(extra), "nf", d["nf"])
for m in miss[:12]:
    i, j, e, (a0, a1) = m
    ro, rd = o.ray(i, j)
    seg, fl = o.intersect(e, i, j)
    print("MISS", i, j, e, "orc", seg.tolist(), "chord", ((seg[:, 1] - seg[:, 0]) * np.linalg.norm(rd)).tolist())
for m in extra[:8]:
    print("EXTRA", m)
err = np.abs(d["rgba"] - res["rgba"]).max(axis=1)
print("max err", err.max(), "bad>1e-4", (err > 1e-4).sum())
