"""Measure the FP32 pipe peaks on this GPU (tools/peaks.cu) with the SM clock
sampled during the run; writes profiles/peaks_r02.json (bench.py's roofline
peak).  Usage on the GPU box: python tools/peaks.py [out.json]"""
import datetime
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import bench
    exe = os.path.join(ROOT, "tools", "peaks")
    if not os.path.exists(exe):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe,
                               exe + ".cu"])
    with bench.Clocks(0) as clk:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    line["clocks"] = clk.summary()
    line["how"] = ("tools/peaks.cu: 8 independent chains per thread of fma.rn.f32 / ex2.approx.ftz.f32 / "
                   "min.f32+max.f32 (and fma.rn.f64 at 1/4 the iterations), 512 threads x 4 CTAs per SM on all SMs, ~10 ms launches, best of 20 (CUDA events)")
    line["when"] = datetime.datetime.utcnow().strftime("%Y-%m-%dT%H:%M:%SZ")
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "peaks_r02.json")
    json.dump(line, open(out, "w"), indent=1)
    print(json.dumps(line))
