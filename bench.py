"""Benchmark of the raycasting hot path (BASELINE.json metric: element-ray
segment evaluations/s and ms/frame; % of the FP32 roofline).

One step = one frame: rc_camera_set + rc_cull + rc_cast_segments
(+ rc_aggregate) + composite on seeded synthetic inputs already resident in
HBM.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_LANES_PER_SM = 128
NUM_SMS = 148


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        mp = {}
    sm_mhz = float(mp.get("sm_max_mhz", 1965.0))
    fp32 = NUM_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    return dict(fp32_tflops=fp32, hbm_gbs=float(mp.get("hbm_gbs", 6650.0)), sm_mhz=sm_mhz,
                source="MEASURED_PEAKS.json sm_max_mhz x 148 SM x 128 FP32 lanes x 2 (guide unit counts)"
                if mp else "fallback 1965 MHz (B200_PROFILING.md)")


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_scene(cfg: int, device):
    import scenegen as sg
    if cfg == 1:
        return sg.config1()
    if cfg == 2:
        return sg.config2(device=device)
    if cfg == 3:
        return sg.config3(device=device)
    if cfg == 4:
        return sg.config4(device=device)
    if cfg == 5:
        return sg.config5(device=device)
    if cfg == 45:   # profiling stand-in for C4: level 7 at 1024^2 has C4's pixels per element
        return sg.shell_uniform(7, 1024, 256, name="C4s", device=device)
    raise ValueError(cfg)


WORKLOAD = {1: "C1: identity cube, uniform level 3 (512 hex), ortho 64x64, N=4",
            2: "C2: identity cube, adaptive levels 3..7 (87,088 hex), perspective 512x512, N=4",
            3: "C3: cubed-sphere shell R=2, uniform level 6 (1,572,864 hex), 1024x1024, N=6",
            4: "C4: cubed-sphere shell R=2, uniform level 8 (100,663,296 hex), 2048x2048, N=6",
            5: "C5: cubed-sphere shell R=2, adaptive levels 6..10, 4096x4096, N=8, 3 coarsening cycles",
            45: "C4s (profiling stand-in): shell R=2, uniform level 7 (12,582,912 hex), 1024x1024, N=6"}


def forest_affine(scene):
    return scene.name.startswith(("C1", "C2"))


def scene_to_host(scene):
    import dataclasses
    import numpy as np
    def h(a):
        return a if isinstance(a, np.ndarray) else a.detach().cpu().numpy()
    return dataclasses.replace(scene, leaf_anchor=h(scene.leaf_anchor), leaf_tree=h(scene.leaf_tree),
                               leaf_level=h(scene.leaf_level), leaf_field=h(scene.leaf_field))


def l2_flush(buf):
    buf.add_(1.0)


def cpu_baseline(scene, stride, threads=0):
    """The oracle as it stands (exact mode) on every `stride`-th pixel row/column."""
    import numpy as np

    import oracle
    o = oracle.OracleScene(scene)
    W, H = scene.camera.width, scene.camera.height
    jj, ii = np.meshgrid(np.arange(stride // 2, H, stride), np.arange(stride // 2, W, stride), indexing="ij")
    pix = (jj * W + ii).ravel().astype(np.int32)
    t0 = time.perf_counter()
    res = o.render(pix, mode="exact", with_hits=False, nthreads=threads)
    dt = time.perf_counter() - t0
    cores = threads or (os.cpu_count() or 1)
    return dict(value=res["total_hits"] / dt, unit="hit pairs/s", cores=cores, kind="oracle",
                sample=f"every {stride}th pixel row and column ({pix.size} pixels, {res['total_hits']} hit pairs), "
                       f"all {scene.num_leaves} leaves culled; fp64 exact mode; {dt:.1f} s wall",
                seconds=dt, hit_pairs=res["total_hits"])


def run_reference(args):
    """--impl reference: the fp64 oracle timed as it stands on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    dev = "cuda" if (args.config >= 3 and torch.cuda.is_available()) else None
    scene = scene_to_host(make_scene(args.config, dev))
    # each step a bounded sample (~5-15 s of host work) so that --steps K ends within minutes
    stride = {1: 1, 2: 16, 3: 64, 4: 128, 5: 256, 45: 64}[args.config]
    for _ in range(args.warmup):
        pass
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(scene, stride))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    line = {"impl": "reference", "metric": "element-ray segment evaluations/s (hit pairs/s)", "value": v,
            "unit": "hit pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * statistics.median([x["seconds"] for x in vals]),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD[args.config], "sample_stride": stride},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": "hit pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=int(os.environ.get("RC_BENCH_CONFIG", "4")))
    ap.add_argument("--impl", default="rc")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (A/B runs of build variants)")
    ap.add_argument("--fold", type=int, default=-1,
                    help="node level of the on-chip fold (row a6); default 2 for curved forests, 0 for affine")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_1809_01334_b200 import rc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    scene = make_scene(args.config, dev if args.config >= 2 else None)
    cam = scene.camera
    W, H = cam.width, cam.height
    N = cam.gl_points
    lib = rc.lib()

    fold = args.fold if args.fold >= 0 else (0 if forest_affine(scene) else 2)
    # --- device-resident inputs: this rank's contiguous SFC range ---------
    # equal leaf counts, cuts moved to node starts of the coarsest level the
    # fold + aggregation cycles reach: every family is local
    n = scene.num_leaves
    if world > 1:
        from paper_1809_01334_b200 import dist as rdist
        A, T, Lv = (torch.as_tensor(x, device=dev) for x in (scene.leaf_anchor, scene.leaf_tree, scene.leaf_level))
        allowed = rdist.node_starts(A, T, Lv, fold + scene.coarsen_cycles)
        lo, hi = rdist.aligned_ranges(torch.ones(n, dtype=torch.float64), world, allowed)[rank]
        del A, T, Lv, allowed
    else:
        lo, hi = 0, n
    forest = rc.Forest.from_scene(scene, first=lo, count=hi - lo, device_copy=True)
    # the forest holds its own device copy: keep the scene on the host only
    # (e2e inputs, CPU baseline) and hand the generator's memory back (C5 needs it)
    scene = scene_to_host(scene)
    torch.cuda.empty_cache()
    img = torch.empty((H, W, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(int(160e6) // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    phase_ev = {}

    def mark(name):
        if phase_ev is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            phase_ev[name] = ev

    def frame():
        mark("start")
        forest.camera_set(cam)
        forest.cull()
        mark("cull")
        forest.cast_segments(fold)
        mark("cast")
        if scene.coarsen_cycles:
            forest.aggregate(scene.coarsen_cycles)
        mark("aggregate")
        if world == 1:
            forest.composite(out=img)
            mark("composite")
            return None
        from paper_1809_01334_b200 import dist as rdist
        out = rdist.exchange_and_composite(forest, scene.tiles, world, rank)
        mark("composite")
        return out

    for _ in range(max(3, args.warmup)):
        frame()
    torch.cuda.synchronize()
    segs = forest.segments()
    hits_local = segs["hit_pairs"]
    cand_local = segs["candidates"]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([hits_local, cand_local], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        hits_total, cand_total = int(t[0]), int(t[1])
    else:
        hits_total, cand_total = hits_local, cand_local

    # --- timed region: K frames, L2 flushed between frames (outside events) ---
    times, cast_ms, phase_ms = [], [], []
    phase_acc = {}
    rc.launch_count(reset=True)
    with Clocks(local) as clk:
        for _ in range(args.steps):
            l2_flush(flush)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            frame()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            cast_ms.append(forest.last_phase_ms(1))
            if world == 1:
                for k, nm in ((4, "composite_bucket"), (5, "composite_fold")):
                    phase_acc[nm] = phase_acc.get(nm, 0.0) + forest.last_phase_ms(k) / args.steps
            names = ["start", "cull", "cast", "aggregate", "composite"]
            for a, b in zip(names, names[1:]):
                phase_acc[b] = phase_acc.get(b, 0.0) + phase_ev[a].elapsed_time(phase_ev[b]) / args.steps
    launches = rc.launch_count()
    ms_local = sum(times) / len(times)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_local, sum(cast_ms) / len(cast_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, cast_avg = float(t[0]), float(t[1])
    else:
        ms_step, cast_avg = ms_local, sum(cast_ms) / len(cast_ms)
    value = hits_total / (ms_step / 1000.0)

    # --- roofline of the dominant kernel (segment kernel) -----------------
    pk = peaks()
    import bench_model
    fl = bench_model.flops(scene.geom_degree if not forest_affine(scene) else 1, N, hits_local, cand_local)
    achieved = fl / (cast_avg / 1000.0) / 1e12
    kname = "k_cast_affine" if forest_affine(scene) else "k_cast_curved (intersection + integration + fold, fused)"
    roof = {"kernel": kname, "bound": "alu",
            "achieved": achieved, "peak": pk["fp32_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["fp32_tflops"],
            "traffic": None, "kernel_ms": cast_avg, "share_of_step": cast_avg / ms_step,
            "algorithmic_flops_per_launch": fl, "peak_source": pk["source"]}
    tpath = os.path.join(ROOT, "profiles", f"traffic_c{args.config}.json")
    if os.path.exists(tpath):
        try:
            roof["traffic"] = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            pass

    # --- end to end through the public API with HOST buffers --------------
    seg_info = forest.segments()
    composite_copy = int(forest.last_phase_ms(3))
    newton_failures = seg_info["newton_failures"]
    fold_info = {"face_failures": seg_info["face_failures"], "fold_levels": fold, "records": seg_info["count"], "raw_segments": seg_info["raw_segments"],
                 "record_level": seg_info["level"], "units": seg_info["units"],
                 "unfolded_units": seg_info["unfolded_units"], "face_tasks": seg_info["face_tasks"],
                 "fallback_tasks": seg_info["fallback_tasks"]}
    forest.close()          # release the device-resident forest before the e2e forests
    del forest
    torch.cuda.empty_cache()
    host = [np.ascontiguousarray(a if isinstance(a, np.ndarray) else a.cpu().numpy())
            for a in (scene.leaf_anchor[lo:hi], scene.leaf_tree[lo:hi], scene.leaf_level[lo:hi],
                      scene.leaf_field[lo:hi])]
    pinned = [torch.from_numpy(a).pin_memory() for a in host]
    pinned_np = [p.numpy() for p in pinned]
    h2d = sum(a.nbytes for a in host)
    img_host = torch.empty((H, W, 4), dtype=torch.float32).pin_memory()
    e2e_times = []
    n_e2e = 0 if args.no_e2e else 2 + (1 if args.config >= 4 else max(1, min(args.steps, 3)))
    for it in range(n_e2e):
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        # rc_forest_create copies the pinned host arrays (the scene generator
        # guarantees SFC order: RC_HOST_COPY_TRUSTED skips the host-side check)
        f2 = rc.Forest(scene.tree_ctrl, scene.geom_degree, scene.field_degree, *pinned_np, scene.kappa0,
                       scene.inv_F, scene.q0, first_global_leaf=lo, trusted=True)
        f2.camera_set(cam)
        f2.cull()
        f2.cast_segments(fold)
        if scene.coarsen_cycles:
            f2.aggregate(scene.coarsen_cycles)
        if world == 1:
            out = f2.composite()
            img_host.copy_(out)
        else:
            from paper_1809_01334_b200 import dist as rdist
            out = rdist.exchange_and_composite(f2, scene.tiles, world, rank)
            img_host.view(-1)[:out.numel()].copy_(out.view(-1))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        f2.close()
        if it >= 2:
            e2e_times.append(dt)
    e2e_s = sum(e2e_times) / len(e2e_times) if e2e_times else float("nan")
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e = {"value": hits_total / e2e_s, "unit": "hit pairs/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": H * W * 16, "ms_per_step": e2e_s * 1000.0}

    if rank == 0:
        line = {"metric": "element-ray segment evaluations/s (hit pairs/s)", "value": value, "unit": "hit pairs/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded, scenegen)",
                "config": {"workload": WORKLOAD[args.config], "leaves": n, "image": [W, H], "gl_points": N,
                           "hit_pairs": hits_total, "candidate_pairs": cand_total,
                           "candidate_pairs_per_s": cand_total / (ms_step / 1000.0),
                           "l2": "flushed between frames (160 MB write outside the events)",
                           "parallelism": f"sfc{world}"},
                "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e,
                "newton_failures": newton_failures, "segments": fold_info,
                "phase_ms": {k: round(v, 3) for k, v in phase_acc.items()},
                "composite_copy": composite_copy}
        if world == 1 and not args.no_cpu_baseline:
            stride = {1: 1, 2: 2, 3: 16, 4: 64, 5: 128, 45: 32}[args.config]   # oracle cull of all leaves is a fixed ~40 s (C4)
            sc_cpu = scene_to_host(scene)
            cb = cpu_baseline(sc_cpu, stride)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
