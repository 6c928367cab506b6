"""Benchmark of the raycasting hot path (BASELINE.json metric: element-ray
segment evaluations/s and ms/frame; % of the FP32 roofline).

One step = one frame: rc_camera_set + rc_cull + rc_cast_segments
(+ rc_aggregate cycles) + tile exchange and composite, on seeded synthetic
inputs already resident in HBM.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Multi-GPU: contiguous SFC ranges, re-cut after a first cull at
equal prefix sums of w_E = rect area + 1 (aligned to the coarsest node level
the fold and cycles reach) with the leaves moved to their new owners (the
pre-partition, timed separately as `repartition_ms`); records go to the tile
owners through librc's NCCL communicator (rc_composite_tiles).
--dist-backend gloo runs the same code with host-staged exchanges (tests:
several ranks on one GPU).
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
    """FP32 FMA-pipe peak for the roofline.  Measured on the box by
    tools/peaks.py (profiles/peaks_r02.json: independent-chain FFMA across all
    SMs, TFLOP/s at 2 flops per FFMA) when present, else derived from the
    guide's unit counts at MEASURED_PEAKS.json's SM clock."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        mp = {}
    sm_mhz = float(mp.get("sm_max_mhz", 1965.0))
    derived = NUM_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    out = dict(fp32_tflops=derived, hbm_gbs=float(mp.get("hbm_gbs", 6650.0)), sm_mhz=sm_mhz,
               source="derived: 148 SM x 128 FP32 lanes x 2 x MEASURED_PEAKS.json sm_max_mhz (guide unit counts)")
    try:
        meas = json.load(open(os.path.join(ROOT, "profiles", "peaks_r02.json")))
        out["fp32_tflops"] = float(meas["ffma_tflops"])
        out["source"] = (f"measured: {meas['how']} ({meas['when']}); derived at {sm_mhz:.0f} MHz would be "
                         f"{derived:.1f}")
        out["mufu_ex2_tops"] = meas.get("mufu_ex2_tops")
        if meas.get("dfma_tflops"):
            out["fp64_tflops"] = float(meas["dfma_tflops"])
            out["fp64_source"] = f"measured: tools/peaks.cu fma.rn.f64 chains ({meas['when']})"
        out["fmnmx_tops"] = meas.get("fmnmx_tops")
    except Exception:
        pass
    return out


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
    if cfg == 55:   # profiling stand-in for C5: maxlevel 8 at 1024^2 (about C5's records per pixel)
        return sg.config5(device=device, maxlevel=8, width=1024)
    if cfg == 6:    # NEXT(3) surface workload: the Mandelbrot hexagon, bent patches
        return sg.mandelbrot_hexagon(3, 11, width=2048, bend=0.35, name="MB")
    if cfg == 33:   # test size: C3's geometry at level 4, 128^2, 4 x 4 tiles, 2 coarsening cycles
        import dataclasses
        sc = sg.shell_uniform(4, 128, 16, gl_points=6, name="C3-L4", tiles=(4, 4), device=device)
        return dataclasses.replace(sc, coarsen_cycles=2)
    raise ValueError(cfg)


WORKLOAD = {1: "C1: identity cube, uniform level 3 (512 hex), ortho 64x64, N=4",
            2: "C2: identity cube, adaptive levels 3..7 (87,088 hex), perspective 512x512, N=4",
            3: "C3: cubed-sphere shell R=2, uniform level 6 (1,572,864 hex), 1024x1024, N=6",
            4: "C4: cubed-sphere shell R=2, uniform level 8 (100,663,296 hex), 2048x2048, N=6",
            5: "C5: cubed-sphere shell R=2, adaptive levels 6..10, 4096x4096, N=8, 3 coarsening cycles",
            6: "MB (surfaces, NEXT(3)): Mandelbrot hexagon, 2 quadtrees, levels 3..11, bent bilinear patches, "
               "2048x2048, Eq. ABphi points",
            45: "C4s (profiling stand-in): shell R=2, uniform level 7 (12,582,912 hex), 1024x1024, N=6",
            55: "C5s (profiling stand-in): shell R=2, adaptive levels ..8, 1024x1024, N=8, 3 coarsening cycles",
            33: "C3-L4 (test size): shell R=2, uniform level 4, 128x128, N=6, 4x4 tiles, 2 coarsening cycles"}

# oracle pixel sample (every s-th row and column) of the CPU baseline and the reference arm
CPU_STRIDE = {1: 1, 2: 2, 3: 16, 4: 64, 5: 128, 6: 4, 45: 32, 55: 32, 33: 1}


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


def instance_cameras(scene, count):
    """Image instances: instance 0 is the config's camera;
    instance k >= 1 turns it by 35 k degrees about the vertical axis through
    the scene centre and narrows the field of view to 0.6 of it (a camera that
    culls part of the forest), same image size and rule."""
    import dataclasses
    import numpy as np
    cam = scene.camera
    cams = [cam]
    piv = np.zeros(3) if scene.geom_degree == 2 or getattr(scene, "dim", 3) == 2 else np.full(3, 0.5)
    for k in range(1, count):
        a = math.radians(35.0 * k)
        Rz = np.array([[math.cos(a), -math.sin(a), 0.0], [math.sin(a), math.cos(a), 0.0], [0.0, 0.0, 1.0]])
        rot = lambda v: Rz @ np.asarray(v, dtype=np.float64)
        cams.append(dataclasses.replace(cam, origin=piv + rot(np.asarray(cam.origin) - piv), view=rot(cam.view),
                                        right=rot(cam.right), up=rot(cam.up), pixel_size=cam.pixel_size * 0.6))
    return cams


def cpu_model():
    model, sockets = None, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() == "Model name":
                model = v.strip()
            if k.strip() == "Socket(s)":
                sockets = v.strip()
    except Exception:
        pass
    return model, sockets


def cpu_baseline(scene, stride, hits_full, one_thread=True):
    """The oracle as it stands (exact mode) on the host cores, SURVEY §8(d):
    the full fp64 cull of every leaf (T_cull), then every `stride`-th pixel
    row and column rendered with that culled list (T_sample); extrapolated
    frame = T_sample * hits_full / hits_sample + T_cull.  A 1-thread run on
    every 4th sampled row gives the single-core rate."""
    import numpy as np

    import oracle
    o = oracle.OracleScene(scene)
    W, H = scene.camera.width, scene.camera.height
    t0 = time.perf_counter()
    vis, amb, rects = o.cull()
    t_cull = time.perf_counter() - t0
    jj, ii = np.meshgrid(np.arange(stride // 2, H, stride), np.arange(stride // 2, W, stride), indexing="ij")
    pix = (jj * W + ii).ravel().astype(np.int32)
    t0 = time.perf_counter()
    res = o.render_pairs(pix, mode="exact", rects=rects)
    t_sample = time.perf_counter() - t0
    hs = max(res["total_hits"], 1)
    cores = os.cpu_count() or 1
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        pass
    scale = (W * H) / pix.size   # stratified sample -> whole image (pixel ratio, as the reference arm)
    frame_s = t_sample * scale + t_cull
    out = dict(value=hs * scale / frame_s, unit="hit pairs/s", cores=cores, kind="oracle",
               sample=f"full fp64 cull of {scene.num_leaves} leaves ({t_cull:.1f} s) + every {stride}th pixel row "
                      f"and column ({pix.size} pixels, {res['total_hits']} hit pairs, {t_sample:.1f} s, exact mode); "
                      f"extrapolated frame = T_sample x {scale:.0f} (pixel ratio) + T_cull",
               extrapolated_ms_per_frame=1000.0 * frame_s, t_cull_s=t_cull, t_sample_s=t_sample,
               frame_hit_pairs_gpu=int(hits_full), frame_hit_pairs_extrapolated=int(hs * scale),
               hit_pairs_sample=int(res["total_hits"]),
               rate_per_core=res["total_hits"] / t_sample / cores, threads=cores)
    if one_thread:
        sub = pix.reshape(jj.shape)[::4].ravel()
        t0 = time.perf_counter()
        r1 = o.render_pairs(sub, mode="exact", rects=rects, nthreads=1)
        t1 = time.perf_counter() - t0
        out["rate_1_thread"] = r1["total_hits"] / t1
        out["sample_1_thread"] = f"{sub.size} pixels, {r1['total_hits']} hit pairs, {t1:.1f} s"
    model, sockets = cpu_model()
    out["cpu_model"], out["sockets"] = model, sockets
    return out


def run_reference(args):
    """--impl reference: the fp64 oracle timed as it stands on host cores, on
    the same workload, metric and pixel sample as cpu_baseline.  The cull is
    done once (its time counts in every step's extrapolated frame); each step
    renders the sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import torch

    import oracle
    dev = "cuda" if (args.config >= 3 and torch.cuda.is_available()) else None
    scene = scene_to_host(make_scene(args.config, dev))
    stride = CPU_STRIDE[args.config]
    o = oracle.OracleScene(scene)
    W, H = scene.camera.width, scene.camera.height
    t0 = time.perf_counter()
    vis, amb, rects = o.cull()
    t_cull = time.perf_counter() - t0
    jj, ii = np.meshgrid(np.arange(stride // 2, H, stride), np.arange(stride // 2, W, stride), indexing="ij")
    pix = (jj * W + ii).ravel().astype(np.int32)
    for _ in range(min(args.warmup, 1)):
        o.render_pairs(pix[:max(1, pix.size // 8)], mode="exact", rects=rects)
    times, hits = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = o.render_pairs(pix, mode="exact", rects=rects)
        times.append(time.perf_counter() - t0)
        hits = res["total_hits"]
    t_sample = statistics.median(times)
    # the stratified sample scaled to the whole image (pixel ratio)
    scale = (W * H) / pix.size
    hits_full = hits * scale
    frame_s = t_sample * scale + t_cull
    v = hits_full / frame_s
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    model, sockets = cpu_model()
    cb = {"value": v, "unit": "hit pairs/s", "cores": cores, "kind": "oracle",
          "sample": f"full fp64 cull ({t_cull:.1f} s, once) + every {stride}th pixel row and column ({pix.size} "
                    f"pixels, {hits} hit pairs, median {t_sample:.1f} s per step); frame = T_sample x "
                    f"{scale:.0f} (pixel ratio) + T_cull", "cpu_model": model, "sockets": sockets}
    line = {"impl": "reference", "metric": "element-ray segment evaluations/s (hit pairs/s)", "value": v,
            "unit": "hit pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * frame_s, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, scenegen)",
            "config": {"workload": WORKLOAD[args.config], "sample_stride": stride},
            "cpu_baseline": cb,
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
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged exchanges (tests: several ranks on one GPU)")
    ap.add_argument("--dump", default="", help="rank 0 writes the assembled image and hit counts (npz)")
    ap.add_argument("--instances", type=int, default=1,
                    help="image instances per frame (PAPER.md:835-841): the config camera + turned, narrower ones")
    ap.add_argument("--prepartition", default="vforest", choices=["vforest", "leaves"],
                    help="N > 1: vforest = copy only the leaves some instance sees, weighted by their summed "
                         "visible pixels (PAPER.md:873-899); leaves = weight and move every leaf")
    ap.add_argument("--all-to-all", action="store_true",
                    help="N > 1: count all-to-all instead of the partners discovered from the partition markers")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_1809_01334_b200 import rc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    tp = comm = None
    if world > 1:
        import torch.distributed as dist

        from paper_1809_01334_b200 import dist as rdist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        tp = rdist.Transport()
    scene = make_scene(args.config, dev if args.config >= 2 else None)
    cam = scene.camera
    cams = instance_cameras(scene, max(1, args.instances))
    NI = len(cams)
    W, H = cam.width, cam.height
    N = cam.gl_points
    rc.lib()

    surface = getattr(scene, "dim", 3) == 2
    surf_kw = dict(dim=2, surface=scene.surface) if surface else {}
    fold = args.fold if args.fold >= 0 else (0 if forest_affine(scene) or surface else 2)
    cycles = scene.coarsen_cycles
    n = scene.num_leaves
    tiles = scene.tiles if world > 1 else (1, 1)
    repart = {}
    if world > 1:
        # --- pre-partition: equal counts, first cull, weighted cut, leaf move
        t0 = time.perf_counter()
        A, T, Lv, F = (torch.as_tensor(x).to(dev) for x in (scene.leaf_anchor, scene.leaf_tree, scene.leaf_level,
                                                             scene.leaf_field))
        allowed = rdist.node_starts(A, T, Lv, fold + cycles)
        old = rdist.aligned_ranges(torch.ones(n, dtype=torch.float64), world, allowed)
        lo, hi = old[rank]
        f0 = rc.Forest(scene.tree_ctrl, scene.geom_degree, scene.field_degree, A[lo:hi], T[lo:hi], Lv[lo:hi],
                       F[lo:hi], scene.kappa0, scene.inv_F, scene.q0, first_global_leaf=lo, **surf_kw)
        if args.prepartition == "vforest":   # only what some instance sees moves
            consts6 = (scene.tree_ctrl, scene.geom_degree, scene.field_degree, scene.kappa0, scene.inv_F, scene.q0,
                       surf_kw)
            forest, keys, ranges, vst = rdist.vforest_prepartition(f0, cams, tp, fold + cycles, consts6)
            f0.close()
            wsum = vst["visible_weight_local"]
            n_vf = vst["vforest_leaves"]
            del A, T, Lv, F, allowed
        else:
            f0.camera_set(cam)
            f0.cull()
            w = f0.leaf_weights()
            f0.close()
            ranges = rdist.distributed_aligned_cuts(w, allowed[lo:hi], lo, n, tp)
            mine = rdist.redistribute_rows([A[lo:hi], T[lo:hi], Lv[lo:hi], F[lo:hi]], old, ranges, tp)
            wsum = float(w.sum())
            n_vf = n
            del A, T, Lv, F, allowed, w
            forest = rc.Forest(scene.tree_ctrl, scene.geom_degree, scene.field_degree, *mine, scene.kappa0,
                               scene.inv_F, scene.q0, first_global_leaf=ranges[rank][0], **surf_kw)
            keys = mine[:3]
            del mine
        lo, hi = ranges[rank]
        torch.cuda.synchronize()
        repart = {"repartition_ms": 1000.0 * (time.perf_counter() - t0), "ranges": ranges, "weight_local": wsum,
                  "equal_count_ranges": old, "prepartition": args.prepartition, "vforest_leaves": n_vf}
        if args.dist_backend == "nccl":
            comm = rc.Comm(world, rank)
    else:
        lo, hi = 0, n
        ranges = [(0, n)]
        forest = rc.Forest.from_scene(scene, first=lo, count=hi - lo, device_copy=True)
        keys = None
    # the forest holds its own device copy: keep the scene on the host only
    # (e2e inputs, CPU baseline) and hand the generator's memory back (C5 needs it)
    scene = scene_to_host(scene)
    torch.cuda.empty_cache()
    img = torch.empty((H, W, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(int(160e6) // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()
    consts = (scene.tree_ctrl, scene.geom_degree, scene.field_degree, scene.kappa0, scene.inv_F, scene.q0, cam)

    phase_ev = {}
    moved = [0]
    imgs = [img] + [torch.empty((H, W, 4), dtype=torch.float32, device=dev) for _ in range(NI - 1)]
    kt = {1: 0.0, 6: 0.0, 7: 0.0}   # instances > 1: summed cast / kernel / prep ms of the last frame
    partners = [None] * NI          # per instance (send_to, recv_from), discovered after the warm-up
    final_keys = [keys] * NI        # this rank's leaf keys at the exchange (after the cycles' repartition)

    def mark(name, k=0):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        phase_ev[(name, k)] = ev

    def frame(f, f_keys, f_rng, collect=None):
        """One frame: every image instance in turn (camera, cull, cast with the
        on-chip fold, cycles, exchange + composite).  Returns (outputs per
        instance, the last instance's aggregation forest)."""
        outs = []
        fa = f
        for k in range(NI):
            if fa is not f:
                fa.close()
            mark("start", k)
            f.camera_set(cams[k])
            f.cull()
            mark("cull", k)
            f.cast_segments(fold)
            mark("cast", k)
            if NI > 1:   # the segment-kernel timings of every instance ([sync] reads)
                for ph in (1, 6, 7):
                    kt[ph] = (kt[ph] if k else 0.0) + f.last_phase_ms(ph)
            fa = f
            if cycles:
                if world > 1:
                    fa, fk, _, _, mv = rdist.aggregate_with_repartition(f, f_keys, f_rng, ranges, cycles,
                                                                       fold + cycles, tp, consts[:6] + (cams[k],))
                    moved[0] = mv
                    final_keys[k] = fk
                else:
                    f.aggregate(cycles)
            mark("aggregate", k)
            if collect is not None:
                sg_ = f.segments()
                collect.append((sg_["hit_pairs"], sg_["candidates"], sg_["hits_per_pixel"].reshape(-1).to(torch.int64)))
            if world == 1:
                f.composite(out=imgs[k])
                mark("composite", k)
                outs.append(imgs[k])
                continue
            if comm is not None:
                if partners[k] is None:
                    comm.set_partners()
                else:
                    comm.set_partners(*partners[k])
            out = rdist.exchange_and_composite(fa, tiles, world, rank, comm=comm, tp=tp,
                                               partners=partners[k] if comm is None else None)
            mark("composite", k)
            outs.append(out)
        return outs, fa

    use_graph = world == 1 and forest_affine(scene) and fold == 0 and not cycles and NI == 1   # launch-bound C1 / C2

    def graph_frame():
        mark("start")
        forest.frame_replay()
        mark("composite")
        return [img], forest

    def run_frame(f, f_keys, f_rng, collect=None):
        out, fa = frame(f, f_keys, f_rng, collect)
        if fa is not f:
            fa.close()
        return out

    for _ in range(max(3, args.warmup)):
        run_frame(forest, keys, (lo, hi))
    partners_ms = None
    if world > 1 and not args.all_to_all:
        # exchange partners from the partition markers: the markers are
        # all-gathered with the partition; the traversal itself is local
        t0 = time.perf_counter()
        for k in range(NI):
            mk = rdist.partition_markers(final_keys[k], scene.num_trees, tp)
            forest.camera_set(cams[k])
            partners[k] = rdist.discover_partners(forest, tiles, mk, tp)
        partners_ms = 1000.0 * (time.perf_counter() - t0)
        for _ in range(2):
            run_frame(forest, keys, (lo, hi))
    if use_graph:
        img = forest.frame_capture(cam)
        imgs[0] = img
        for _ in range(3):
            forest.frame_replay()
    torch.cuda.synchronize()
    per_inst = []
    if not use_graph:
        run_frame(forest, keys, (lo, hi), collect=per_inst)
    else:
        sg_ = forest.segments()
        per_inst.append((sg_["hit_pairs"], sg_["candidates"], sg_["hits_per_pixel"].reshape(-1).to(torch.int64)))
    hits_local = sum(int(c[0]) for c in per_inst)
    cand_local = sum(int(c[1]) for c in per_inst)
    if world > 1:
        t = tp.all_gather(torch.tensor([hits_local, cand_local], dtype=torch.int64)).sum(dim=0)
        hits_total, cand_total = int(t[0]), int(t[1])
    else:
        hits_total, cand_total = hits_local, cand_local

    # --- timed region: K frames, L2 flushed between frames (outside events) ---
    times, cast_ms, kern_ms, prep_ms, phase_acc = [], [], [], [], {}
    rc.launch_count(reset=True)
    last_out = None
    with Clocks(local % ndev) as clk:
        for _ in range(args.steps):
            l2_flush(flush)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            last_out, fa = graph_frame() if use_graph else frame(forest, keys, (lo, hi))
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            ph_ms = kt if NI > 1 else {ph: forest.last_phase_ms(ph) for ph in (1, 6, 7)}
            cast_ms.append(ph_ms[1])
            kern_ms.append(ph_ms[6])
            prep_ms.append(ph_ms[7])
            if fa is not forest:
                fa.close()
            if use_graph:   # one graph: no phase events inside (the kernel time is the last ordinary frame's)
                phase_acc["graph_frame"] = phase_acc.get("graph_frame", 0.0) + \
                    phase_ev[("start", 0)].elapsed_time(phase_ev[("composite", 0)]) / args.steps
                continue
            if world == 1:
                for k, nm in ((4, "composite_bucket"), (5, "composite_fold")):
                    phase_acc[nm] = phase_acc.get(nm, 0.0) + forest.last_phase_ms(k) / args.steps
            names = ["start", "cull", "cast", "aggregate", "composite"]
            for k in range(NI):
                for a, b in zip(names, names[1:]):
                    phase_acc[b] = phase_acc.get(b, 0.0) + phase_ev[(a, k)].elapsed_time(phase_ev[(b, k)]) / args.steps
    launches = rc.launch_count()
    ms_local = sum(times) / len(times)
    cast_local = sum(cast_ms) / len(cast_ms)
    # the dominant kernel's own launches (CUDA events around each launch inside librc,
    # rc_last_phase_ms 6); the cast phase adds the element preparation kernel and memsets
    kern_local = sum(kern_ms) / len(kern_ms) if kern_ms and min(kern_ms) > 0 else cast_local
    prep_local = sum(prep_ms) / len(prep_ms) if prep_ms and min(prep_ms) >= 0 else None
    if world > 1:
        ms_step, cast_avg = tp.max(ms_local), tp.max(cast_local)
    else:
        ms_step, cast_avg = ms_local, cast_local
    value = hits_total / (ms_step / 1000.0)

    if args.dump:
        dumps = {}
        for k in range(NI):
            hpp = per_inst[k][2]
            if world > 1:
                image = rdist.gather_image(last_out[k], tiles, W, H, tp)
                hpp = tp.all_gather(hpp).sum(dim=0)
            else:
                image = last_out[k].cpu()
            sfx = "" if k == 0 else f"_{k}"
            if rank == 0:
                dumps["image" + sfx] = image.numpy()
                dumps["hits_per_pixel" + sfx] = hpp.cpu().numpy()
        if rank == 0:
            np.savez(args.dump, hit_pairs=hits_total, ranges=np.array(ranges), moved=moved[0], instances=NI, **dumps)

    # --- roofline of the dominant kernel (segment kernel) -----------------
    pk = peaks()
    import bench_model
    if surface:   # NEXT(3): fp64 ray-patch geometry
        fl = bench_model.surface_flops(hits_local, cand_local)
        kname, bound, peak = "k_cast_surface (ray-patch quadratic + Eq. ABphi)", "fp64_fma", pk.get("fp64_tflops")
    else:
        fl = bench_model.flops(scene.geom_degree if not forest_affine(scene) else 1, N, hits_local, cand_local)
        kname = "k_cast_affine" if forest_affine(scene) else "k_cast_curved (intersection + integration + fold, fused)"
        bound, peak = "fp32_fma", pk["fp32_tflops"]
    achieved = fl / (kern_local / 1000.0) / 1e12
    roof = {"kernel": kname, "bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": None, "kernel_ms": kern_local,
            "share_of_step": kern_local / ms_local, "algorithmic_flops_per_launch": fl,
            "launches_per_step": "all segment-kernel launches of one frame (curved: one per slot batch); "
                                 "flops and ms are per frame",
            "cast_phase_ms": cast_local, "prep_kernel_ms": prep_local,
            "frac_cast_phase": (fl / (cast_local / 1000.0) / 1e12) / peak if peak else None,
            "peak_source": pk["source"] if not surface else pk.get("fp64_source")}
    tpath = os.path.join(ROOT, "profiles", f"traffic_c{args.config}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            roof["traffic"] = tj.get("bytes_per_frame", tj.get("bytes_per_launch"))   # per frame, like the flops
            roof["traffic_source"] = tj.get("source")
        except Exception:
            pass

    # --- end to end through the public API with HOST buffers --------------
    seg_info = forest.segments()
    composite_copy = int(forest.last_phase_ms(3))
    newton_failures = seg_info["newton_failures"]
    fold_info = {"face_failures": seg_info["face_failures"], "fold_levels": fold, "records": seg_info["count"],
                 "raw_segments": seg_info["raw_segments"], "record_level": seg_info["level"],
                 "units": seg_info["units"], "unfolded_units": seg_info["unfolded_units"],
                 "face_tasks": seg_info["face_tasks"], "fallback_tasks": seg_info["fallback_tasks"]}
    if world > 1:   # this rank's inputs after the pre-partition (vforest rows or moved leaf rows)
        host = [a.cpu().numpy() for a in forest.leaves()]
    else:
        host = [np.ascontiguousarray(a if isinstance(a, np.ndarray) else a.cpu().numpy())
                for a in (scene.leaf_anchor[lo:hi], scene.leaf_tree[lo:hi], scene.leaf_level[lo:hi],
                          scene.leaf_field[lo:hi])]
    forest.close()          # release the device-resident forest before the e2e forests
    del forest
    torch.cuda.empty_cache()
    pinned = [torch.from_numpy(a).pin_memory() for a in host]
    pinned_np = [p.numpy() for p in pinned]
    h2d = sum(a.nbytes for a in host)
    img_host = torch.empty((NI, H, W, 4), dtype=torch.float32).pin_memory()
    e2e_times = []
    n_e2e = 0 if args.no_e2e else 2 + (1 if args.config in (4, 5) else max(1, min(args.steps, 3)))

    def new_forest(stream=None):
        # rc_forest_create copies the pinned host arrays (the scene generator
        # guarantees SFC order: RC_HOST_COPY_TRUSTED skips the host-side check)
        return rc.Forest(scene.tree_ctrl, scene.geom_degree, scene.field_degree, *pinned_np, scene.kappa0,
                         scene.inv_F, scene.q0, first_global_leaf=lo, trusted=True, stream=stream, **surf_kw)

    def e2e_step(f2):
        k2 = [torch.from_numpy(a).to(dev) for a in host[:3]] if (world > 1 and cycles) else None
        outs, fa = frame(f2, k2, (lo, hi))
        for k, out in enumerate(outs):
            img_host[k].view(-1)[:out.numel()].copy_(out.reshape(-1))
        stream.synchronize()
        if fa is not f2:
            fa.close()
        f2.close()

    for it in range(n_e2e):   # sequential steps: upload, frame, read-back
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e2e_step(new_forest())
        dt = time.perf_counter() - t0
        if it >= 2:
            e2e_times.append(dt)
    e2e_seq_s = sum(e2e_times) / len(e2e_times) if e2e_times else float("nan")
    e2e_s, pipelined = e2e_seq_s, False
    # pipelined steps (one GPU, when two forests fit): step i+1's upload runs on
    # a copy stream from a second host thread while step i's frame computes
    # (the DMA engines overlap the kernels); every step still uploads its inputs
    # and reads its image back inside the timed region
    n_pipe = 0 if args.no_e2e or world > 1 else (5 if args.config in (4, 5) else 4)
    if n_pipe and torch.cuda.mem_get_info()[0] > 3 * h2d:
        import threading
        up = torch.cuda.Stream()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cur = new_forest(up.cuda_stream)
        for i in range(n_pipe):
            nxt, err = [], []

            def upload():
                try:
                    nxt.append(new_forest(up.cuda_stream))
                except Exception as ex:   # surfaced below
                    err.append(ex)
            th = threading.Thread(target=upload) if i + 1 < n_pipe else None
            if th:
                th.start()
            e2e_step(cur)
            if th:
                th.join()
                if err:
                    raise err[0]
                cur = nxt[0]
        torch.cuda.synchronize()
        e2e_pipe_s = (time.perf_counter() - t0) / n_pipe
        if e2e_pipe_s < e2e_s:
            e2e_s, pipelined = e2e_pipe_s, True
    if world > 1:
        e2e_s = tp.max(e2e_s)
    e2e = {"value": hits_total / e2e_s, "unit": "hit pairs/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": sum(int(o.numel()) * 4 for o in last_out) if last_out else NI * H * W * 16,
           "ms_per_step": e2e_s * 1000.0, "pipelined": pipelined,
           "sequential_ms_per_step": e2e_seq_s * 1000.0,
           "how": "rc_forest_create from pinned host buffers + the frame + image read-back per step; pipelined: "
                  "the next step's upload (copy stream, second host thread) overlaps this step's frame"}

    if rank == 0:
        line = {"metric": "element-ray segment evaluations/s (hit pairs/s)", "value": value, "unit": "hit pairs/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded, scenegen)",
                "config": {"workload": WORKLOAD[args.config], "leaves": n, "image": [W, H], "gl_points": N,
                           "hit_pairs": hits_total, "candidate_pairs": cand_total,
                           "candidate_pairs_per_s": cand_total / (ms_step / 1000.0),
                           "l2": "flushed between frames (160 MB write outside the events)",
                           "parallelism": f"sfc{world}", "tiles": list(tiles), "cuda_graph_frame": use_graph,
                           "dist_backend": args.dist_backend if world > 1 else None, "instances": NI},
                "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e,
                "newton_failures": newton_failures, "segments": fold_info,
                "phase_ms": {k: round(v, 3) for k, v in phase_acc.items()},
                "composite_copy": composite_copy}
        if world > 1:
            line["partition"] = {"repartition_ms": repart["repartition_ms"], "ranges": repart["ranges"],
                                 "cycle_records_moved_rank0": moved[0], "prepartition": repart["prepartition"],
                                 "vforest_leaves": repart["vforest_leaves"], "partners_ms": partners_ms,
                                 "partners_rank0": partners if not args.all_to_all else None}
        if world == 1 and not args.no_cpu_baseline:
            sc_cpu = scene_to_host(scene)
            cb = cpu_baseline(sc_cpu, CPU_STRIDE[args.config], hits_total)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if world > 1:
        if comm is not None:
            comm.close()
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
