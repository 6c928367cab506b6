"""profiles/traffic_c4.json from an ncu metrics CSV of one C4 frame:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:'k_cast_curved|k_prep_slots' --csv python tools/profile_frame.py --config 4 --frames 1
All launches of the frame are summed per kernel.  bench.py reads bytes_per_frame as roofline.traffic.

  python tools/traffic_json.py CSV SOURCE_NAME [TAG]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, source, tag=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    acc = {}
    for r in rows:
        name, metric, val = r[4], r[12], float(r[14].replace(",", ""))
        k = "k_cast_curved" if "k_cast_curved" in name else ("k_prep_slots" if "k_prep_slots" in name else None)
        if k is None:
            continue
        d = acc.setdefault(k, {"launches": set(), "read": 0.0, "write": 0.0, "ns": 0.0})
        d["launches"].add(r[0])
        if metric == "dram__bytes_read.sum":
            d["read"] += val
        elif metric == "dram__bytes_write.sum":
            d["write"] += val
        elif metric == "gpu__time_duration.sum":
            d["ns"] += val
    c, p = acc["k_cast_curved"], acc.get("k_prep_slots")
    out = {"config": 4, "kernel": "k_cast_curved<2,6,0>", "launches_per_frame": len(c["launches"]),
           "dram_bytes_read_per_frame": int(c["read"]), "dram_bytes_write_per_frame": int(c["write"]),
           "bytes_per_frame": int(c["read"] + c["write"]),
           "bytes_per_launch": (c["read"] + c["write"]) / max(1, len(c["launches"])),
           "kernel_ns_per_frame_under_ncu": int(c["ns"])}
    if p:
        out["prep_kernel"] = {"kernel": "k_prep_slots<2>", "launches_per_frame": len(p["launches"]),
                              "dram_bytes_read_per_frame": int(p["read"]), "dram_bytes_write_per_frame": int(p["write"]),
                              "ns_per_frame_under_ncu": int(p["ns"])}
    out["how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
                  "-k regex:'k_cast_curved|k_prep_slots' --csv python tools/profile_frame.py --config 4 --frames 1 "
                  f"(gpurun {tag}); all launches of one frame summed")
    out["source"] = source
    out["algorithmic_bytes_note"] = (
        "method inputs read once (anchor/tree/level/field 125 B x 1.0e8 leaves = 12.6 GB) + records written "
        "(4.84e8 x 32 B = 15.5 GB) = 28 GB per frame; the segment kernel reads the prepared element slots "
        "(672 B per visible leaf, written by k_prep_slots) instead of the raw leaves and writes the records plus "
        "per-CTA scratch evicted from L2 before its discard; at ~0.2 TB/s the kernel is not bandwidth-bound "
        "(FP32 pipe roofline, DESIGN.md section 6)")
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic_c4.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
