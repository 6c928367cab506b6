"""Per-kernel device time per frame from an ncu --metrics gpu__time_duration.sum launch list.
python tools/launch_summary.py launches.csv FRAMES"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("void ", "")[:64]
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for k, v in agg.items() if "k_bumps" not in k and "gen" not in k)
print("%-64s %7s %12s %7s" % ("kernel", "launch", "ms/frame", "share"))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-64s %7d %12.3f %6.1f%%" % (k, n, t / 1e6 / frames, 100 * t / tot if "k_bumps" not in k else 0))
