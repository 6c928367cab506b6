"""Stall samples of an ncu source-page capture per source line (innermost and
outermost-in-kernel lines of each SASS instruction, nvdisasm -gi).
python tools/prof_lines.py REPORT.ncu-rep OBJ KERNEL_MANGLED_SUBSTR [TOP]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text.") and kname in l][0]
addr, cur = {}, None
for l in sass[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)(.*)', l)
    if m:
        chain = [(os.path.basename(m.group(1)), int(m.group(2)))] + \
            [(os.path.basename(a), int(b)) for a, b in re.findall(r'inlined at "(.*?)", line (\d+)', m.group(3))]
        cur = chain
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        addr[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, iE, iW = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
isd = [hdr.index(h) for h in stalls]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), float(r[iE] or 0), float(r[iW] or 0), [float(r[i] or 0) for i in isd]))
    except Exception:
        pass
base = min(d[0] for d in data)
src_cache = {}


def src_line(fn, ln):
    if fn not in src_cache:
        p = os.path.join("paper_1809_01334_b200/csrc", fn)
        src_cache[fn] = open(p).read().split("\n") if os.path.exists(p) else []
    s = src_cache[fn]
    return s[ln - 1].strip()[:70] if 0 < ln <= len(s) else ""


for which in ("inner", "outer"):
    agg = collections.defaultdict(lambda: [0.0, 0.0, [0.0] * len(stalls)])
    for a, n, w, st in data:
        ch = addr.get(a - base)
        key = ("?", 0) if not ch else (ch[0] if which == "inner" else ch[-1])
        agg[key][0] += n
        agg[key][1] += w
        agg[key][2] = [x + y for x, y in zip(agg[key][2], st)]
    tn = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"== by {which} line: inst% samp%  top stalls")
    for k, (n, w, st) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        t3 = sorted(zip(stalls, st), key=lambda x: -x[1])[:3]
        print("%-18s %5.1f %5.1f  %-70s  %s" % ("%s:%d" % k, 100 * n / tn, 100 * w / tw, src_line(*k),
                                              ", ".join("%s %.0f%%" % (s[6:], 100 * v / max(w, 1)) for s, v in t3)))
