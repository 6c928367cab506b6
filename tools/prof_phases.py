"""Attribute an ncu source-page capture of k_cast_curved to the kernel's
phases (by the outermost inlined-at line of each SASS instruction inside the
kernel body, nvdisasm -gi), with the stall-reason breakdown per phase.
python tools/prof_phases.py REPORT.ncu-rep [OBJ]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep = sys.argv[1]
obj = sys.argv[2] if len(sys.argv) > 2 else "paper_1809_01334_b200/build/cast_curved.cu.o"
src = open("paper_1809_01334_b200/csrc/cast_curved.cu").read().split("\n")


def line_of(pat, start=0):
    for i in range(start, len(src)):
        if pat in src[i]:
            return i + 1
    raise KeyError(pat)


k0 = line_of("k_cast_curved(CamConst cc")
bounds = [("loop head", k0), ("phase 0 prep", line_of("// ---- phase 0", k0)),
          ("phase 1 isect", line_of("// ---- phase 1: intersection", k0)),
          ("phase 2 integ", line_of("// ---- phase 2: integration", k0)),
          ("phase 3 fold", line_of("// ---- phase 3: fold", k0)), ("epilogue", line_of("#pragma unroll", line_of("// ---- phase 3: fold", k0)))]


def phase(ln):
    name = "?"
    for nm, b in bounds:
        if ln >= b:
            name = nm
    return name


tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith(".text.") and "k_cast_curvedILi2ELi6E" in l][0]
addr, cur = {}, None
for l in sass[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)(.*)', l)
    if m:
        chain = [(os.path.basename(m.group(1)), int(m.group(2)))] + \
            [(os.path.basename(a), int(b)) for a, b in re.findall(r'inlined at "(.*?)", line (\d+)', m.group(3))]
        outer = [ln for fn, ln in chain if fn == "cast_curved.cu" and ln >= k0]
        cur = phase(outer[-1]) if outer else "called fn"
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
agg = collections.defaultdict(lambda: [0.0, 0.0, [0.0] * len(stalls)])
for a, n, w, st in data:
    p = addr.get(a - base, "?")
    agg[p][0] += n
    agg[p][1] += w
    agg[p][2] = [x + y for x, y in zip(agg[p][2], st)]
tn = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print("%-14s %7s %7s   top stalls (share of the phase's samples)" % ("phase", "inst%", "samp%"))
for p, (n, w, st) in sorted(agg.items(), key=lambda x: -x[1][1]):
    top = sorted(zip(stalls, st), key=lambda x: -x[1])[:5]
    print("%-14s %6.1f%% %6.1f%%   %s" % (p, 100 * n / tn, 100 * w / tw,
                                        ", ".join("%s %.0f%%" % (s[6:], 100 * v / max(w, 1)) for s, v in top)))
