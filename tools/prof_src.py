"""Warp-stall samples of an ncu --import-source capture per CUDA source line and
per enclosing device function, using ncu's own cuda,sass attribution (which
keeps inlined code on its real line, unlike the call-site view of prof_lines.py).
python tools/prof_src.py REPORT.ncu-rep [TOP] [FIRST_LINE LAST_LINE]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
src_path = next(r[1] for r in rows if r and r[0] == "File Path")
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if r and r[0].isdigit():
        try:
            lines.append((int(r[0]), r[1].strip(), int(r[iS]), int(r[iE])))
        except ValueError:
            pass
tot = sum(x[2] for x in lines) or 1
te = sum(x[3] for x in lines) or 1
src = open(src_path).read().split("\n") if src_path and re.match(r"/", src_path) else []
starts = [(i + 1, l) for i, l in enumerate(src) if re.match(r"^(__device__|__global__)", l)]


def func_of(n):
    best = (0, "?")
    for s, l in starts:
        if s <= n:
            best = (s, l)
    return best


print(f"{src_path}: {tot} warp-stall samples")
agg = {}
for n, _, s, e in lines:
    k = func_of(n)
    a = agg.setdefault(k, [0, 0])
    a[0] += s
    a[1] += e
print("== by function: samp% inst%")
for (ln, txt), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{100 * s / tot:5.1f} {100 * e / te:5.1f}  {ln:5d} {txt[:90]}")
sel = [x for x in lines if rng is None or rng[0] <= x[0] <= rng[1]]
print("== by line: samp% inst%")
for n, txt, s, e in sorted(sel, key=lambda x: -x[2])[:top]:
    print(f"{100 * s / tot:5.2f} {100 * e / te:5.2f}  {n:5d} {txt[:100]}")
