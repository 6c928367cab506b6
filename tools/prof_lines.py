"""Attribute ncu SASS-level executed instructions and stall samples to CUDA
source lines (nvdisasm -g line info of the in-tree object)."""
import collections, csv, os, re, subprocess, sys, tempfile
rep, func = sys.argv[1], sys.argv[2]
obj = sys.argv[3] if len(sys.argv) > 3 else "paper_1809_01334_b200/build/cast_curved.cu.o"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
src_csv = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(src_csv.splitlines()))
kernels = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
st = 2 if rows[0][0].startswith("Kernel") else 1
hdr = rows[st - 1]
iE, iW = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[st:]:
    try:
        data.append((int(r[0], 16), float(r[iE] or 0), float(r[iW] or 0)))
    except Exception:
        pass
data.sort()
base = data[0][0]
# map function offsets -> (file, line); the ncu addresses are relative to the kernel's own text section
addr = {}
infile = None
start = [i for i, l in enumerate(sass) if l.startswith(".text.") and func in l][0]
cur = None
for l in sass[start + 1:]:
    if l.startswith(".text.") or l.startswith("//------"):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        addr[int(m.group(1), 16)] = cur
by = collections.defaultdict(lambda: [0.0, 0.0])
tot = sum(x[1] for x in data) or 1
totw = sum(x[2] for x in data) or 1
for a, n, w in data:
    k = addr.get(a - base)
    by[k][0] += n
    by[k][1] += w
srcs = {}
for k, (n, w) in sorted(by.items(), key=lambda x: -x[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    line = ""
    if k:
        fn = k[0]
        if fn not in srcs:
            for root in ("paper_1809_01334_b200/csrc",):
                pth = os.path.join(root, fn)
                if os.path.exists(pth):
                    srcs[fn] = open(pth).read().split("\n")
        line = srcs.get(fn, [""] * (k[1] + 1))[k[1] - 1].strip()[:95]
    print("%5.1f%% %5.1f%%  %s:%s  %s" % (100 * n / tot, 100 * w / totw, k[0] if k else "?", k[1] if k else "?", line))
print("total warp instructions %.3e" % tot)
