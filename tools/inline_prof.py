"""Executed warp-instructions of one kernel in an ncu report, attributed to
the INLINE call chain of each SASS instruction (nvdisasm -gi), printed as a
tree of rs_pipe.cuh call sites.  Usage:
  inline_prof.py report.ncu-rep lib.so kernel_mangled_substr items [min_frac] [depth]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, lib, ksub, items = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
minf = float(sys.argv[5]) if len(sys.argv) > 5 else 0.005
maxd = int(sys.argv[6]) if len(sys.argv) > 6 else 8
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie = h.index(os.environ.get("COL", "Instructions Executed"))
data = [(int(r[0], 16), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]
d = tempfile.mkdtemp()
if lib.endswith(".cubin"):
    import shutil
    shutil.copy(lib, d)
else:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
chains = {}
for cub in sorted(os.listdir(d)):
    if not cub.endswith(".cubin"):
        continue
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
    start = next((i for i, l in enumerate(dis) if l.startswith(".text.") and ksub in l and l.rstrip().endswith(":")), None)
    if start is None:
        continue
    cur, pend = [], []
    for l in dis[start + 1:]:
        if l.startswith(".text.") and l.rstrip().endswith(":"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)( inlined at "([^"]+)", line (\d+))?', l)
        if m:
            pend.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m2:
            if pend:
                cur = pend       # innermost first
                pend = []
            chains[int(m2.group(1), 16)] = [f"{f}:{n}" for f, n in cur if f.startswith("rs_")]
    break
base = data[0][0]
tot = sum(n for _, n in data)
tree = collections.defaultdict(int)
for a, n in data:
    ch = chains.get(a - base, [])
    path = tuple(reversed(ch))      # outermost first
    for k in range(1, min(len(path), maxd) + 1):
        tree[path[:k]] += n
srcl = {}
def text(site):
    f, n = site.split(":")
    p = os.path.join(os.environ.get("SRCROOT", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")),
                     "paper_2006_07478_b200", "csrc", f)
    if f not in srcl:
        try:
            srcl[f] = open(p).read().split("\n")
        except OSError:
            srcl[f] = []
    L = srcl[f]
    return L[int(n) - 1].strip()[:70] if int(n) - 1 < len(L) else ""
print(f"total {tot} warp-inst, {tot / items:.3f} per item")
for path in sorted(tree, key=lambda p: [(-tree[p[:k]], p[k - 1]) for k in range(1, len(p) + 1)]):
    n = tree[path]
    if n < minf * tot:
        continue
    print(f"{'  ' * (len(path) - 1)}{path[-1]:16s} {100 * n / tot:6.2f}% {n / items:.4f}/item  {text(path[-1])}")
