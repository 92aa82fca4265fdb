"""Attribute ncu per-instruction execution counts to source lines (needs the
cubin of the profiled library).  Usage: ncu_lines.py report.ncu-rep lib.so kernel_substr"""
import csv, io, re, subprocess, sys, os, tempfile, collections
rep, lib, ksub = sys.argv[1:4]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), int(r[ie] or 0), int(r[ss] or 0)) for r in rows[2:] if len(r) > ie]
base = data[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
# find kernel section
start = None
for i, l in enumerate(dis):
    if l.startswith(".text.") and ksub in l and l.rstrip().endswith(":"):
        start = i
        break
cur = None
addr2line = {}
for l in dis[start + 1:]:
    if l.startswith(".text.") and l.rstrip().endswith(":"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m2 and cur:
        addr2line[int(m2.group(1), 16)] = cur
agg = collections.Counter(); stl = collections.Counter()
for a, n, s in data:
    ln = addr2line.get(a - base)
    agg[ln] += n; stl[ln] += s
tot = sum(agg.values()); tots = sum(stl.values()) or 1
print(f"total executed {tot}, mapped {sum(v for k, v in agg.items() if k)}")
for k, v in agg.most_common(45):
    print(f"{100*v/tot:5.1f}%  stalls {100*stl[k]/tots:5.1f}%  {k}")
if len(sys.argv) > 4:
    # coarse grouping by source ranges: "file:lo-hi=name,..."
    for spec in sys.argv[4].split(","):
        rng, name = spec.split("=")
        f, lh = rng.split(":")
        lo, hi = map(int, lh.split("-"))
        v = sum(n for k, n in agg.items() if k and k[0] == f and lo <= k[1] <= hi)
        s = sum(n for k, n in stl.items() if k and k[0] == f and lo <= k[1] <= hi)
        print(f"{name:>12}: inst {100*v/tot:5.1f}%  stalls {100*s/tots:5.1f}%")
