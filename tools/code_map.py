"""Static hot-code map of one kernel in an ncu report: instructions executed
at least THRESH x the hottest, grouped by the source function they come from
(nearest preceding __device__/struct definition in the file) -- the i-cache
footprint per function.  Usage: code_map.py report.ncu-rep lib.so kernel_substr [thresh]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
thresh = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie = h.index("Instructions Executed")
ni = h.index("stall_no_inst") if "stall_no_inst" in h else None
sa = h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), int(r[ie] or 0)) for r in rows[2:] if len(r) > ie]
stall = {int(r[0], 16): (int(r[ni] or 0) if ni is not None else 0, int(r[sa] or 0)) for r in rows[2:] if len(r) > ie}
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
addr2line = {}
for cub in sorted(os.listdir(d)):
    if not cub.endswith(".cubin"):
        continue
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.split("\n")
    start = next((i for i, l in enumerate(dis) if l.startswith(".text.") and ksub in l and l.rstrip().endswith(":")), None)
    if start is None:
        continue
    cur = None
    for l in dis[start + 1:]:
        if l.startswith(".text.") and l.rstrip().endswith(":"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1), int(m.group(2)))
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m2 and cur:
            addr2line[int(m2.group(1), 16)] = cur
    break
funcs = {}


def func_of(path, line):
    if path not in funcs:
        starts = []
        try:
            for i, l in enumerate(open(path), 1):
                m = re.search(r"(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)
                if m and "__forceinline__ bool operator" not in l:
                    starts.append((i, m.group(1)))
                elif re.match(r"\s*(?:struct|template <int K)", l) and "struct" in l:
                    starts.append((i, l.strip()[:30]))
        except OSError:
            pass
        funcs[path] = starts
    name = "?"
    for i, n in funcs[path]:
        if i <= line:
            name = n
        else:
            break
    return os.path.basename(path) + ":" + name


base = data[0][0]
mx = max(n for _, n in data)
cnt = collections.Counter()
exe = collections.Counter()
noi = collections.Counter()
alls = collections.Counter()
for a, n in data:
    k = addr2line.get(a - base, ("?", 0))
    f = func_of(*k) if k[0] != "?" else "?"
    noi[f] += stall[a][0]
    alls[f] += stall[a][1]
    if n >= thresh * mx:
        cnt[f] += 1
        exe[f] += n
tot = sum(cnt.values())
tn, ta = max(1, sum(noi.values())), max(1, sum(alls.values()))
print(f"hot static instructions (>= {thresh} x hottest): {tot} ({tot * 16 / 1024:.1f} KB); "
      f"no_inst stall samples {tn} of {ta} ({100 * tn / ta:.1f}%)")
print("instr     KB   exec%  stall%  no_inst%  function")
for f, c in cnt.most_common():
    print(f"{c:6d} {c * 16 / 1024:6.1f} {exe[f] / sum(exe.values()) * 100:6.1f} {100 * alls[f] / ta:6.1f} "
          f"{100 * noi[f] / tn:7.1f}   {f}")
