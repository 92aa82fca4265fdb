"""Per-source-line executed-instruction attribution of one kernel in an ncu
report.  Usage: line_prof.py report.ncu-rep lib.so kernel_mangled_substr items [top]"""
import csv, io, subprocess, re, collections, os, sys, tempfile
rep, lib, ksub, items = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 60
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), int(r[ie] or 0), int(r[ss] or 0)) for r in rows[2:] if len(r) > ie]
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
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m2 and cur:
            addr2line[int(m2.group(1), 16)] = cur
    break
base = data[0][0]
tot = sum(x[1] for x in data)
byl = collections.Counter(); byls = collections.Counter()
for a, n, s in data:
    k = addr2line.get(a - base, ("?", 0)); byl[k] += n; byls[k] += s
print(f"total {tot} warp-inst, {tot / items:.3f} per item")
for k, n in byl.most_common(top):
    print(f"{k[0]}:{k[1]} {100 * n / tot:5.2f}% {n / items:.3f}/item stalls {byls[k]}")
