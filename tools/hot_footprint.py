"""Hot instruction footprint of a profiled kernel: how many distinct SASS
instructions carry given fractions of the executed instructions (I-cache
working set).  Usage: hot_footprint.py report.ncu-rep"""
import csv, io, subprocess, sys
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie = h.index("Instructions Executed")
n = sorted((int(r[ie] or 0) for r in rows[2:] if len(r) > ie), reverse=True)
tot = sum(n)
print(f"static instructions {len(n)} ({len(n) * 16 / 1024:.1f} KB), executed {tot}")
acc = 0
marks = [0.5, 0.8, 0.9, 0.95, 0.99, 0.999]
for i, x in enumerate(n):
    acc += x
    while marks and acc >= marks[0] * tot:
        print(f"  {marks[0] * 100:5.1f}% of executed in {i + 1} instructions ({(i + 1) * 16 / 1024:.1f} KB)")
        marks.pop(0)
thr = [1e-3, 1e-4, 1e-5]
for t in thr:
    k = sum(1 for x in n if x >= t * n[0])
    print(f"  instructions executed >= {t:g} x hottest: {k} ({k * 16 / 1024:.1f} KB)")
