"""A/B of libraries on signal-strategy sweep points (GPU box): main-kernel ms."""
import os, sys, subprocess, json
code = r'''
import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
res = {}
for L in (1, 4, 32, 256, 4096):
    off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device="cuda"))
    R = off.numel() - 1
    p = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy="signal", flags=rs.RS_FLAG_TIMING)
    out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
    ms = []
    for i in range(3):
        p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
    assert p.check() == 0
    res[f"sigL{L}"] = statistics.median(ms[1:])
print(json.dumps(res))
'''
libs = sys.argv[1:]
out = {l: [] for l in libs}
for rep in range(2):
    for l in libs:
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RS_LIB=os.path.abspath(l)), capture_output=True, text=True)
        try:
            out[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            print(l, r.stderr[-800:])
for l, v in out.items():
    if v:
        print(os.path.basename(l), {k: round(min(x[k] for x in v), 3) for k in v[0]})
