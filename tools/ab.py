"""A/B timing of library variants in one process sequence (GPU box).
Usage: python tools/ab.py libA.so libB.so ...  (alternates runs to cancel drift)"""
import os, sys, subprocess, json
libs = sys.argv[1:]
code = r'''
import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
res = {}
for L in ((4096, 256) if not os.environ.get("AB_NOSWEEP") else ()):
    lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda")
    off = synth.torch_offsets(lens); R = off.numel() - 1
    for K in (3, 1):
        p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
        ms = []
        for i in range(6):
            p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
        res[f"L{L}K{K}"] = statistics.median(ms[1:])
if os.environ.get("AB_TEXT"):
    b, toff = synth.torch_text(1 << 30, seed=4)
    R = toff.numel() - 1
    for strat in ("signal", "tagged"):
        p = rs.Pipeline(synth.text_stages(), "count_xor64", strategy=strat, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, b.numel())
        ms = []
        for i in range(6):
            p.run(b, toff, out, ws); ms.append(p.kernel_times()[1])
        res[f"text_{strat}"] = statistics.median(ms[1:])
if os.environ.get("AB_GRAPH"):
    w, goff = synth.torch_rmat_csr(24, 16, seed=3)
    R = goff.numel() - 1
    for strat in ("signal", "tagged"):
        p = rs.Pipeline([("lt_u32", 1 << 31)], "count_min_u32", strategy=strat, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, w.numel())
        ms = []
        for i in range(6):
            p.run(w, goff, out, ws); ms.append(p.kernel_times()[1])
        res[f"graph_{strat}"] = statistics.median(ms[1:])
print(json.dumps(res))
'''
out = {l: [] for l in libs}
for rep in range(2):
    for l in libs:
        env = dict(os.environ, RS_LIB=os.path.abspath(l))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        try:
            out[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            print(l, r.stderr[-500:])
for l, rs_ in out.items():
    keys = rs_[0].keys() if rs_ else []
    print(os.path.basename(l), {k: round(min(x[k] for x in rs_), 3) for k in keys})
