"""Perf probe: time the pipeline kernel for a few configurations (GPU box)."""
import argparse, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1 << 29)
ap.add_argument("--L", type=int, default=4096)
ap.add_argument("--K", type=int, default=3)
ap.add_argument("--strategy", default="signal")
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--qcap", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--matrix", action="store_true")
ap.add_argument("--qmatrix", action="store_true")
ap.add_argument("--kmatrix", action="store_true")
ap.add_argument("--scap", type=int, default=0)
a = ap.parse_args()

vals = synth.torch_values(a.N, "i32", seed=1)
def one(L, K, strategy, chunk, grid, qcap, reps, scap=0, seq=False):
    lens = torch.full((a.N // L,), L, dtype=torch.int64, device="cuda")
    off = synth.torch_offsets(lens)
    p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strategy, chunk=chunk, grid=grid,
                    queue_cap=qcap, signal_cap=scap, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | (0 if seq else rs.RS_FLAG_WARP_SPECIALIZED))
    R = off.numel() - 1
    out = p.alloc_outputs(R); ws = p.alloc_workspace(R, a.N)
    ms = []
    for i in range(reps + 1):
        p.run(vals, off, out, ws)
        t = p.kernel_times()
        if i: ms.append(t[1])
    m = statistics.median(ms)
    gbs = (4 * a.N + 16 * R) / (m / 1e3) / 1e9
    print(f"L={L} K={K} {strategy} {'seq' if seq else 'ws'} q={qcap} s={scap} chunk={chunk} grid={grid} geom={p.geometry()} main={m:.3f} ms  {a.N/(m/1e3)/1e9:.1f} Gitems/s  {gbs:.0f} GB/s  err={p.check()}", flush=True)

# reference: plain bandwidth of a torch reduction over the same array
x = vals
for _ in range(2): torch.sum(x, dtype=torch.int64)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); [torch.sum(x, dtype=torch.int64) for _ in range(5)]; e.record(); torch.cuda.synchronize()
print(f"torch.sum baseline: {s.elapsed_time(e)/5:.3f} ms = {4*a.N/(s.elapsed_time(e)/5/1e3)/1e9:.0f} GB/s")
if a.matrix:
    for K in (0, 1, 3):
        for st in ("signal", "tagged"):
            one(a.L, K, st, a.chunk, a.grid, a.qcap, a.reps)
    for ch in (2048, 32768):
        one(a.L, 3, "signal", ch, a.grid, a.qcap, a.reps)
    for L in (32, 256):
        for st in ("signal", "tagged"):
            one(L, 3, st, a.chunk, a.grid, a.qcap, a.reps)
elif a.kmatrix:
    for seq in (False, True):
        for K in (0, 1, 2, 3):
            one(a.L, K, "signal", a.chunk, a.grid, 2048, a.reps, 0, seq)
elif a.qmatrix:
    for st in ("signal", "tagged"):
        for q in (512, 1024, 2048):
            for sc in ((32, 128) if st == "signal" else (32,)):
                one(a.L, 3, st, a.chunk, a.grid, q, a.reps, sc)
    for L in (32, 256):
        for st in ("signal", "tagged"):
            one(L, 3, st, a.chunk, a.grid, 1024, a.reps)
else:
    one(a.L, a.K, a.strategy, a.chunk, a.grid, a.qcap, a.reps, a.scap)
