"""Debug helper: locate tagged-strategy mismatches (run on the GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs

def run(vals, off, stages, strategy, **cfg):
    p = rs.Pipeline(stages, "sum_i64", strategy=strategy, **cfg)
    e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
    out = p.alloc_outputs(off.size - 1); ws = p.alloc_workspace(off.size - 1, vals.size)
    p.run(e, o, out, ws); torch.cuda.synchronize()
    return out[0].cpu().numpy(), p.stats(), p.check()

for L, base, K, grid in [(4096, 3, 0, 0), (4096, 0, 0, 0), (4096, 3, 1, 0), (128, 3, 0, 0), (128, 0, 0, 0), (128, 3, 0, 1), (1, 3, 0, 0), (1, 0, 0, 0), (4096, 3, 3, 0)]:
    N = 1 << 16
    R = N // L
    off = synth.offsets(np.full(R, L, np.int64), base=base)
    vals = np.arange(int(off[-1]) + 1, dtype=np.int32) % 1000 + 1   # easy-to-read values: element g -> g%1000+1
    stages = [("hash_lt", 0x9E3779B1, 256)] * K
    ref = oracle.brute(vals, off, stages, "sum_i64")[0]
    for strat in ("signal", "tagged"):
        got, st, code = run(vals, off, stages, strat, grid=grid)
        bad = np.nonzero(got != ref)[0]
        print(f"L={L} base={base} K={K} grid={grid} {strat}: err={code} bad={bad.size} {bad[:6]}")
        for r in bad[:4]:
            print(f"   r={r} off=[{off[r]},{off[r+1]}) got={got[r]} ref={ref[r]} diff={got[r]-ref[r]}")
