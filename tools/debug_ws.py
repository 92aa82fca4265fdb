"""Debug helper: warp-specialised kernel mismatches (run on the GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs

def run(vals, off, stages, strategy, mode, **cfg):
    flags = rs.RS_FLAG_STATS | (rs.RS_FLAG_WARP_SPECIALIZED if mode == "ws" else 0)
    p = rs.Pipeline(stages, "sum_i64", strategy=strategy, flags=flags, **cfg)
    e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
    out = p.alloc_outputs(off.size - 1); ws = p.alloc_workspace(off.size - 1, vals.size)
    p.run(e, o, out, ws); torch.cuda.synchronize()
    try:
        code = p.check()
    except Exception as ex:
        code = str(ex)
    return out[0].cpu().numpy(), p.stats(), code

PASS = ("hash_lt", 0x9E3779B1, 256)
cases = [("L64 K0", 64, [], 0), ("L64 K1", 64, [PASS], 0), ("L64 K3", 64, [PASS] * 3, 0),
         ("var20 K1", -20, [PASS], 0), ("var20 K1 g1", -20, [PASS], 1), ("L4096 K1", 4096, [PASS], 0),
         ("tiny", None, None, 0)]
for name, L, stages, grid in cases:
    if L is None:
        vals, off, stages, _ = synth.tiny()
    else:
        R = (1 << 15) // abs(L)
        lens = synth.lengths(R, "fixed" if L > 0 else "var", L=abs(L), seed=3)
        off = synth.offsets(lens)
        vals = (np.arange(int(off[-1]) + 1) % 1000 + 1).astype(np.int32)
    ref = oracle.brute(vals, off, stages, "sum_i64")[0]
    kc = oracle.node_counts(vals, off, stages).sum(axis=0)
    for strat in ("signal", "tagged"):
        for mode in ("ws", "seq"):
            got, st, code = run(vals, off, stages, strat, mode, grid=grid)
            bad = np.nonzero(got != ref)[0]
            print(f"{name:12s} {strat:6s} {mode}: err={code} bad={bad.size} {bad[:8]} items={list(st[:,2])} exp={list(kc)} sig={list(st[:,3])}", flush=True)
            for r in bad[:3]:
                print(f"     r={r} off=[{off[r]},{off[r+1]}) got={got[r]} ref={ref[r]} diff={got[r]-ref[r]}")
