"""Debug matrix for the in-place ring: small cases vs the oracle (GPU box)."""
import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs
vals, off, stages, agg = synth.tiny()
e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
R = off.size - 1
for K in (0, 1, 2, 3):
    st = synth.sweep_stages(K)
    ref = oracle.brute(vals, off, st, agg)[0]
    for strat, fl, q0, grid in itertools.product(("signal", "tagged"), (0, rs.RS_FLAG_UNFUSED), (128, 256, 512), (0, 1)):
        p = rs.Pipeline(st, agg, strategy=strat, flags=rs.RS_FLAG_STATS | fl, q0_stage=q0, grid=grid)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, e.numel())
        p.run(e, o, out, ws); torch.cuda.synchronize()
        got = out[0].cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        try:
            err = p.check()
        except Exception as ex:
            err = str(ex)[-30:]
        print(f"K={K} {strat} unfused={bool(fl)} q0={q0} grid={grid}: err={err} bad={bad.size} {bad[:6].tolist()}", flush=True)
