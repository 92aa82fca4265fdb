import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, synth
import paper_2006_07478_b200 as rs
vals, off, stages, agg = synth.tiny()
ref = oracle.brute(vals, off, stages, agg)[0]
for K in (0, 1, 2):
    for strat in ("tagged", "signal"):
        st = stages[:K]
        ref = oracle.brute(vals, off, st, agg)[0]
        p = rs.Pipeline(st, agg, strategy=strat)
        e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
        out = p.alloc_outputs(off.size - 1); ws = p.alloc_workspace(off.size - 1, vals.size)
        p.run(e, o, out, ws); torch.cuda.synchronize()
        got = out[0].cpu().numpy()
        print(K, strat, "bad", int((got != ref).sum()), "stats", p.stats().tolist(), "err", p.check())
