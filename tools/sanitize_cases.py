"""Small cases of every strategy/mode for compute-sanitizer (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs
bad_total = 0
for L in (3, 100):
    lens = synth.lengths(4000 // L + 5, "var", L=L, seed=L)
    off = synth.offsets(lens, base=2)
    vals = synth.values(int(off[-1]) + 3, "i32", seed=L)
    e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
    R = off.size - 1
    for K in (0, 2, 3):
        st = synth.sweep_stages(K)
        ref = oracle.brute(vals, off, st, "sum_i64")[0]
        for strat in ("signal", "tagged", "context"):
            for fl in (0, rs.RS_FLAG_UNFUSED):
                p = rs.Pipeline(st, "sum_i64", strategy=strat, flags=rs.RS_FLAG_STATS | fl, grid=2, q0_stage=128,
                                chunk=2048)
                out = p.alloc_outputs(R); ws = p.alloc_workspace(R, e.numel())
                p.run(e, o, out, ws); torch.cuda.synchronize()
                got = out[0].cpu().numpy()
                nb = int((got != ref).sum())
                bad_total += nb
                if nb or p.check():
                    print("MISMATCH", L, K, strat, fl, nb)
print("done, mismatches:", bad_total)
