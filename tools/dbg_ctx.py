"""Context-strategy debug matrix vs the oracle (GPU box)."""
import os, sys, itertools, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs
fails = 0
cases = 0
for L, K, fl, thr, grid, q0, seed in itertools.product((1, 3, 20, 200, 5000), (0, 1, 2, 3, 4), (0, rs.RS_FLAG_UNFUSED),
                                                         (192, 1), (0, 1), (0, 128), (1,)):
    R = max(3, (1 << 16) // L)
    lens = synth.lengths(R, "var", L=L, seed=L + K)
    off = synth.offsets(lens, base=3)
    vals = synth.values(int(off[-1]) + 5, "i32", seed=L * 7 + K)
    st = [("hash_lt", [0x9E3779B1, 0x85EBCA6B, 0xC2B2AE35, 0x27D4EB2F][k], thr) for k in range(K)]
    ref = oracle.brute(vals, off, st, "sum_i64")[0]
    e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
    try:
        p = rs.Pipeline(st, "sum_i64", strategy="context", flags=rs.RS_FLAG_STATS | fl, grid=grid, q0_stage=q0)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, e.numel())
        p.run(e, o, out, ws); torch.cuda.synchronize()
        err = 0
        try:
            p.check()
        except Exception as ex:
            err = str(ex)[-25:]
        got = out[0].cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        st_ = p.stats()
        cnt_ok = st_[0][2] == off[-1] - off[0]
    except Exception as ex:
        err, bad, cnt_ok = str(ex)[-60:], np.arange(1), False
    cases += 1
    if err or bad.size or not cnt_ok:
        fails += 1
        print(f"FAIL L={L} K={K} unfused={bool(fl)} thr={thr} grid={grid} q0={q0}: err={err} bad={bad.size} {bad[:5].tolist()} cnt_ok={cnt_ok}", flush=True)
print(f"{cases - fails}/{cases} ok")
