"""Small cases of every strategy / mode / exit for compute-sanitizer (GPU box):
signal, tagged, context, hybrid, AUTO; fused and unfused; the element-wise
exit and the taxi parser; parent contexts; the trace kernels; the text SWAR
path; the short-region kernel.  Prints mismatches against the oracle (expected: none)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2006_07478_b200 as rs
import synth

bad = 0


def run(p, vals, off, **kw):
    e = torch.from_numpy(vals).cuda()
    o = torch.from_numpy(off).cuda()
    R = off.size - 1
    out = p.alloc_outputs(R)
    ws = p.alloc_workspace(R, e.numel())
    p.run(e, o, out, ws, **kw)
    torch.cuda.synchronize()
    return [t.cpu().numpy() if t is not None else None for t in out], p.check()


for L in (3, 100):
    lens = synth.lengths(4000 // L + 5, "var", L=L, seed=L)
    off = synth.offsets(lens, base=2)
    vals = synth.values(int(off[-1]) + 3, "i32", seed=L)
    for K in (0, 2, 3):
        st = synth.sweep_stages(K)
        ref = oracle.brute(vals, off, st, "sum_i64")[0]
        cases = [("signal", {}), ("tagged", {}), ("context", {}), ("auto", {})]
        if K >= 2:
            cases.append(("hybrid", {"tag_from": 1}))
        for strat, kw in cases:
            for fl in (0, rs.RS_FLAG_UNFUSED):
                p = rs.Pipeline(st, "sum_i64", strategy=strat, flags=rs.RS_FLAG_STATS | fl, grid=2, q0_stage=128,
                                chunk=2048, **kw)
                got, code = run(p, vals, off)
                nb = int((got[0] != ref).sum())
                bad += nb
                if nb or code:
                    print("MISMATCH", L, K, strat, fl, nb, code)
    # short-region kernel (RS_FLAG_SHORT_ON), default and small geometry
    for K in (1, 3):
        st = synth.sweep_stages(K)
        ref = oracle.brute(vals, off, st, "sum_i64")[0]
        for kw in ({}, {"queue_cap": 512, "signal_cap": 4, "q0_stage": 128}):
            p = rs.Pipeline(st, "sum_i64", flags=rs.RS_FLAG_STATS | rs.RS_FLAG_SHORT_ON, grid=2, chunk=2048, **kw)
            got, code = run(p, vals, off)
            nb = int((got[0] != ref).sum())
            bad += nb + (code != 0)
            if nb or code:
                print("SHORT MISMATCH", L, K, kw, nb, code)
    # parent context, trace kernels
    ctx = np.random.default_rng(L).integers(0, 2**32, off.size - 1, dtype=np.uint64).astype(np.uint32)
    st = [("hash_lt", 0x9E3779B1, 192), ("parent_lt", ctx)]
    ref = oracle.brute(vals, off, st, "sum_i64")[0]
    p = rs.Pipeline([st[0], ("parent_lt",)], "sum_i64", grid=2, chunk=2048)
    got, code = run(p, vals, off, parent_ctx=torch.from_numpy(ctx.view(np.int32)).cuda())
    bad += int((got[0] != ref).sum()) + (code != 0)
    p = rs.Pipeline(synth.sweep_stages(2), "sum_i64", flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TRACE, grid=2, chunk=2048)
    p.set_trace(torch.zeros(1 << 20, dtype=torch.uint8, device="cuda"))
    got, code = run(p, vals, off)
    bad += int((got[0] != oracle.brute(vals, off, synth.sweep_stages(2), "sum_i64")[0]).sum()) + (code != 0)
    # element-wise exit
    for strat in ("signal", "tagged"):
        p = rs.Pipeline(synth.sweep_stages(2), "emit_value", elem="i32", strategy=strat, grid=2, chunk=2048)
        rv, rr = oracle.emit(vals, off, synth.sweep_stages(2))
        v = torch.empty(rv.size + 8, dtype=torch.int32, device="cuda")
        r = torch.empty(rv.size + 8, dtype=torch.int32, device="cuda")
        c = torch.empty(1, dtype=torch.int64, device="cuda")
        ws = p.alloc_workspace(off.size - 1, vals.size)
        p.run_emit(torch.from_numpy(vals).cuda(), torch.from_numpy(off).cuda(), v, r, c, ws)
        torch.cuda.synchronize()
        if int(c.item()) != rv.size or p.check():
            bad += 1
            print("EMIT MISMATCH", strat)
    # tree topology (SPLIT + two leaves) and the node-generated drop-count signal
    for K in (0, 2):
        st = synth.sweep_stages(K)
        ra, rb = oracle.brute_split(vals, off, st, ("hash_lt", 0x27D4EB2F, 128))
        p = rs.Pipeline(st, "split_sum_i64", split=("hash_lt", 0x27D4EB2F, 128), grid=2, chunk=2048, q0_stage=128)
        got, code = run(p, vals, off)
        nb = int((got[0] != ra).sum() + (got[1] != rb).sum())
        bad += nb + (code != 0)
        if nb or code:
            print("TREE MISMATCH", L, K, nb, code)
    st = synth.sweep_stages(2)
    kc = oracle.node_counts(vals, off, st)
    p = rs.Pipeline(st, "sum_i64_drops", grid=2, chunk=2048, q0_stage=128)
    got, code = run(p, vals, off)
    nb = int((got[0] != oracle.brute(vals, off, st, "sum_i64")[0]).sum() + (got[1] != kc[:, 0] - kc[:, 1]).sum())
    bad += nb + (code != 0)
    if nb or code:
        print("DROPS MISMATCH", L, nb, code)
# text (SWAR path) and the taxi parser
b, off = synth.text(200000, seed=3, line_mean=300.0)
for strat in ("signal", "tagged"):
    for fl in (0, rs.RS_FLAG_UNFUSED):
        p = rs.Pipeline(synth.text_stages(), "count_xor64", strategy=strat, flags=rs.RS_FLAG_STATS | fl, grid=2,
                        chunk=2048)
        got, code = run(p, b, off)
        ref = oracle.brute(b, off, synth.text_stages(), "count_xor64")
        nb = sum(int((g.view(np.uint64) != r).sum()) for g, r in zip(got, ref))
        bad += nb + (code != 0)
        if nb or code:
            print("TEXT MISMATCH", strat, fl, nb, code)
b, off, exp = synth.taxi(150, seed=4)
for strat, kw in (("signal", {}), ("tagged", {}), ("hybrid", {"tag_from": 1})):
    p = rs.Pipeline(synth.taxi_stages(), "emit_pair", strategy=strat, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_UNFUSED,
                    grid=2, chunk=2048, **kw)
    v = torch.empty(2 * exp.shape[0] + 16, dtype=torch.int32, device="cuda")
    r = torch.empty(exp.shape[0] + 8, dtype=torch.int32, device="cuda")
    c = torch.empty(1, dtype=torch.int64, device="cuda")
    ws = p.alloc_workspace(off.size - 1, b.size)
    p.run_emit(torch.from_numpy(b).cuda(), torch.from_numpy(off).cuda(), v, r, c, ws)
    torch.cuda.synchronize()
    if int(c.item()) != exp.shape[0] or p.check():
        bad += 1
        print("TAXI MISMATCH", strat)
print("done, mismatches:", bad)
