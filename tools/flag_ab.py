"""A/B of pipeline flag variants in one process (GPU box): main-kernel ms
(median of 5 after warm-up) per workload x strategy x variant.
Usage: python tools/flag_ab.py [extra_flag ...]   (default: UNFUSED vs fused)"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs

base = rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING
variants = {"fused": base, "unfused": base | rs.RS_FLAG_UNFUSED}


def timeit(vals, off, stages, agg, strategy, flags, **kw):
    p = rs.Pipeline(stages, agg, strategy=strategy, flags=flags, **kw)
    R = off.numel() - 1
    out = p.alloc_outputs(R)
    ws = p.alloc_workspace(R, vals.numel())
    ms = []
    for i in range(6):
        p.run(vals, off, out, ws)
        ms.append(p.kernel_times()[1])
    assert p.check() == 0
    return statistics.median(ms[1:]), p.geometry(), out


N = 1 << 29
work = []
vals = synth.torch_values(N, "i32", seed=1)
for L in [int(x) for x in os.environ.get("AB_L", "4096,256,32").split(",") if x]:
    off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device="cuda"))
    for K in (1, 3):
        work.append((f"L{L}K{K}", vals, off, synth.sweep_stages(K), "sum_i64"))
lz = synth.torch_lengths(N // 320, "zipf", seed=5)
offz = synth.torch_offsets(lz)
assert int(offz[-1]) <= N
work.append(("zipfK3", vals, offz, synth.sweep_stages(3), "sum_i64"))
for name, v, o, st, agg in work:
    for strat in ("signal", "tagged"):
        res = {}
        outs = []
        for vn, fl in variants.items():
            ms, geo, out = timeit(v, o, st, agg, strat, fl)
            res[vn] = (round(ms, 3), geo)
            outs.append(out[0].clone())
        same = all(torch.equal(outs[0], x) for x in outs[1:])
        print(name, strat, res, "same" if same else "DIFF", flush=True)
del vals
torch.cuda.empty_cache()
# graph and text
w, off = synth.torch_rmat_csr(24, 16, seed=3)
b, toff = synth.torch_text(1 << 30, seed=4)
for name, v, o, st, agg in (("graph", w, off, [("lt_u32", 1 << 31)], "count_min_u32"),
                            ("text", b, toff, synth.text_stages(), "count_xor64")):
    for strat in ("signal", "tagged"):
        res = {}
        outs = []
        for vn, fl in variants.items():
            ms, geo, out = timeit(v, o, st, agg, strat, fl)
            res[vn] = (round(ms, 3), geo)
            outs.append([x.clone() for x in out])
        same = all(all(torch.equal(a, c) for a, c in zip(outs[0], x)) for x in outs[1:])
        print(name, strat, res, "same" if same else "DIFF", flush=True)
