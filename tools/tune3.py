"""Capacity sweep for the (fused) sequential kernel: K x L x strategy x
(q0_stage, queue_cap, signal_cap) -> main-kernel ms (GPU box)."""
import os, sys, statistics, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
Ks = [int(x) for x in os.environ.get("T_K", "1,2,3").split(",")]
Ls = [int(x) for x in os.environ.get("T_L", "4096,256").split(",")]
for L, K, strat in itertools.product(Ls, Ks, ["signal", "tagged"]):
    off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device="cuda"))
    R = off.numel() - 1
    res = []
    for q0, q, s in itertools.product([256, 512], [512, 1024, 2048], [32, 128]):
        if strat == "tagged" and s != 32:
            continue
        try:
            p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat, q0_stage=q0, queue_cap=q, signal_cap=s,
                            flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
            out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
            ms = []
            for i in range(4):
                p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
            g = p.geometry()
            res.append((statistics.median(ms[1:]), q0, q, s, g["grid"] * g["warps_per_cta"] // 148))
        except Exception as e:
            res.append((1e9, q0, q, s, str(e)[:40]))
    res.sort()
    d = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat)
    print(f"L={L} K={K} {strat}: best " + "  ".join(f"{m:.3f}ms q0={a} q={b} s={c} i={i}" for m, a, b, c, i in res[:4]), flush=True)
