"""Occupancy experiment: configs that fit more instances per SM."""
import os, sys, statistics, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
lens = torch.full((N // 4096,), 4096, dtype=torch.int64, device="cuda")
off = synth.torch_offsets(lens)
R = off.numel() - 1
for K in (3, 1):
    for q0, q, s in [(512, 2048, 128), (256, 1024, 64), (256, 1024, 32), (128, 1024, 32), (256, 512, 32), (128, 512, 16)]:
        p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", q0_stage=q0, queue_cap=q, signal_cap=s,
                        flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | rs.RS_FLAG_PROFILE)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
        ms = []
        for i in range(3):
            p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
        pr = p.profile(); g = p.geometry()
        tot = sum(pr[:K + 3]); inst = pr[10]
        names = ["enum"] + [f"F{i}" for i in range(1, K + 1)] + ["AGG", "wait"]
        frac = " ".join(f"{n}={100*c/tot:.0f}%" for n, c in zip(names, pr[:K + 3]))
        m = statistics.median(ms[1:])
        print(f"K={K} q0={q0} q={q} s={s} inst/SM={g['grid']*g['warps_per_cta']/148:.1f} main={m:.3f}ms {(4*N+16*R)/(m/1e3)/1e9:.0f}GB/s cyc/item/inst={tot/N:.1f} items/sweep={N/max(1,pr[8]):.0f} {frac}", flush=True)
