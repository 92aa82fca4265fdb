"""Per-node cycle breakdown of the sequential kernel (RS_FLAG_PROFILE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
for L, K, strat, q in [(4096, 3, "signal", 2048), (4096, 3, "signal", 1024), (4096, 1, "signal", 2048), (4096, 3, "tagged", 1024), (256, 3, "signal", 2048), (32, 3, "tagged", 1024)]:
    lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda")
    off = synth.torch_offsets(lens)
    p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat, queue_cap=q,
                    flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | rs.RS_FLAG_PROFILE)
    R = off.numel() - 1
    out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
    p.run(vals, off, out, ws); p.run(vals, off, out, ws)
    t = p.kernel_times()
    pr = p.profile()
    inst = pr[10]
    tot = sum(pr[:K + 3])
    names = ["enum"] + [f"F{i}" for i in range(1, K + 1)] + ["AGG", "TMAwait"]
    frac = " ".join(f"{n}={100*c/tot:.1f}%" for n, c in zip(names, pr[:K + 3]))
    per_inst_cyc = tot / inst
    print(f"L={L} K={K} {strat} q={q}: main={t[1]:.3f} ms  inst={inst}  cycles/inst={per_inst_cyc/1e6:.2f}M  sweeps/inst={pr[8]/inst:.0f} waits/inst={pr[9]/inst:.0f} items/sweep={N/max(1,pr[8]):.0f}  {frac}", flush=True)
