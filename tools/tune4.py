"""In-place ring sweep: (L, K, strategy) x q0_stage -> main-kernel ms, instances
per SM, and a parity check of each variant against the default (GPU box)."""
import os, sys, statistics, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
Ks = [int(x) for x in os.environ.get("T_K", "1,3").split(",")]
Ls = [int(x) for x in os.environ.get("T_L", "4096,256").split(",")]
Q0 = [tuple(int(y) for y in x.split("/")) for x in os.environ.get("T_Q0", "512/2048,512/4096,1024/4096,1024/8192,2048/8192").split(",")]
strats = os.environ.get("T_S", "signal,tagged").split(",")
for L, K, strat in itertools.product(Ls, Ks, strats):
    off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device="cuda"))
    R = off.numel() - 1
    res = []
    ref = None
    for q0, qc in Q0:
        try:
            p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat, q0_stage=q0, queue_cap=qc,
                            flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
            out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
            ms = []
            for i in range(5):
                p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
            assert p.check() == 0
            o = out[0].clone()
            same = "" if ref is None else ("same" if torch.equal(ref, o) else "DIFF")
            ref = o if ref is None else ref
            g = p.geometry()
            res.append((statistics.median(ms[1:]), f"{q0}/{qc}", g["grid"] * g["warps_per_cta"] // 148, same))
        except Exception as e:
            res.append((1e9, f"{q0}/{qc}", str(e)[:60], ""))
    print(f"L={L} K={K} {strat}: " + "  ".join(f"q0={a}:{m:.3f}ms i={i} {s}" for m, a, i, s in res), flush=True)
