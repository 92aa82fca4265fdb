"""Signal vs tagged crossover (GPU box): main-kernel ms for fixed and variable
region lengths L and stage counts K (N = 2^28 int32, HASH_LT(192) stages,
SUM_I64).  Prints, per K, the smallest L at which the signal strategy wins."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 28
vals = synth.torch_values(N, "i32", seed=1)
Ls = [64, 128, 256, 512, 1024, 2048, 4096]
res = {}
for dist in ("fixed", "var"):
    for L in Ls:
        lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda") if dist == "fixed" else \
            synth.torch_lengths(int(N / L * 0.95), "var", L=L, seed=L)   # U{0..2L}: keep the total within N
        off = synth.torch_offsets(lens)
        R = off.numel() - 1
        for K in (0, 1, 2, 3, 4):
            t = {}
            for strat in ("signal", "tagged"):
                p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat, flags=rs.RS_FLAG_TIMING)
                out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
                ms = []
                for i in range(4):
                    p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
                assert p.check() == 0
                t[strat] = statistics.median(ms[1:])
            res[(dist, L, K)] = t
            print(dist, L, K, {k: round(v, 3) for k, v in t.items()}, flush=True)
for dist in ("fixed", "var"):
    for K in (0, 1, 2, 3, 4):
        win = [L for L in Ls if res[(dist, L, K)]["signal"] <= res[(dist, L, K)]["tagged"]]
        print(f"{dist} K={K}: signal wins at L in {win}")
