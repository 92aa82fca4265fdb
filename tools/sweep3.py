"""Three-strategy sweep (GPU box): main-kernel ms and lane fractions for fixed
and U{0..2L} region lengths, N = 2^29 int32, 3 HASH_LT stages, SUM_I64."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
scaps = [int(x) for x in os.environ.get("S_CAP", "0").split(",")]
for dist in ("fixed", "var"):
    for L in (1, 4, 32, 256, 4096):
        lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda") if dist == "fixed" else \
            synth.torch_lengths(int(N / L * 0.95), "var", L=L, seed=L)
        off = synth.torch_offsets(lens)
        R = off.numel() - 1
        row = {}
        for strat in ("signal", "tagged", "context"):
            for sc in (scaps if strat == "context" else [0]):
                p = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy=strat, signal_cap=sc,
                                flags=rs.RS_FLAG_TIMING | rs.RS_FLAG_STATS)
                out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
                ms = []
                for i in range(3 if L > 1 or strat != "signal" else 2):
                    p.run(vals, off, out, ws); ms.append(p.kernel_times()[1])
                assert p.check() == 0
                st = p.stats()
                lf = [round(float(s[2]) / max(1, 128 * int(s[0])), 3) for s in st[1:]]
                row[f"{strat}{sc or ''}"] = (round(statistics.median(ms[1:]), 3), lf)
        print(dist, L, row, flush=True)
