"""Chunk-size sweep (GPU box): main-kernel ms per (L, K, strategy, chunk)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
for L, K, strat in ((4096, 3, "signal"), (4096, 3, "tagged"), (256, 3, "signal"), (256, 3, "tagged"), (4096, 1, "signal")):
    off = synth.torch_offsets(torch.full((N // L,), L, dtype=torch.int64, device="cuda"))
    R = off.numel() - 1
    row = []
    for C in (4096, 8192, 16384, 32768, 65536):
        p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strat, chunk=C, flags=rs.RS_FLAG_TIMING)
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
        ms = []
        for i in range(5):
            p.run(vals, off, out, ws); ms.append(p.kernel_times())
        assert p.check() == 0
        m = statistics.median(x[1] for x in ms[1:]); tot = statistics.median(sum(x) for x in ms[1:])
        row.append(f"C={C}:{m:.3f}/{tot:.3f}")
    print(f"L={L} K={K} {strat}: " + "  ".join(row), flush=True)
