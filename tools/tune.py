"""Config sweep for the sequential pipeline kernel (GPU box)."""
import os, sys, statistics, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs

N = 1 << 29
vals = synth.torch_values(N, "i32", seed=1)
def run(L, strategy, **cfg):
    lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda")
    off = synth.torch_offsets(lens)
    try:
        p = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy=strategy, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING, **cfg)
        R = off.numel() - 1
        out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
        ms = []
        for i in range(4):
            p.run(vals, off, out, ws)
            t = p.kernel_times()
            if i: ms.append(t[1])
        g = p.geometry()
        inst = g["grid"] * g["warps_per_cta"] / 148
        m = statistics.median(ms)
        print(f"L={L} {strategy:6s} {cfg} inst/SM={inst:.1f} main={m:.3f} ms {(4*N+16*R)/(m/1e3)/1e9:.0f} GB/s err={p.check()}", flush=True)
    except Exception as e:
        print(f"L={L} {strategy} {cfg} FAILED {e}", flush=True)

for st, q0, q, s in itertools.product(["signal"], [256, 512], [512, 1024, 2048], [32, 128]):
    run(4096, st, q0_stage=q0, queue_cap=q, signal_cap=s)
for q0, q in itertools.product([128, 256], [512, 1024]):
    run(4096, "tagged", q0_stage=q0, queue_cap=q)
