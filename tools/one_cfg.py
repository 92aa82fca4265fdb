"""Run one configuration (for ncu): K, q0_stage, queue_cap, signal_cap, L, strategy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
K, q0, q, s, L = (int(x) for x in sys.argv[1:6])
strategy = sys.argv[6] if len(sys.argv) > 6 else "signal"
N = 1 << 28
vals = synth.torch_values(N, "i32", seed=1)
lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda")
off = synth.torch_offsets(lens)
R = off.numel() - 1
p = rs.Pipeline(synth.sweep_stages(K), "sum_i64", strategy=strategy, q0_stage=q0, queue_cap=q, signal_cap=s,
                flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
for i in range(2):
    p.run(vals, off, out, ws)
print("main ms", p.kernel_times()[1], p.geometry())
