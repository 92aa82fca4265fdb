"""Run the D4 text workload once (for ncu): N bytes (default 2^30), strategy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2006_07478_b200 as rs
strategy = sys.argv[1] if len(sys.argv) > 1 else "signal"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
b, off = synth.torch_text(N, seed=4)
p = rs.Pipeline(synth.text_stages(), "count_xor64", strategy=strategy, flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING)
R = off.numel() - 1
out = p.alloc_outputs(R); ws = p.alloc_workspace(R, N)
for i in range(2):
    p.run(b, off, out, ws)
print("main ms", p.kernel_times()[1], p.geometry(), p.check())
