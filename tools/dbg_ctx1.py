"""One failing context case with the watchdog dump (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs
L, K, unf, thr = [int(x) for x in sys.argv[1:5]]
R = max(3, (1 << 16) // L)
lens = synth.lengths(R, "var", L=L, seed=L + K)
off = synth.offsets(lens, base=3)
vals = synth.values(int(off[-1]) + 5, "i32", seed=L * 7 + K)
st = [("hash_lt", [0x9E3779B1, 0x85EBCA6B, 0xC2B2AE35, 0x27D4EB2F][k], thr) for k in range(K)]
e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
p = rs.Pipeline(st, "sum_i64", strategy="context", flags=rs.RS_FLAG_STATS | (rs.RS_FLAG_UNFUSED if unf else 0), grid=1)
out = p.alloc_outputs(R); ws = p.alloc_workspace(R, e.numel())
p.run(e, o, out, ws); torch.cuda.synchronize()
base = (ws.data_ptr() + 255) & ~255
w = ws[base - ws.data_ptr():base - ws.data_ptr() + 256].cpu().numpy().view(np.uint32)
print("err", w[1], "dump", w[16:24].tolist())
for k in range(K + 1):
    print(f"edge {k}: qh qt sh st qstart headstamp", w[24 + 6 * k:30 + 6 * k].tolist())
print("stats", p.stats().tolist())
