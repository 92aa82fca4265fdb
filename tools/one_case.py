"""Run one small WS case (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2006_07478_b200 as rs
R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lens = synth.lengths(R, "var", L=20, seed=3)
off = synth.offsets(lens)
vals = (np.arange(int(off[-1]) + 1) % 1000 + 1).astype(np.int32)
stages = [("hash_lt", 0x9E3779B1, 256)]
ref = oracle.brute(vals, off, stages, "sum_i64")[0]
p = rs.Pipeline(stages, "sum_i64", strategy="signal", grid=1)
e = torch.from_numpy(vals).cuda(); o = torch.from_numpy(off).cuda()
out = p.alloc_outputs(R); ws = p.alloc_workspace(R, vals.size)
p.run(e, o, out, ws); torch.cuda.synchronize()
got = out[0].cpu().numpy()
bad = np.nonzero(got != ref)[0]
print("bad", bad.size, bad[:10], "stats", p.stats().tolist())
ws_ptr = (ws.data_ptr() + 255) & ~255
torch.cuda.synchronize()
raw = ws[(ws_ptr - ws.data_ptr()):(ws_ptr - ws.data_ptr()) + 128].cpu().numpy().view(np.uint32)
print("err", raw[1], "dbg n,lim,head,tail,spend,stamp,key,kind,shead,stail,landed,blk,ctl.tail,ctl.stail:", raw[16:30].tolist())
raw2 = ws[(ws_ptr - ws.data_ptr()) + 128:(ws_ptr - ws.data_ptr()) + 256].cpu().numpy().view(np.uint32)
print("lanes ps,pe,pc_ps,pc_pe:", raw2.reshape(-1, 4)[:8].tolist())
print("off[95:102]", off[95:102].tolist())
