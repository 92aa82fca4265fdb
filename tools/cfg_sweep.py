"""Kernel time of the headline workload (sweep_fixed_L4096 unless --workload)
over ring / TMA-stage / signal-ring sizes (one GPU).  Usage:
  python tools/cfg_sweep.py [--workload W] [--strategy S] qcap:stage:scap ..."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import __graft_entry__

__graft_entry__.build()
import paper_2006_07478_b200 as rs

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="sweep_fixed_L4096")
ap.add_argument("--strategy", default="signal")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--tag-from", type=int, default=0)
ap.add_argument("cfgs", nargs="*")
a = ap.parse_args()
spec = bench.workload_spec(a.workload)
dev = torch.device("cuda:0")
vals, off = bench.make_inputs(spec, seed=0x5EED + 2, device=dev)
R = off.numel() - 1
n = int(off[-1].item() - off[0].item())
for c in (a.cfgs or ["0:0:0"]):
    q, s, sc = (int(x) for x in c.split(":"))
    try:
        p = rs.Pipeline(spec["stages"], spec["agg"], strategy=a.strategy, queue_cap=q, q0_stage=s, signal_cap=sc,
                        flags=rs.RS_FLAG_STATS | rs.RS_FLAG_TIMING | a.flags, chunk=a.chunk, tag_from=a.tag_from)
        out = p.alloc_outputs(R, dev)
        ws = p.alloc_workspace(R, vals.numel(), dev)
        for _ in range(3):
            p.run(vals, off, out, ws)
        ms = []
        for _ in range(a.reps):
            p.run(vals, off, out, ws)
            ms.append(p.kernel_times()[1])
        g = p.geometry()
        if a.profile:
            pp = rs.Pipeline(spec["stages"], spec["agg"], strategy=a.strategy, queue_cap=q, q0_stage=s, signal_cap=sc,
                             flags=rs.RS_FLAG_STATS | rs.RS_FLAG_PROFILE)
            pp.run(vals, off, out, ws)
            pr = pp.profile()
            K = len(spec["stages"])
            print("  profile cycles: enum", pr[0], "nodes", pr[1:K + 2], "tma-wait", pr[K + 2], "sweeps", pr[8],
                  "waits", pr[9], "instances", pr[10], " children/sweep", n / max(1, pr[8]), "refill", pr[11], "fence", pr[12],
                  "part_info", pr[13], "tma-issue", pr[14], "stages", pr[15], flush=True)
        t = statistics.median(ms)
        print(f"{a.workload} {a.strategy} C={a.chunk} q={q} stage={s} scap={sc}: {t:.4f} ms  {n / t / 1e6:.1f} G/s  "
              f"hbm {bench.alg_bytes(n, R, spec['agg']) / t / 1e6 / bench.hbm_peak()[0]:.3f}  err {p.check()}  {g}",
              flush=True)
        del p, out, ws
    except Exception as e:
        print(c, "failed", e, flush=True)
