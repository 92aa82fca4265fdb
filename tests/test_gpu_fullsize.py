"""Full-size parity: EVERY region of every BASELINE.json configuration, at the
sizes and in the launch configuration bench.py times, against the oracle's
plain per-region fold (run on the host cores, sharded by whole regions).

Configs (bench.workload_spec, DESIGN.md §8 input recipe):
  sweep fixed L = 4096 and U{0..8192}, N = 2^29 int32 (configs[1])
  Zipf(1.2) region lengths, N = 2^30 int32            (configs[4], 1-GPU point)
  R-MAT scale 24 CSR, 2^28 u32 edge weights           (configs[2])
  4 GiB text, lines as regions (offsets reach 2^32)   (configs[3])
  sweep fixed L = 1 and U{0..8} (L = 4), N = 2^29     (configs[1], short end: the
                                                       short-region signal kernel)
each under the signal, tagged, per-lane context (4-byte elements) and AUTO
strategies.  Integer aggregates are compared bit-exactly.
"""
import os
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def rs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2006_07478_b200 as rs
    return rs


def _host(t):
    x = t.cpu().numpy()
    return x


@pytest.mark.parametrize("workload", ["sweep_fixed_L4096", "sweep_var_L4096", "zipf", "graph", "text",
                                      "sweep_fixed_L1", "sweep_var_L4"])
def test_full_size_all_regions(rs, workload):
    import bench
    spec = bench.workload_spec(workload)
    dev = torch.device("cuda:0")
    vals, off = bench.make_inputs(spec, seed=0x5EED + 2, device=dev)
    R = off.numel() - 1
    n = int(off[-1].item() - off[0].item())
    vh = _host(vals)
    if spec["dtype"] == "u32":
        vh = vh.view(np.uint32)
    elif spec["dtype"] == "u8":
        vh = vh.view(np.uint8)
    oh = _host(off)
    if workload == "text":
        assert int(oh[-1]) == 1 << 32          # the last line ends at byte 2^32: indices past u32
    ref = oracle.brute_sharded(vh, oh, spec["stages"], spec["agg"])
    strategies = ["signal", "tagged", "auto"] + (["context"] if spec["dtype"] != "u8" else [])
    if spec["L"] and spec["L"] < 96:           # the short-region kernel (default choice) and the general one
        strategies = [("signal", 0), ("signal", rs.RS_FLAG_SHORT_OFF), "tagged"]
    for strat in strategies:
        strat, fl = strat if isinstance(strat, tuple) else (strat, 0)
        p = rs.Pipeline(spec["stages"], spec["agg"], strategy=strat, flags=rs.RS_FLAG_STATS | fl)
        out = p.alloc_outputs(R, dev)
        ws = p.alloc_workspace(R, vals.numel(), dev)
        p.run(vals, off, out, ws)
        torch.cuda.synchronize()
        assert p.check() == 0, (workload, strat)
        st = p.stats()
        assert st[0][2] == n, (workload, strat, "enumerated children != sum of region sizes")
        for k, r in enumerate(ref):
            if r is None:
                continue
            g = _host(out[k])
            g = g.view(r.dtype) if g.dtype.itemsize == r.dtype.itemsize else g.astype(r.dtype)
            bad = np.nonzero(g != r)[0]
            assert bad.size == 0, f"{workload}/{strat}: {bad.size} of {R} regions differ (output {k}), first {bad[:5]}"
        del out, ws, p
        torch.cuda.empty_cache()
    del vals, off
    torch.cuda.empty_cache()
