"""GPU trace-mode check: with RS_FLAG_TRACE every node logs the
Begin/End signals it consumes and each ensemble it fires.  Elements are their
own global index, so an ensemble's smallest and largest item locate all of its
items in the stream.  Per instance and node the host checks:

1. bracketing: the events match (Begin(r) ENSEMBLE* End(r))*  (
   Begin/End forwarded in stream order);
2. no mixed ensembles: every item of an ensemble lies in the open region r,
   off[r] <= item < off[r+1]  (ensemble <= credit; Lemma 1);
3. counts: the items a node consumes between Begin(r) and End(r), summed over
   the parts a region was split into, equal the oracle's k_r(n) (Lemma 1,
   P:332-336), and every region -- empty ones included -- is bracketed at
   every node (A1).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2006_07478_b200 as rs
    return rs


def _inputs(seed, R=1500):
    g = np.random.default_rng(seed)
    lens = g.integers(0, 300, R)
    lens[g.random(R) < 0.15] = 0                      # empty regions
    lens[g.integers(0, R, 6)] = g.integers(3000, 12000, 6)   # regions split across chunks
    off = synth.offsets(lens.astype(np.int64), base=int(g.integers(0, 8)))
    vals = np.arange(int(off[-1]) + 3, dtype=np.int32)    # item = its global element index
    return vals, off


def check_trace(ev, off, kc, n_nodes):
    R = off.size - 1
    inst, seq, nodetype = ev[:, 0], ev[:, 1], ev[:, 2]
    order = np.lexsort((seq, inst))
    ev = ev[order]
    count = np.zeros((n_nodes + 1, R), np.int64)
    seen = np.zeros((n_nodes + 1, R), bool)
    open_ = {}
    last_inst = None
    for e in ev:
        i, node, typ = int(e[0]), int(e[2] & 0xff), int(e[2] >> 8)
        if i != last_inst:
            assert all(v is None for v in open_.values()), f"instance {last_inst} ended inside a bracket"
            open_ = {}
            last_inst = i
        cur = open_.get(node)
        if typ == 2:                                  # BEGIN
            assert cur is None, f"node {node}: Begin inside an open bracket"
            r = int(e[4])
            assert 0 <= r < R
            if not (e[3] >> 31):
                assert int(e[3]) == r, "a whole-region key is its region id"
            open_[node] = (int(e[3]), r)
            seen[node, r] = True
        elif typ == 3:                                # END
            assert cur is not None and cur[0] == int(e[3]), f"node {node}: End without its Begin"
            open_[node] = None
        else:                                         # ENSEMBLE
            assert typ == 1
            assert cur is not None, f"node {node}: ensemble outside a bracket"
            r = cur[1]
            c, lo, hi = int(e[5]), int(e[6]), int(e[7])
            assert 0 < c <= 128
            assert off[r] <= lo <= hi < off[r + 1], f"node {node}: ensemble [{lo},{hi}] outside region {r}"
            count[node, r] += c
    assert all(v is None for v in open_.values())
    for node in range(1, n_nodes + 1):
        assert seen[node].all(), f"node {node}: {np.count_nonzero(~seen[node])} regions never bracketed"
        np.testing.assert_array_equal(count[node], kc[:, node - 1], err_msg=f"node {node} items per region")


@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("nst,cfg", [
    (2, dict()), (3, dict(chunk=2048, queue_cap=512, signal_cap=4, q0_stage=128)),
    (1, dict(grid=1, chunk=2048)), (4, dict(grid=3, chunk=4096, signal_cap=8))])
def test_trace_bracketing(rs, mode, nst, cfg):
    vals, off = _inputs(nst * 10 + (mode == "fused"))
    stages = synth.sweep_stages(nst)
    flags = rs.RS_FLAG_STATS | rs.RS_FLAG_TRACE | (rs.RS_FLAG_UNFUSED if mode == "unfused" else 0)
    p = rs.Pipeline(stages, "sum_i64", strategy="signal", flags=flags, **cfg)
    dev = torch.device("cuda:0")
    e = torch.from_numpy(vals).to(dev)
    o = torch.from_numpy(off).to(dev)
    R = off.size - 1
    buf = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    p.set_trace(buf)
    out = p.alloc_outputs(R, dev)
    ws = p.alloc_workspace(R, e.numel(), dev)
    p.run(e, o, out, ws)
    torch.cuda.synchronize()
    assert p.check() == 0
    np.testing.assert_array_equal(out[0].cpu().numpy(), oracle.brute(vals, off, stages, "sum_i64")[0])
    ev = p.read_trace()
    kc = oracle.node_counts(vals, off, stages)
    # fused: the last stage performs the aggregate's actions and logs as node nst
    n_nodes = nst if (mode == "fused" and nst >= 1) else nst + 1
    check_trace(ev, off, kc, n_nodes)
    assert set(np.unique(ev[:, 2] & 0xff)) == set(range(1, n_nodes + 1))


def test_trace_rejected_combinations(rs):
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline(synth.sweep_stages(2), "sum_i64", strategy="tagged", flags=rs.RS_FLAG_TRACE)
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    p = rs.Pipeline(synth.sweep_stages(2), "sum_i64", flags=rs.RS_FLAG_TRACE)
    o = torch.tensor([0, 4], dtype=torch.int64, device="cuda")
    v = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(rs.RSError) as e:            # no trace buffer attached
        p.run(v, o, p.alloc_outputs(1), p.alloc_workspace(1, 4))
    assert e.value.status == rs.RS_ERR_INVALID_ARG
