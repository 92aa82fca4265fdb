"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer aggregates and counts must match bit-exactly; fp32 sums within a
relative 1e-5 (north star; DESIGN.md §3 A15).  Inputs are seeded synthetic
streams with the shapes of BASELINE.json's configs (synth/).
"""
import math
import random

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

AGG_DTYPE = {"sum_i64": "i32", "sum_f32": "f32", "count_min_u32": "u32"}


@pytest.fixture(scope="module")
def rs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2006_07478_b200 as rs
    return rs


def run_gpu(rs, vals, off, stages, agg, strategy="signal", mode="seq", **cfg):
    # modes: "seq" (default: aggregate fused into the last stage), "unfused"
    # (separate AGGREGATE node, the paper's node structure)
    flags = rs.RS_FLAG_STATS | {"unfused": rs.RS_FLAG_UNFUSED}.get(mode, 0)
    p = rs.Pipeline(stages, agg, strategy=strategy, flags=flags, **cfg)
    dev = torch.device("cuda:0")
    e = torch.from_numpy(np.ascontiguousarray(vals)).to(dev)
    o = torch.from_numpy(np.ascontiguousarray(off)).to(dev)
    R = off.size - 1
    out = p.alloc_outputs(R, dev)
    ws = p.alloc_workspace(R, e.numel(), dev)
    p.run(e, o, out, ws)
    torch.cuda.synchronize()
    code = p.check()
    assert code == 0, f"device error {code}"
    res = [t.cpu().numpy() if t is not None else None for t in out]
    if agg == "count_min_u32":
        res = [r.view(np.uint32) for r in res]
    return res, p.stats(), p


def assert_parity(got, ref, agg):
    if agg == "sum_f32":
        r = ref[0]
        g = got[0].astype(np.float64)
        err = np.abs(g - r)
        tol = 1e-5 * np.abs(r)
        bad = np.nonzero(err > tol)[0]
        assert bad.size == 0, f"{bad.size} fp32 regions out of tolerance, e.g. r={bad[:3]} got={g[bad[:3]]} ref={r[bad[:3]]}"
    else:
        for g, r in zip(got, ref):
            if r is None:
                continue
            bad = np.nonzero(g != r)[0]
            assert bad.size == 0, f"{bad.size} regions differ, first {bad[:5]} got {g[bad[:5]]} ref {r[bad[:5]]}"


@pytest.mark.parametrize("strategy", ["signal", "tagged"])
def test_tiny_d1(rs, strategy):
    vals, off, stages, agg = synth.tiny()
    ref = oracle.brute(vals, off, stages, agg)
    got, st, _ = run_gpu(rs, vals, off, stages, agg, strategy, chunk=8192)   # uniform chunks (no finer tail)
    assert_parity(got, ref, agg)
    kc = oracle.node_counts(vals, off, stages)
    assert st[0][2] == off[-1] - off[0]                      # enumerated children = sum of sizes
    for j in range(len(stages) + 1):
        assert st[j + 1][2] == kc[:, j].sum()                # items reaching each node
    if strategy == "signal":
        # Begin + End per region part: regions crossing a chunk boundary are
        # split into one part per chunk they touch (A18)
        C = 8192
        b = np.arange(C, int(off[-1]), C)
        splits = sum(int(((off[:-1] < x) & (off[1:] > x)).sum()) for x in b)
        assert st[0][3] == 2 * (off.size - 1 + splits)
        bound = oracle.occupancy_bound(kc, 128)
        for j in range(len(stages) + 1):
            lane = st[j + 1][2] / (128 * st[j + 1][0])
            assert lane <= bound[j] + 1e-12


def _case(seed, agg, R=None, dist=None, L=None, base=None):
    rnd = random.Random(seed)
    R = R if R is not None else rnd.choice([1, 7, 100, 1000, 5000])
    dist = dist or rnd.choice(["fixed", "var", "uniform", "zipf"])
    L = L if L is not None else rnd.choice([0, 1, 3, 17, 128, 129, 700, 5000])
    lens = synth.lengths(R, dist, L=L, lo=0, hi=max(1, 2 * L), seed=seed, zipf_max=max(2, L))
    base = base if base is not None else rnd.choice([0, 1, 2, 3, 5])
    off = synth.offsets(lens, base=base)
    vals = synth.values(int(off[-1]) + rnd.randint(0, 7), AGG_DTYPE[agg], seed=seed + 1)
    nst = rnd.randint(0, 4)
    stages = []
    for k in range(nst):
        if agg == "count_min_u32":
            stages.append(("lt_u32", rnd.choice([0, 1 << 31, 1 << 32, rnd.getrandbits(32)])))
        elif agg == "sum_f32" and rnd.random() < 0.4:
            stages.append(("scale_f32", 3.14))
        elif agg == "sum_i64" and rnd.random() < 0.3:
            stages.append(("affine_i32", rnd.getrandbits(32), rnd.getrandbits(32)))
        else:
            stages.append(("hash_lt", rnd.getrandbits(32) | 1, rnd.choice([0, 64, 192, 256])))
    return vals, off, stages


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("strategy", ["signal", "tagged", "context"])
@pytest.mark.parametrize("mode", ["seq", "unfused"])
def test_random_parity(rs, seed, strategy, mode):
    agg = ["sum_i64", "sum_f32", "count_min_u32"][seed % 3]
    vals, off, stages = _case(seed, agg)
    rnd = random.Random(seed * 7 + 1)
    cfg = dict(chunk=rnd.choice([2048, 4096, 8192]), grid=rnd.choice([0, 0, 1, 3]),
               queue_cap=rnd.choice([256, 512]), signal_cap=rnd.choice([4, 16, 128]),
               q0_stage=rnd.choice([0, 128, 256]))   # in-place rings down to 512 items (heavy relocation)
    if strategy == "context":
        cfg["signal_cap"] = rnd.choice([4, 32, 64, 512])
    ref = oracle.brute(vals, off, stages, agg)
    got, st, _ = run_gpu(rs, vals, off, stages, agg, strategy, mode, **cfg)
    assert_parity(got, ref, agg)
    assert st[0][2] == off[-1] - off[0]


@pytest.mark.parametrize("strategy", ["signal", "tagged", "context"])
@pytest.mark.parametrize("L", [1, 4, 32, 127, 128, 129, 256, 4096, 100000])
@pytest.mark.parametrize("mode", ["seq", "unfused"])
def test_region_lengths(rs, strategy, L, mode):
    """Region lengths 1..4096 (north star) plus regions far longer than a chunk."""
    N = 1 << 18
    R = max(1, N // L)
    for dist in ("fixed", "var"):
        lens = synth.lengths(R, dist, L=L, seed=L)
        off = synth.offsets(lens, base=3)
        vals = synth.values(int(off[-1]), "i32", seed=L + 5)
        stages = synth.sweep_stages(3)
        ref = oracle.brute(vals, off, stages, "sum_i64")
        got, st, _ = run_gpu(rs, vals, off, stages, "sum_i64", strategy, mode)
        assert_parity(got, ref, "sum_i64")


@pytest.mark.parametrize("strategy", ["signal", "tagged", "context"])
def test_empty_and_degenerate(rs, strategy):
    stages = synth.sweep_stages(2)
    # all regions empty (N = 0)
    off = np.zeros(50, np.int64)
    got, st, _ = run_gpu(rs, np.zeros(4, np.int32), off, stages, "sum_i64", strategy)
    assert (got[0] == 0).all()
    # a single element; a single huge region; empty regions at chunk boundaries
    for lens in ([1], [300000], [0] * 3 + [8192 - 3] + [0] * 5 + [8192] + [0, 0, 1]):
        off = synth.offsets(np.array(lens, np.int64), base=0)
        vals = synth.values(int(off[-1]) + 1, "i32", seed=1)
        ref = oracle.brute(vals, off, stages, "sum_i64")
        got, _, _ = run_gpu(rs, vals, off, stages, "sum_i64", strategy, chunk=2048)
        assert_parity(got, ref, "sum_i64")
    # count/min identity for empty regions: count 0, min 0xFFFFFFFF
    off = np.array([0, 0, 3, 3], np.int64)
    vals = np.array([5, 2, 9, 0], np.uint32)
    got, _, _ = run_gpu(rs, vals, off, [("lt_u32", 1 << 32)], "count_min_u32", strategy)
    assert list(got[0]) == [0, 3, 0] and list(got[1]) == [0xFFFFFFFF, 2, 0xFFFFFFFF]


def test_strategies_bit_identical(rs):
    """Signal and tagged strategies give bit-identical integer aggregates."""
    lens = synth.lengths(20000, "zipf", seed=3, zipf_max=4096)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", 4)
    stages = synth.sweep_stages(3)
    a, _, _ = run_gpu(rs, vals, off, stages, "sum_i64", "signal")
    b, _, _ = run_gpu(rs, vals, off, stages, "sum_i64", "tagged")
    c, _, _ = run_gpu(rs, vals, off, stages, "sum_i64", "context")
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[0], c[0])


def test_batching_invariance(rs):
    """Aggregates do not depend on batching: sub-ranges of the parent stream
    with offsets[0] != 0 over the same element array reproduce the full run."""
    lens = synth.lengths(30000, "var", L=60, seed=8)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", 9)
    stages = synth.sweep_stages(3)
    full, _, _ = run_gpu(rs, vals, off, stages, "sum_i64")
    parts = []
    for a, b in ((0, 1), (1, 9999), (9999, 10000), (10000, 30000)):
        g, _, _ = run_gpu(rs, vals, off[a:b + 1], stages, "sum_i64")
        parts.append(g[0])
    np.testing.assert_array_equal(np.concatenate(parts), full[0])


def test_grid_and_capacity_invariance(rs):
    lens = synth.lengths(5000, "var", L=40, seed=11)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", 12)
    stages = synth.sweep_stages(3)
    ref = oracle.brute(vals, off, stages, "sum_i64")
    for cfg in (dict(grid=1), dict(grid=2, chunk=2048), dict(queue_cap=1024, signal_cap=8), dict(signal_cap=4),
                dict(queue_cap=256), dict(q0_stage=128, queue_cap=256), dict(q0_stage=128, queue_cap=1024),
                dict(q0_stage=2048, queue_cap=16384, chunk=2048)):
        for strat in ("signal", "tagged"):
            for mode in ("seq", "unfused"):
                got, _, _ = run_gpu(rs, vals, off, stages, "sum_i64", strat, mode, **cfg)
                assert_parity(got, ref, "sum_i64")


@pytest.mark.parametrize("R", [32, 64, 96, 128, 256, 512, 1024])
@pytest.mark.parametrize("mode", ["seq", "unfused"])
def test_occupancy_closed_form_gpu(rs, R, mode):
    """One instance (grid=1), fixed regions dividing the chunk, pass-all
    stages, full-first: the aggregate's lane fraction equals R/(w ceil(R/w))
    exactly, as the oracle's interpreter gives."""
    nreg = (1 << 16) // R
    off = np.arange(0, nreg * R + 1, R, dtype=np.int64)
    vals = synth.values(int(off[-1]), "i32", R)
    stages = [("hash_lt", 0x9E3779B1, 256)] * 2
    chunk = 1 << max(11, int(off[-1] - 1).bit_length())     # one chunk: no region is split
    got, st, _ = run_gpu(rs, vals, off, stages, "sum_i64", "signal", mode, grid=1, chunk=chunk)
    ref = oracle.interp(vals, off, stages, "sum_i64", w=128, qcap=1024, scap=256)
    np.testing.assert_array_equal(got[0], ref["out"][0])
    num, den = R, 128 * math.ceil(R / 128)
    for n in range(1, len(stages) + 2):
        assert st[n][2] * den == st[n][0] * 128 * num, (n, st[n])
        assert st[n][0] == ref["stats"][n][0]


def test_tagged_full_ensembles(rs):
    """Tagged strategy keeps ensembles full regardless of region length."""
    lens = synth.lengths(1 << 16, "fixed", L=3)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", 2)
    got, st, _ = run_gpu(rs, vals, off, [("hash_lt", 3, 256)], "sum_i64", "tagged", grid=1)
    assert st[1][1] >= st[1][0] - 2       # all but the stream-tail ensembles are full


def test_validate_flag_catches_bad_offsets(rs):
    vals = synth.values(100, "i32", 0)
    off = np.array([0, 50, 40, 100], np.int64)
    p = rs.Pipeline([], "sum_i64", flags=rs.RS_FLAG_STATS | rs.RS_FLAG_VALIDATE)
    e = torch.from_numpy(vals).cuda()
    o = torch.from_numpy(off).cuda()
    out = p.alloc_outputs(3)
    ws = p.alloc_workspace(3, 100)
    p.run(e, o, out, ws)
    torch.cuda.synchronize()
    with pytest.raises(rs.RSError):
        p.check()
    # offsets beyond n_elems are caught even without VALIDATE (no out-of-bounds TMA)
    p2 = rs.Pipeline([], "sum_i64")
    o2 = torch.tensor([0, 50, 200], dtype=torch.int64, device="cuda")
    out2 = p2.alloc_outputs(2)
    ws2 = p2.alloc_workspace(2, 100)
    p2.run(e, o2, out2, ws2)
    torch.cuda.synchronize()
    with pytest.raises(rs.RSError):
        p2.check()


def test_run_host_e2e(rs):
    vals, off, stages, agg = synth.tiny()
    ref = oracle.brute(vals, off, stages, agg)[0]
    p = rs.Pipeline(stages, agg)
    out = np.zeros(off.size - 1, np.int64)
    p.run_host(vals, off, out)
    np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("strategy", ["signal", "tagged"])
def test_full_size_sampled(rs, strategy):
    """BASELINE config sizes in the bench launch configuration: N = 2^29 int32
    children, L = 4096 (and Zipf), 3 filters; oracle on sampled regions plus
    the device-side child-count invariant."""
    N = 1 << 29
    for dist, L in (("fixed", 4096), ("zipf", 0)):
        if dist == "fixed":
            lens = torch.full((N // L,), L, dtype=torch.int64, device="cuda")
        else:
            lens = synth.torch_lengths(N // 208, "zipf", seed=5, device="cuda")
        off = synth.torch_offsets(lens)
        n = int(off[-1].item())
        vals = synth.torch_values(n, "i32", seed=7, device="cuda")
        stages = synth.sweep_stages(3)
        p = rs.Pipeline(stages, "sum_i64", strategy=strategy)
        R = off.numel() - 1
        out = p.alloc_outputs(R)
        ws = p.alloc_workspace(R, n)
        p.run(vals, off, out, ws)
        torch.cuda.synchronize()
        assert p.check() == 0
        st = p.stats()
        assert st[0][2] == n
        rng = np.random.default_rng(1)
        idx = np.unique(np.concatenate([rng.integers(0, R, 400), [0, R - 1]]))
        off_h = off.cpu().numpy()
        got = out[0].cpu().numpy()
        for r in idx:
            a, b = int(off_h[r]), int(off_h[r + 1])
            v = vals[a:b].cpu().numpy()
            ref = oracle.brute(v, np.array([0, b - a], np.int64), stages, "sum_i64")[0][0]
            assert got[r] == ref, (dist, r)
        del vals, off, out, ws
        torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["seq", "unfused"])
@pytest.mark.parametrize("strategy", ["signal", "tagged"])
@pytest.mark.parametrize("line_mean,cls,base,chunk", [
    (1397.0, b"{", 0, 8192), (1397.0, b"{", 7, 2048), (20.0, b"{0123456789", 13, 2048), (5000.0, b"", 3, 2048),
    (64.0, bytes(range(48, 58)) + b"{", 1, 2048)])
def test_text_count_xor64(rs, strategy, line_mean, cls, base, chunk, mode):
    """D4 shape: byte stream split on newlines, CLASS filter, COUNT + XOR64 of
    mix64(i << 8 | byte) per line (reading A19) -- bit-exact; lines longer than
    a chunk, unaligned starts (16-byte TMA blocks), and no filter at all (the
    aggregate reads the byte ring directly)."""
    b, off = synth.text(400000, seed=int(line_mean) + base, line_mean=line_mean)
    if base:
        b = np.concatenate([np.full(base, ord("x"), np.uint8), b])
        off = off + base
    stages = [("class", synth.class_table(cls))] if cls else []
    ref = oracle.brute(b, off, stages, "count_xor64")
    got, st, _ = run_gpu(rs, b, off, stages, "count_xor64", strategy, mode, chunk=chunk)
    got = [g.view(np.uint64) for g in got]
    assert_parity(got, ref, "count_xor64")
    assert st[0][2] == off[-1] - off[0]


@pytest.mark.parametrize("mode", ["seq", "unfused"])
@pytest.mark.parametrize("strategy", ["signal", "tagged"])
def test_graph_rmat_count_min(rs, strategy, mode):
    """D3 shape: edges grouped by source vertex of an R-MAT graph (skewed
    degrees: most vertices empty, a few with thousands of edges spanning
    chunks), LT(2^31) weight filter, COUNT + MIN per vertex -- bit-exact."""
    w, off = synth.torch_rmat_csr(16, 16, seed=5, device="cuda")
    wv = w.cpu().numpy().view(np.uint32)
    offh = off.cpu().numpy()
    stages = [("lt_u32", 1 << 31)]
    ref = oracle.brute(wv, offh, stages, "count_min_u32")
    got, st, _ = run_gpu(rs, wv, offh, stages, "count_min_u32", strategy, mode, chunk=2048)
    assert_parity(got, ref, "count_min_u32")
    assert (np.diff(offh) == 0).mean() > 0.3          # R-MAT: many isolated vertices


@pytest.mark.parametrize("L", [16, 3000])
def test_auto_strategy(rs, L):
    """RS_STRATEGY_AUTO: short regions run tagged, long
    regions signal; either way the aggregates equal the oracle's."""
    lens = synth.lengths(max(4, (1 << 17) // L), "fixed", L=L, seed=2)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", seed=3)
    stages = synth.sweep_stages(3)
    ref = oracle.brute(vals, off, stages, "sum_i64")
    got, st, p = run_gpu(rs, vals, off, stages, "sum_i64", "auto")
    assert_parity(got, ref, "sum_i64")
    assert p.last_strategy() == ("tagged" if L < 768 else "signal")
    assert st[0][2] == off[-1] - off[0]


@pytest.mark.parametrize("thr", [0, 1, 64, 256])
@pytest.mark.parametrize("L", [1, 3, 40, 300])
def test_context_empty_region_runs(rs, thr, L):
    """Per-lane context strategy under runs of empty regions:
    heavy filters leave most regions without survivors, so many boundaries share
    a stamp and fill the boundary queues (reading R3 cuts ensembles / fires
    partials under that pressure); aggregates, counts and per-node items exact."""
    lens = synth.lengths(max(8, (1 << 16) // L), "var", L=L, seed=L + thr)
    off = synth.offsets(lens, base=1)
    vals = synth.values(int(off[-1]) + 3, "i32", seed=thr + 1)
    stages = [("hash_lt", 0x9E3779B1, thr), ("hash_lt", 0x85EBCA6B, 192)]
    for agg in ("sum_i64", "sum_f32", "count_min_u32"):
        v = synth.values(int(off[-1]) + 3, AGG_DTYPE[agg], seed=thr + 2) if agg != "sum_i64" else vals
        st = stages if agg != "count_min_u32" else [("lt_u32", thr << 24), ("lt_u32", 3 << 30)]
        ref = oracle.brute(v, off, st, agg)
        for mode, scap in (("seq", 256), ("unfused", 256), ("seq", 8), ("unfused", 32)):
            got, stt, _ = run_gpu(rs, v, off, st, agg, "context", mode, grid=1, signal_cap=scap)
            assert_parity(got, ref, agg)
            kc = oracle.node_counts(v, off, st)
            for j in range(len(st) + 1):
                assert stt[j + 1][2] == kc[:, j].sum()


def test_comm_world1_gather_and_barrier(rs):
    """The C ABI's NCCL gather at world size 1 (the box has one GPU): the root's
    own slice is placed at its region base; barrier and destroy work."""
    uid = rs.Comm.unique_id()
    c = rs.Comm(uid, 0, 1)
    try:
        loc = (torch.arange(100, dtype=torch.int64, device="cuda") * 3, None)
        root = (torch.full((100,), -1, dtype=torch.int64, device="cuda"), None)
        c.gather("sum_i64", loc, [0, 100], root, root=0)
        c.barrier()
        torch.cuda.synchronize()
        assert torch.equal(root[0], loc[0])
        cnt = (torch.arange(7, dtype=torch.int32, device="cuda"), torch.arange(7, 14, dtype=torch.int32, device="cuda"))
        rc = (torch.zeros(7, dtype=torch.int32, device="cuda"), torch.zeros(7, dtype=torch.int32, device="cuda"))
        c.gather("count_min_u32", cnt, [0, 7], rc, root=0)
        torch.cuda.synchronize()
        assert torch.equal(rc[0], cnt[0]) and torch.equal(rc[1], cnt[1])
        # local_regions that disagrees with region_base is rejected before any NCCL call
        import ctypes as C
        base = (C.c_int64 * 2)(0, 50)
        agg = rs.rs_aggregates(loc[0].data_ptr(), None)
        st = rs.lib().rs_gather_aggregates(c.h, rs.OPS["sum_i64"], agg, 100, base,
                                           rs.rs_aggregates(root[0].data_ptr(), None), 0, None)
        assert st == rs.RS_ERR_INVALID_ARG
    finally:
        c.close()


def test_ipc_export_offset(rs):
    """rs_ipc_export reports the buffer's offset inside its allocation (the
    caching allocator hands out sub-ranges), so a peer maps base + offset."""
    big = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    sub = big[4096:]
    h, off = rs.ipc_export(sub.data_ptr())
    assert len(h) == 64 and off >= 4096 and (off - 4096) == rs.ipc_export(big.data_ptr())[1]


def test_parent_context_signal(rs):
    """PARENT_LT (getParent, Fig. 5): each item is kept iff
    it is below its region's context value -- bit-exact against the oracle, with
    regions split across chunks (the context of a split region is loaded by
    every part) and empty regions."""
    g = np.random.default_rng(5)
    lens = synth.lengths(3000, "zipf", seed=9, zipf_max=6000)
    lens[::11] = 0
    off = synth.offsets(lens, base=3)
    vals = synth.values(int(off[-1]) + 2, "i32", seed=10)
    ctx = g.integers(0, 2**32, off.size - 1, dtype=np.uint64).astype(np.uint32)
    for stages in ([("parent_lt", ctx)], [("hash_lt", 0x9E3779B1, 192), ("parent_lt", ctx)],
                   [("parent_lt", ctx), ("hash_lt", 0x85EBCA6B, 192), ("parent_lt", ctx)]):
        ref = oracle.brute(vals, off, stages, "sum_i64")
        dev_stages = [s if s[0] != "parent_lt" else ("parent_lt",) for s in stages]
        for mode in ("seq", "unfused"):
            flags = rs.RS_FLAG_STATS | (rs.RS_FLAG_UNFUSED if mode == "unfused" else 0)
            p = rs.Pipeline(dev_stages, "sum_i64", strategy="signal", flags=flags, chunk=2048)
            e = torch.from_numpy(vals).cuda()
            o = torch.from_numpy(off).cuda()
            cx = torch.from_numpy(ctx.view(np.int32)).cuda()
            R = off.size - 1
            out = p.alloc_outputs(R)
            ws = p.alloc_workspace(R, e.numel())
            p.run(e, o, out, ws, parent_ctx=cx)
            torch.cuda.synchronize()
            assert p.check() == 0
            np.testing.assert_array_equal(out[0].cpu().numpy(), ref[0])
            with pytest.raises(rs.RSError):       # the context array is required
                p.run(e, o, out, ws)
    with pytest.raises(rs.RSError) as ex:
        rs.Pipeline([("parent_lt",)], "sum_i64", strategy="tagged")
    assert ex.value.status == rs.RS_ERR_UNSUPPORTED


def test_auto_decides_on_call_children(rs):
    """AUTO decides from the call's own children count off[R] - off[0], not
    from the array bound (a one-region batch over a large array runs the
    strategy its own length calls for)."""
    lens = synth.lengths(4000, "fixed", L=16)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]) + (1 << 22), "i32", seed=4)      # array far longer than the regions
    stages = synth.sweep_stages(3)
    got, _, p = run_gpu(rs, vals, off, stages, "sum_i64", "auto")
    assert p.last_strategy() == "tagged"
    assert_parity(got, oracle.brute(vals, off, stages, "sum_i64"), "sum_i64")


@pytest.mark.parametrize("strategy", ["signal", "tagged", "auto"])
@pytest.mark.parametrize("mode", ["seq", "unfused"])
def test_emit_elementwise_exit(rs, strategy, mode):
    """RS_NODE_EMIT: every surviving item leaves the
    pipeline as (value, region) -- compared with the oracle as a multiset (the
    order across instances is unspecified), with split and empty regions,
    transforms before the exit, and the count / overflow contract."""
    lens = synth.lengths(6000, "zipf", seed=13, zipf_max=9000)
    lens[::9] = 0
    off = synth.offsets(lens, base=5)
    vals = synth.values(int(off[-1]) + 3, "i32", seed=14)
    for stages in ([], [("hash_lt", 0x9E3779B1, 192)], synth.sweep_stages(3) + [("affine_i32", 5, 11)]):
        ref_v, ref_r = oracle.emit(vals, off, stages)
        flags = rs.RS_FLAG_STATS | (rs.RS_FLAG_UNFUSED if mode == "unfused" else 0)
        p = rs.Pipeline(stages, "emit_value", elem="i32", strategy=strategy, flags=flags, chunk=2048)
        e = torch.from_numpy(vals).cuda()
        o = torch.from_numpy(off).cuda()
        R = off.size - 1
        cap = int(ref_v.size) + 16
        v = torch.empty(cap, dtype=torch.int32, device="cuda")
        r = torch.empty(cap, dtype=torch.int32, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        ws = p.alloc_workspace(R, e.numel())
        p.run_emit(e, o, v, r, cnt, ws)
        torch.cuda.synchronize()
        assert p.check() == 0
        n = int(cnt.item())
        assert n == ref_v.size
        got = np.stack([r[:n].cpu().numpy().view(np.uint32), v[:n].cpu().numpy().view(np.uint32)], 1)
        exp = np.stack([ref_r, ref_v], 1)
        got = got[np.lexsort((got[:, 1], got[:, 0]))]
        exp = exp[np.lexsort((exp[:, 1], exp[:, 0]))]
        np.testing.assert_array_equal(got, exp)
        st = p.stats()
        assert st[0][2] == off[-1] - off[0]
        # overflow: the count reports every survivor, check() reports code 8
        if ref_v.size > 10:
            small = 10
            p.run_emit(e, o, v[:small], r[:small], cnt, ws)
            torch.cuda.synchronize()
            assert int(cnt.item()) == ref_v.size
            with pytest.raises(rs.RSError):
                p.check()
    with pytest.raises(rs.RSError):          # an EMIT pipeline does not run through rs_pipeline_run
        p.run(e, o, (v, None), ws)


@pytest.mark.parametrize("strategy", ["signal", "tagged"])
@pytest.mark.parametrize("mode", ["seq", "unfused"])
@pytest.mark.parametrize("stage1", [True, False])
def test_taxi_two_stage(rs, strategy, mode, stage1):
    """The taxi-style two-stage app: lines of text are
    the regions; stage 1 keeps the '{' bytes (CLASS), stage 2 verifies and
    parses each "{x,y}" (reading from the byte stream, so pairs may cross
    chunk boundaries), swaps it and emits (line, y, x).  Compared as a
    multiset with the oracle and with the pairs the corpus generator wrote."""
    b, off, exp = synth.taxi(800, seed=21)
    b = np.concatenate([np.full(3, ord("x"), np.uint8), b])     # unaligned stream start
    off = off + 3
    stages = synth.taxi_stages() if stage1 else []
    yx, r = oracle.emit_pair(b, off, stages)
    np.testing.assert_array_equal(np.stack([r, yx[:, 0], yx[:, 1]], 1), exp)
    flags = rs.RS_FLAG_STATS | (rs.RS_FLAG_UNFUSED if mode == "unfused" else 0)
    p = rs.Pipeline(stages, "emit_pair", strategy=strategy, flags=flags, chunk=2048)
    e = torch.from_numpy(b).cuda()
    o = torch.from_numpy(off).cuda()
    R = off.size - 1
    cap = exp.shape[0] + 8
    v = torch.empty(2 * cap, dtype=torch.int32, device="cuda")
    rg = torch.empty(cap, dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    ws = p.alloc_workspace(R, e.numel())
    p.run_emit(e, o, v, rg, cnt, ws)
    torch.cuda.synchronize()
    assert p.check() == 0
    n = int(cnt.item())
    assert n == exp.shape[0]
    vv = v[:2 * n].cpu().numpy().view(np.uint32).reshape(n, 2)
    got = np.stack([rg[:n].cpu().numpy().view(np.uint32), vv[:, 0], vv[:, 1]], 1)
    got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
    ref = exp[np.lexsort((exp[:, 2], exp[:, 1], exp[:, 0]))]
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("nst,tag_from,mode", [(1, 1, "unfused"), (2, 1, "seq"), (3, 1, "seq"), (3, 2, "seq"),
                                              (3, 3, "unfused"), (4, 2, "unfused"), (4, 3, "seq")])
def test_hybrid_per_stage(rs, nst, tag_from, mode):
    """RS_STRATEGY_HYBRID: signals up to
    edge tag_from, tags after it.  Bit-identical integer aggregates with the
    oracle over short, long, empty and chunk-spanning regions; the stages
    before the converter keep the signal strategy's ensembles (bounded by
    regions) and the stages after it run full ensembles like the tagged one."""
    for L, dist in ((40, "var"), (700, "fixed"), (3000, "var")):
        lens = synth.lengths(max(8, (1 << 17) // L), dist, L=L, seed=L + nst)
        off = synth.offsets(lens, base=2)
        vals = synth.values(int(off[-1]) + 5, "i32", seed=L + 1)
        stages = synth.sweep_stages(nst)
        ref = oracle.brute(vals, off, stages, "sum_i64")
        got, st, _ = run_gpu(rs, vals, off, stages, "sum_i64", "hybrid", mode, tag_from=tag_from, chunk=2048,
                             queue_cap=1024 if L == 40 else 0)
        assert_parity(got, ref, "sum_i64")
        kc = oracle.node_counts(vals, off, stages)
        assert st[0][2] == off[-1] - off[0]
        for j in range(nst + (1 if mode == "unfused" else 0)):
            assert st[j + 1][2] == kc[:, j].sum()
        if L == 40:
            # after the converter, ensembles are full except at chunk / stream tails
            n_after = tag_from + 1
            if n_after <= nst or mode == "unfused":
                d, f = st[n_after][0], st[n_after][1]
                assert f >= 0.8 * d, (n_after, st[n_after])
    with pytest.raises(rs.RSError):
        rs.Pipeline(synth.sweep_stages(2), "sum_i64", strategy="hybrid", tag_from=2)   # fused: tag_from <= 1


@pytest.mark.parametrize("mode", ["unfused"])
def test_taxi_hybrid(rs, mode):
    """The paper's best taxi variant: stage 1 (the '{' filter)
    runs signal-delimited, stage 2 (parse + emit) runs on tagged items."""
    b, off, exp = synth.taxi(600, seed=23)
    p = rs.Pipeline(synth.taxi_stages(), "emit_pair", strategy="hybrid", tag_from=1,
                    flags=rs.RS_FLAG_STATS | rs.RS_FLAG_UNFUSED, chunk=2048, grid=1)   # one instance: no early drain
    e = torch.from_numpy(b).cuda()
    o = torch.from_numpy(off).cuda()
    R = off.size - 1
    cap = exp.shape[0] + 8
    v = torch.empty(2 * cap, dtype=torch.int32, device="cuda")
    rg = torch.empty(cap, dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    ws = p.alloc_workspace(R, e.numel())
    p.run_emit(e, o, v, rg, cnt, ws)
    torch.cuda.synchronize()
    assert p.check() == 0
    n = int(cnt.item())
    assert n == exp.shape[0]
    vv = v[:2 * n].cpu().numpy().view(np.uint32).reshape(n, 2)
    got = np.stack([rg[:n].cpu().numpy().view(np.uint32), vv[:, 0], vv[:, 1]], 1)
    got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
    ref = exp[np.lexsort((exp[:, 2], exp[:, 1], exp[:, 0]))]
    np.testing.assert_array_equal(got, ref)
    st = p.stats()
    assert st[2][1] >= 0.9 * st[2][0]          # stage 2 on tagged items: full ensembles
    assert st[1][1] >= 0.8 * st[1][0]          # stage 1 (long lines, signal-delimited): mostly full (91%)


@pytest.mark.parametrize("nst", [0, 1, 2])
@pytest.mark.parametrize("L,dist", [(3, "var"), (200, "zipf"), (5000, "var")])
def test_tree_fanout(rs, nst, L, dist):
    """Tree topology (Fig. 1b): a SPLIT node routes each
    item to leaf A or leaf B; every Begin/End reaches both leaves with per-child
    credits.  Both leaves' per-region sums equal the oracle's, bit-exactly, over
    short, skewed and chunk-spanning regions with empty ones; every region is
    bracketed at both leaves (each leaf consumes 2 signals per region part)."""
    lens = synth.lengths(max(8, (1 << 17) // L), dist, L=L, seed=L + nst, zipf_max=max(2, 2 * L))
    lens[::7] = 0
    off = synth.offsets(lens, base=1)
    vals = synth.values(int(off[-1]) + 2, "i32", seed=nst + 3)
    stages = synth.sweep_stages(nst)
    split = ("hash_lt", 0x27D4EB2F, 128)
    ra, rb = oracle.brute_split(vals, off, stages, split)
    for cfg in (dict(chunk=2048), dict(chunk=4096, queue_cap=256, signal_cap=4, q0_stage=128, grid=2)):
        p = rs.Pipeline(stages, "split_sum_i64", split=split, **cfg)
        e = torch.from_numpy(vals).cuda()
        o = torch.from_numpy(off).cuda()
        R = off.size - 1
        out = p.alloc_outputs(R)
        ws = p.alloc_workspace(R, e.numel())
        p.run(e, o, out, ws)
        torch.cuda.synchronize()
        assert p.check() == 0
        np.testing.assert_array_equal(out[0].cpu().numpy(), ra)
        np.testing.assert_array_equal(out[1].cpu().numpy(), rb)
        st = p.stats()
        assert st.shape[0] == nst + 4
        kc = oracle.node_counts(vals, off, stages)
        assert st[nst + 1][2] == kc[:, nst].sum()                 # the split consumes the survivors
        assert st[nst + 2][2] + st[nst + 3][2] == kc[:, nst].sum()  # and partitions them
        assert st[nst + 2][3] == st[nst + 3][3] == st[nst + 1][3]   # both children see every signal


def test_tree_rejected_shapes(rs):
    with pytest.raises(rs.RSError):
        rs.Pipeline(synth.sweep_stages(3), "split_sum_i64", split=("hash_lt", 3, 100))   # > 2 stages before SPLIT
    with pytest.raises(rs.RSError):
        rs.Pipeline([], "split_sum_i64", split=("hash_lt", 3, 100), strategy="tagged")


@pytest.mark.parametrize("mode,nst", [("seq", 2), ("seq", 3), ("unfused", 1), ("unfused", 3)])
def test_node_generated_signal(rs, mode, nst):
    """A node-generated signal ("a node ... may also
    generate additional signals"): the first stage counts the items it drops
    in each region and announces the count with a signal of its own just
    before End; the later stages forward it in stream position (credits) and
    the aggregate records it.  v0 = the oracle's sums, v1 = items reaching
    stage 1 minus items leaving it (oracle node counts), per region, with
    regions split across chunks (parts add up in the fixup) and empty ones."""
    lens = synth.lengths(3000, "zipf", seed=nst + 11, zipf_max=7000)
    lens[::5] = 0
    off = synth.offsets(lens, base=2)
    vals = synth.values(int(off[-1]) + 1, "i32", seed=nst)
    stages = synth.sweep_stages(nst)
    ref = oracle.brute(vals, off, stages, "sum_i64")[0]
    kc = oracle.node_counts(vals, off, stages)
    drops = kc[:, 0] - kc[:, 1]
    for cfg in (dict(chunk=2048), dict(chunk=4096, signal_cap=4, queue_cap=512, q0_stage=128, grid=3)):
        got, st, p = run_gpu(rs, vals, off, stages, "sum_i64_drops", "signal", mode, **cfg)
        np.testing.assert_array_equal(got[0], ref)
        np.testing.assert_array_equal(got[1], drops)
        assert st[2][3] == st[1][3] + st[1][3] // 2       # node 2 consumes Begin, End and the new signal per part
