"""GPU parity of the short-region (SH) signal kernel (rs.h RS_FLAG_SHORT_ON).

The SH kernel fires the same ensembles and consumes the same signals in the
same order as the general signal kernel (it only batches the per-signal
bookkeeping warp-parallel), so against the oracle its per-region aggregates
are bit-exact and its per-node counters equal the general kernel's.  Cases:
regions shorter / around / longer than w = 128 (mixed, so batches stop at a
long segment and resume), empty regions, unaligned starts, regions split
across chunks, 1-4 stages incl. an all-drop and a keep-all stage, tiny signal
rings (batches bounded by the output signal queue), grid = 1, PARENT_LT (not
batched: falls back to the general pass), and the default device-side choice.
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


def _run(rs, vals, off, stages, flags, parent_ctx=None, **cfg):
    dev_stages = [s if s[0] != "parent_lt" else ("parent_lt",) for s in stages]
    p = rs.Pipeline(dev_stages, "sum_i64", strategy="signal", flags=rs.RS_FLAG_STATS | flags, **cfg)
    e = torch.from_numpy(np.ascontiguousarray(vals)).cuda()
    o = torch.from_numpy(np.ascontiguousarray(off)).cuda()
    R = off.size - 1
    out = p.alloc_outputs(R)
    ws = p.alloc_workspace(R, e.numel())
    kw = {}
    if parent_ctx is not None:
        kw["parent_ctx"] = torch.from_numpy(parent_ctx.view(np.int32)).cuda()
    p.run(e, o, out, ws, **kw)
    torch.cuda.synchronize()
    assert p.check() == 0
    return out[0].cpu().numpy(), np.array(p.stats())


def _compare(rs, vals, off, stages, parent_ctx=None, **cfg):
    ref = oracle.brute(vals, off, stages, "sum_i64")[0]
    got_s, st_s = _run(rs, vals, off, stages, rs.RS_FLAG_SHORT_ON, parent_ctx, **cfg)
    got_g, st_g = _run(rs, vals, off, stages, rs.RS_FLAG_SHORT_OFF, parent_ctx, **cfg)
    bad = np.nonzero(got_s != ref)[0]
    assert bad.size == 0, f"{bad.size} regions differ, first {bad[:5]}: {got_s[bad[:5]]} vs {ref[bad[:5]]}"
    np.testing.assert_array_equal(got_g, ref)
    np.testing.assert_array_equal(st_s, st_g)       # same firings, items and signals per node
    kc = oracle.node_counts(vals, off, stages)
    for j in range(len(stages) + 1):
        assert st_s[j + 1][2] == kc[:, j].sum()


@pytest.mark.parametrize("L", [1, 2, 4, 31, 32, 33, 100, 127, 128, 129, 300])
@pytest.mark.parametrize("dist", ["fixed", "var"])
@pytest.mark.parametrize("nst", [1, 3])
def test_short_lengths(rs, L, dist, nst):
    lens = synth.lengths(20000 if L < 64 else 3000, dist, L=L, seed=L + 7)
    off = synth.offsets(lens, base=L % 5)
    vals = synth.values(int(off[-1]) + 3, "i32", seed=L)
    _compare(rs, vals, off, synth.sweep_stages(nst))


@pytest.mark.parametrize("seed", range(8))
def test_short_mixed(rs, seed):
    """Mostly short regions with empty runs and occasional long ones (batches
    stop at a segment of w or more and resume after the general pass)."""
    g = np.random.default_rng(seed)
    R = 30000
    lens = g.integers(0, 8, R)
    lens[g.random(R) < 0.2] = 0
    longs = g.random(R) < 0.01
    lens[longs] = g.integers(100, 3000, int(longs.sum()))
    off = synth.offsets(lens.astype(np.int64), base=int(g.integers(0, 6)))
    vals = synth.values(int(off[-1]) + 5, "i32", seed=seed)
    nst = 1 + seed % 4
    stages = []
    for k in range(nst):
        t = [0, 64, 192, 256][(seed + k) % 4]
        stages.append(("hash_lt", int(g.integers(0, 2**32)) | 1, t))
    _compare(rs, vals, off, stages, chunk=2048 if seed % 2 else 0)


@pytest.mark.parametrize("scap", [4, 8, 32])
@pytest.mark.parametrize("qcap", [512, 0])
def test_short_small_queues(rs, scap, qcap):
    lens = synth.lengths(12000, "var", L=3, seed=3)
    off = synth.offsets(lens, base=1)
    vals = synth.values(int(off[-1]) + 1, "i32", seed=4)
    _compare(rs, vals, off, synth.sweep_stages(3), signal_cap=scap, queue_cap=qcap, chunk=2048)


def test_short_grid1_and_affine(rs):
    lens = synth.lengths(4000, "var", L=5, seed=11)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", seed=12)
    stages = [("affine_i32", 0x01000193, 7), ("hash_lt", 0x9E3779B1, 128)]
    _compare(rs, vals, off, stages, grid=1)


def test_short_parent_context(rs):
    """PARENT_LT nodes are never batched (their op reads the open region's
    context); the other nodes of the same kernel are."""
    g = np.random.default_rng(2)
    lens = synth.lengths(10000, "var", L=4, seed=21)
    off = synth.offsets(lens, base=2)
    vals = synth.values(int(off[-1]) + 1, "i32", seed=22)
    ctx = g.integers(0, 2**32, off.size - 1, dtype=np.uint64).astype(np.uint32)
    stages = [("hash_lt", 0x9E3779B1, 192), ("parent_lt", ctx), ("hash_lt", 0x85EBCA6B, 192)]
    _compare(rs, vals, off, stages, parent_ctx=ctx)


@pytest.mark.parametrize("L", [1, 5, 40, 130])
def test_short_count_min(rs, L):
    """COUNT_MIN_U32 (the R-MAT config's aggregate): count and min per region
    through the short-region kernel, against the oracle and the general
    kernel's counters."""
    lens = synth.lengths(15000 if L < 64 else 3000, "var", L=L, seed=L + 3)
    off = synth.offsets(lens, base=1)
    vals = synth.values(int(off[-1]) + 2, "u32", seed=L + 4)
    for stages in ([("lt_u32", 1 << 31)], [("lt_u32", 3 << 30), ("lt_u32", 1 << 31)]):
        ref = oracle.brute(vals, off, stages, "count_min_u32")
        got = []
        for fl in (rs.RS_FLAG_SHORT_ON, rs.RS_FLAG_SHORT_OFF):
            p = rs.Pipeline(stages, "count_min_u32", strategy="signal", flags=rs.RS_FLAG_STATS | fl, chunk=2048)
            e = torch.from_numpy(vals.view(np.int32)).cuda()
            o = torch.from_numpy(off).cuda()
            R = off.size - 1
            out = p.alloc_outputs(R)
            ws = p.alloc_workspace(R, e.numel())
            p.run(e, o, out, ws)
            torch.cuda.synchronize()
            assert p.check() == 0
            res = [t.cpu().numpy().view(np.uint32) for t in out]
            for g, r in zip(res, ref):
                np.testing.assert_array_equal(g, r)
            got.append(np.array(p.stats()))
        np.testing.assert_array_equal(got[0], got[1])


def test_short_default_choice(rs):
    """Default flags: both kernels are enqueued for short-looking calls and the
    prepass picks by the call's own children count; either way the results
    are the oracle's."""
    for L in (2, 64, 127, 128, 500):
        lens = synth.lengths(5000, "fixed", L=L)
        off = synth.offsets(lens)
        vals = synth.values(int(off[-1]), "i32", seed=L)
        stages = synth.sweep_stages(3)
        got, _ = _run(rs, vals, off, stages, 0)
        np.testing.assert_array_equal(got, oracle.brute(vals, off, stages, "sum_i64")[0])
