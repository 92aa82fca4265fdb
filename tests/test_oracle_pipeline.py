"""Pins for the oracle's per-region fold and pipeline interpreter, CPU only.

The two evaluators in oracle.c are pinned against things outside themselves:
the paper's/SPEC's worked examples (golden files), closed forms, library
identities (numpy cumsum / reduceat), inputs constructed so the filter result
is known by construction, and the lemmas' invariants.  P = PAPER.md lines,
S = SPEC.md lines.
"""
import math
import os
import random

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PASS_ALL = ("hash_lt", 0x9E3779B1, 256)          # T = 256 keeps every value (A13)
AGGS = ["sum_i64", "sum_f32", "count_min_u32", "count_xor64"]
AGG_DTYPE = {"sum_i64": "i32", "sum_f32": "f32", "count_min_u32": "u32", "count_xor64": "u8"}


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _eq(a, b, agg):
    if agg == "sum_f32":
        np.testing.assert_allclose(a[0], b[0], rtol=1e-12, atol=0)
    else:
        np.testing.assert_array_equal(a[0], b[0])
        if a[1] is not None:
            np.testing.assert_array_equal(a[1], b[1])


# ------------------------------------------------------------ worked examples
def test_fixed_sum_S440():
    rows = _rows("fixed_sum_s440.txt")
    vals = np.array([int(x) for x in rows[0]], np.int32)
    L = int(rows[1][0])
    expect = [int(x) for x in rows[2]]
    off = np.arange(0, vals.size + 1, L, dtype=np.int64)
    assert list(oracle.brute(vals, off, [], "sum_i64")[0]) == expect
    for strat in ("signal", "tagged"):
        assert list(oracle.interp(vals, off, [PASS_ALL], "sum_i64", strategy=strat)["out"][0]) == expect


def test_aggregate_push_S385():
    """region {1,2,3} -> 6; empty region -> 0 (begin/end still run, A1)."""
    vals = np.array([1, 2, 3], np.int32)
    off = np.array([0, 3, 3], np.int64)
    assert list(oracle.brute(vals, off, [], "sum_i64")[0]) == [6, 0]
    r = oracle.interp(vals, off, [PASS_ALL], "sum_i64", trace_cap=100)
    assert list(r["out"][0]) == [6, 0]
    # begin/end exactly once per parent per node, including the empty one
    tr = r["trace"]
    for node in (1, 2):
        sig = tr[(tr[:, 0] == node) & (tr[:, 1] == 2)]
        assert [tuple(x) for x in sig[:, 2:]] == [(1, 0), (2, 0), (1, 1), (2, 1)]


def _ensembles(trace, node):
    """Ensembles at `node` as lists of global element indices."""
    out, cur = [], None
    for n, t, a, b in trace:
        if n != node:
            continue
        if t == 0:
            cur = []
            out.append(cur)
        elif t == 1:
            cur.append(int(a))
    return out


def test_w1_hand_trace():
    rows = {r[0]: r[1:] for r in _rows("w1_trace.txt")}
    off = np.array([int(x) for x in rows["offsets"]], np.int64)
    vals = np.array([int(x) for x in rows["elements"]], np.int32)
    sums = [int(x) for x in rows["sums"]]
    for strat, key in (("signal", "signal_F_ensembles"), ("tagged", "tagged_F_ensembles")):
        r = oracle.interp(vals, off, [PASS_ALL], "sum_i64", strategy=strat, w=2, trace_cap=200)
        assert list(r["out"][0]) == sums
        ens = [[int(vals[g]) for g in e] for e in _ensembles(r["trace"], 1)]
        assert ens == [[int(x) for x in s.split(",")] for s in rows[key]]
        st = r["stats"][1]
        assert st[2] / (2 * st[0]) == pytest.approx(5 / 6)      # lane fraction 5/6


# ------------------------------------------------------- library identities
@pytest.mark.parametrize("seed", range(5))
def test_sum_prefix_identity(seed):
    """sum_r = P[off[r+1]] - P[off[r]] with P the int64 cumsum (numpy), exact.
    Pins region assignment + summation independently of the oracle's loops."""
    lens = synth.lengths(500, "var", L=20, seed=seed)
    off = synth.offsets(lens, base=7)
    vals = synth.values(int(off[-1]), "i32", seed=seed + 1)
    P = np.concatenate([[0], np.cumsum(vals.astype(np.int64))])
    expect = P[off[1:]] - P[off[:-1]]
    np.testing.assert_array_equal(oracle.brute(vals, off, [PASS_ALL], "sum_i64")[0], expect)


def _inv32(a):
    return pow(a, -1, 1 << 32)


@pytest.mark.parametrize("T", [0, 1, 100, 192, 255, 256])
def test_hash_lt_by_construction(T):
    """HASH_LT(A, T) keeps v iff top byte of (v*A mod 2^32) < T (reading A13).
    Build v = x * A^-1 mod 2^32 from x with chosen top bytes: the kept set is
    known without evaluating the predicate."""
    rnd = np.random.default_rng(T)
    A = synth.HASH_A[0]
    top = rnd.integers(0, 256, size=4000, dtype=np.uint64)
    x = (top << np.uint64(24)) | rnd.integers(0, 1 << 24, size=4000, dtype=np.uint64)
    v = ((x * np.uint64(_inv32(A))) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    off = np.arange(0, 4001, 40, dtype=np.int64)
    keep = top < T
    kept_vals = np.where(keep, v.astype(np.int64), 0)
    expect = np.add.reduceat(kept_vals, off[:-1])
    np.testing.assert_array_equal(oracle.brute(v, off, [("hash_lt", A, T)], "sum_i64")[0], expect)
    kc = oracle.node_counts(v, off, [("hash_lt", A, T)])
    np.testing.assert_array_equal(kc[:, 1], np.add.reduceat(keep.astype(np.int64), off[:-1]))


def test_hash_lt_stage_order_and_drop():
    """A filter drops at the first failing stage; later stages never see it
    (P:113-118): with T=0 first, every later count is 0."""
    vals = synth.values(1000, "i32", 3)
    off = np.arange(0, 1001, 10, dtype=np.int64)
    kc = oracle.node_counts(vals, off, [("hash_lt", 3, 0), PASS_ALL])
    assert kc[:, 0].sum() == 1000 and kc[:, 1].sum() == 0 and kc[:, 2].sum() == 0


def test_count_min_u32_reduceat():
    lens = synth.lengths(300, "var", L=10, seed=4)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "u32", seed=5)
    b = 1 << 31
    cnt, mn = oracle.brute(vals, off, [("lt_u32", b)], "count_min_u32")
    keep = vals < b
    exp_cnt = np.array([keep[off[r]:off[r + 1]].sum() for r in range(lens.size)], np.uint32)
    masked = np.where(keep, vals, np.uint32(0xFFFFFFFF))
    nz = lens > 0
    exp_min = np.full(lens.size, 0xFFFFFFFF, np.uint32)
    red = np.minimum.reduceat(masked, off[:-1][nz])          # reduceat is only valid on non-empty segments
    exp_min[nz] = red
    np.testing.assert_array_equal(cnt, exp_cnt)
    np.testing.assert_array_equal(mn, exp_min)


def test_count_xor64_single_survivor():
    """COUNT_XOR64 with exactly one surviving byte at local index i gives
    count 1 and xor = mix64(i<<8 | byte) (A19); mix64 itself is pinned by the
    SplitMix64 vectors and its inverse (test_oracle_protocol)."""
    rnd = random.Random(9)
    lens, data, expect = [], [], []
    table = bytearray(32)
    table[ord("{") >> 3] |= 1 << (ord("{") & 7)
    for r in range(200):
        n = rnd.randint(1, 50)
        line = bytearray(rnd.choice(b"abc0123,.}") for _ in range(n))
        if r % 5:
            i = rnd.randrange(n)
            line[i] = ord("{")
            expect.append((1, oracle.mix64((i << 8) | ord("{"))))
        else:
            expect.append((0, 0))
        lens.append(n)
        data.extend(line)
    off = synth.offsets(np.array(lens, np.int64))
    cnt, x = oracle.brute(np.frombuffer(bytes(data), np.uint8), off, [("class", bytes(table))], "count_xor64")
    assert [(int(a), int(b)) for a, b in zip(cnt, x)] == expect


def test_sum_f32_scale_reference():
    """Fig. 5's push(3.14*v) with fp32 RN multiply (A14) summed in double (A15):
    compare against math.fsum of numpy float32 products (exact double sum)."""
    lens = synth.lengths(100, "var", L=30, seed=6)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "f32", seed=7)
    got = oracle.brute(vals, off, [("scale_f32", 3.14)], "sum_f32")[0]
    prod = (np.float32(3.14) * vals).astype(np.float32)
    for r in range(lens.size):
        ref = math.fsum(float(x) for x in prod[off[r]:off[r + 1]])
        assert got[r] == pytest.approx(ref, rel=1e-12, abs=0)


def test_affine_wraps():
    vals = np.array([2**31 - 1, -5, 7], np.int32)
    off = np.array([0, 3], np.int64)
    got = oracle.brute(vals, off, [("affine_i32", 3, 1)], "sum_i64")[0][0]
    exp = sum(int(np.int32(np.uint32((int(v) * 3 + 1) & 0xFFFFFFFF).view(np.int32))) for v in vals.view(np.uint32))
    assert got == exp


# ------------------------------------------------ interpreter vs brute force
def _random_case(rnd, agg):
    R = rnd.randint(0, 60)
    dist = rnd.choice(["var", "fixed", "uniform"])
    L = rnd.randint(0, 40)
    lens = synth.lengths(R, dist, L=L, lo=0, hi=max(1, L), seed=rnd.randrange(1 << 30))
    off = synth.offsets(lens, base=rnd.randint(0, 3))
    vals = synth.values(int(off[-1]) + 4, AGG_DTYPE[agg], seed=rnd.randrange(1 << 30))
    nst = rnd.randint(0, 4)
    stages = []
    for k in range(nst):
        if agg == "count_xor64":
            stages.append(("class", bytes(rnd.getrandbits(8) for _ in range(32))))
        elif agg == "count_min_u32":
            stages.append(("lt_u32", rnd.randint(0, 1 << 32)))
        elif agg == "sum_f32" and rnd.random() < 0.4:
            stages.append(("scale_f32", rnd.choice([3.14, 0.5, -2.0])))
        elif agg == "sum_i64" and rnd.random() < 0.3:
            stages.append(("affine_i32", rnd.getrandbits(32), rnd.getrandbits(32)))
        else:
            stages.append(("hash_lt", rnd.getrandbits(32) | 1, rnd.randint(0, 256)))
    return vals, off, stages


@pytest.mark.parametrize("seed", range(60))
def test_interp_matches_brute(seed):
    """The interpreter (queues, credits, two-phase firing, any policy, any
    capacity >= 1) reaches the plain fold: Lemma 1 + Lemma 2
    (P:364-368).  check=True asserts credit conservation / Claim 1 after
    every protocol step; a livelock would raise (Claim 2)."""
    rnd = random.Random(seed)
    agg = AGGS[seed % 4]
    vals, off, stages = _random_case(rnd, agg)
    ref = oracle.brute(vals, off, stages, agg)
    for strat in ("signal", "tagged"):
        for pol in ("full_first", "deepest_first", "random"):
            r = oracle.interp(vals, off, stages, agg, strategy=strat, w=rnd.choice([1, 2, 4, 32, 128]),
                              qcap=rnd.randint(1, 16), scap=rnd.randint(1, 16), policy=pol,
                              seed=rnd.randrange(1 << 30), check=True)
            _eq(r["out"], ref, agg)
            # enumerated child count = sum of parent sizes (north-star invariant)
            assert r["stats"][0][2] == off[-1] - off[0]
            kc = oracle.node_counts(vals, off, stages)
            for j in range(len(stages) + 1):
                assert r["stats"][j + 1][2] == kc[:, j].sum()


def _per_node_sequences(trace, n_nodes):
    seq = {n: [] for n in range(1, n_nodes)}
    for n, t, a, b in trace:
        if t == 1:
            seq[n].append(("d", int(a)))
        elif t == 2:
            seq[n].append(("s", int(a), int(b)))
    return seq


@pytest.mark.parametrize("seed", range(20))
def test_lemma1_pipeline_sequences(seed):
    """Per node, the consumed sequence is exactly Begin(r), r's surviving items
    in order, End(r), for r = 0..R-1 — the merged-FIFO form of Lemma 1
     and the bracketing (Begin data* End)* of S:390; no ensemble
    holds items of two regions.  The sequences are equal
    under every policy."""
    rnd = random.Random(100 + seed)
    vals, off, stages = _random_case(rnd, "sum_i64")
    R = off.size - 1
    n_nodes = len(stages) + 2
    # expected survivors per node, computed by direct stage application via the oracle's counts
    # plus the brute positions: item g reaches node j+1 iff it survives stages[:j]
    reach = []
    for j in range(len(stages) + 1):
        sub = oracle.node_counts(vals, off, stages[:j]) if j else None
        reach.append(sub)
    seqs = []
    for pol in ("full_first", "deepest_first", "random"):
        r = oracle.interp(vals, off, stages, "sum_i64", w=rnd.choice([2, 8, 128]), qcap=rnd.randint(1, 12),
                          scap=rnd.randint(1, 12), policy=pol, seed=seed, trace_cap=200000)
        tr = r["trace"]
        seq = _per_node_sequences(tr, n_nodes)
        for n in range(1, n_nodes):
            s = seq[n]
            pos = 0
            for reg in range(R):
                assert s[pos] == ("s", 1, reg)
                pos += 1
                items = []
                while s[pos][0] == "d":
                    items.append(s[pos][1])
                    pos += 1
                assert all(off[reg] <= g < off[reg + 1] for g in items)
                assert items == sorted(items)
                assert s[pos] == ("s", 2, reg)
                pos += 1
            assert pos == len(s)
        # no ensemble spans regions (signal strategy)
        for n in range(1, n_nodes):
            for e in _ensembles(tr, n):
                regs = {int(np.searchsorted(off, g, side="right") - 1) for g in e}
                assert len(regs) <= 1
        seqs.append(seq)
    assert seqs[0] == seqs[1] == seqs[2]


# -------------------------------------------------------------- occupancy
def test_occupancy_closed_form():
    """S:304/S:599 and acceptance criterion 4: fixed regions of size R, w=128,
    pass-all stages, full-first -> summing node lane fraction R/(w ceil(R/w))."""
    for R, num, den in (map(int, r) for r in _rows("occupancy_closed_form.txt")):
        nreg = max(8, (1 << 15) // R)
        off = np.arange(0, nreg * R + 1, R, dtype=np.int64)
        vals = synth.values(int(off[-1]), "i32", seed=R)
        for stages in ([], [PASS_ALL], [PASS_ALL, PASS_ALL]):
            r = oracle.interp(vals, off, stages, "sum_i64", w=128, qcap=1024, scap=256)
            st = r["stats"][-1]
            assert st[2] * den == st[0] * 128 * num, (R, stages)
            kc = oracle.node_counts(vals, off, stages)
            assert oracle.occupancy_bound(kc, 128)[-1] == pytest.approx(num / den)


@pytest.mark.parametrize("seed", range(10))
def test_occupancy_never_exceeds_bound(seed):
    """Signal strategy: ensembles never span regions, so every node's lane
    fraction is <= sum k / (w sum ceil(k/w)); full-first attains
    it on the aggregate for pass-all stages."""
    rnd = random.Random(seed)
    vals, off, stages = _random_case(rnd, "sum_i64")
    w = rnd.choice([4, 32, 128])
    r = oracle.interp(vals, off, stages, "sum_i64", w=w, qcap=8 * w, scap=2 * w)
    kc = oracle.node_counts(vals, off, stages)
    bound = oracle.occupancy_bound(kc, w)
    for j in range(len(stages) + 1):
        st = r["stats"][j + 1]
        if st[0]:
            assert st[2] / (w * st[0]) <= bound[j] + 1e-12


def test_tagged_ensembles_stay_full():
    """Tagged strategy: ensembles span regions, so with pass-all
    stages only the stream tail is non-full."""
    lens = synth.lengths(2000, "fixed", L=3)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", 1)
    r = oracle.interp(vals, off, [PASS_ALL], "sum_i64", strategy="tagged", w=128)
    st = r["stats"][1]
    assert st[0] == math.ceil(6000 / 128) and st[1] == 6000 // 128


# ------------------------------------------------------ batching invariance
def test_batching_invariance():
    """Region aggregates are independent of batching (north star; regions are
    independent contexts P:71-79): evaluating region sub-ranges with
    offsets[0] != 0 reproduces the full result."""
    vals, off, stages, agg = synth.tiny()
    full = oracle.brute(vals, off, stages, agg)[0]
    parts = []
    for a, b in ((0, 137), (137, 600), (600, 1000)):
        parts.append(oracle.interp(vals, off[a:b + 1], stages, agg)["out"][0])
    np.testing.assert_array_equal(np.concatenate(parts), full)


def test_determinism():
    vals, off, stages, agg = synth.tiny()
    a = oracle.interp(vals, off, stages, agg, policy="random", seed=5)
    b = oracle.interp(vals, off, stages, agg, policy="random", seed=5)
    np.testing.assert_array_equal(a["out"][0], b["out"][0])
    np.testing.assert_array_equal(a["stats"], b["stats"])


def test_empty_inputs():
    vals = np.zeros(0, np.int32)
    for off in (np.array([0], np.int64), np.array([0, 0, 0], np.int64)):
        for strat in ("signal", "tagged"):
            r = oracle.interp(vals, off, [PASS_ALL], "sum_i64", strategy=strat)
            assert list(r["out"][0]) == [0] * (off.size - 1)
    cnt, mn = oracle.brute(np.zeros(0, np.uint32), np.array([0, 0], np.int64), [], "count_min_u32")
    assert cnt[0] == 0 and mn[0] == 0xFFFFFFFF


def test_bad_offsets_rejected():
    with pytest.raises(oracle.OracleError):
        oracle.brute(np.zeros(4, np.int32), np.array([0, 3, 2], np.int64), [], "sum_i64")


# ------------------------------------------- sharded fold (full-size checks)
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_brute_sharded_prefix_identity(threads):
    """or_brute_range / brute_sharded place every shard's regions at their
    global indices: pinned against the numpy int64 cumsum identity
    sum_r = P[off[r+1]] - P[off[r]] (not against brute itself), with
    offsets[0] != 0, empty regions, and more threads than some shards need."""
    lens = synth.lengths(3000, "zipf", seed=threads, zipf_max=500)
    lens[::7] = 0
    off = synth.offsets(lens, base=11)
    vals = synth.values(int(off[-1]), "i32", seed=threads + 1)
    P = np.concatenate([[0], np.cumsum(vals.astype(np.int64))])
    expect = P[off[1:]] - P[off[:-1]]
    got = oracle.brute_sharded(vals, off, [PASS_ALL], "sum_i64", threads=threads)[0]
    np.testing.assert_array_equal(got, expect)
    # a two-output aggregate: counts by bincount of each element's region
    u = synth.values(int(off[-1]), "u32", seed=threads + 2)
    cnt, mn = oracle.brute_sharded(u, off, [], "count_min_u32", threads=threads)
    reg = np.searchsorted(off, np.arange(off[0], off[-1]), side="right") - 1
    np.testing.assert_array_equal(cnt, np.bincount(reg, minlength=off.size - 1))
    ref_mn = np.full(off.size - 1, 0xFFFFFFFF, np.uint64)
    np.minimum.at(ref_mn, reg, u[off[0]:].astype(np.uint64))
    np.testing.assert_array_equal(mn.astype(np.uint64), ref_mn)


# ------------------------------------------------- parent context (getParent)
def test_parent_lt_by_construction():
    """PARENT_LT keeps item v of parent r iff (uint32)v < ctx[r] (a node reads
    its parent object; Fig. 5 getParent).  ctx[r] is set
    to one more than the k_r-th smallest value of region r, so exactly the k_r
    smallest survive; their sum comes from numpy's sort, not the oracle."""
    g = np.random.default_rng(3)
    lens = synth.lengths(400, "uniform", lo=0, hi=60, seed=4)
    off = synth.offsets(lens, base=5)
    n = int(off[-1])
    vals = g.permutation(np.arange(1, n + 1, dtype=np.int64) * 7).astype(np.uint32).view(np.int32)   # distinct, < 2^31
    ctx = np.zeros(off.size - 1, np.uint32)
    expect = np.zeros(off.size - 1, np.int64)
    u = vals.view(np.uint32)
    for r in range(off.size - 1):
        seg = np.sort(u[off[r]:off[r + 1]].astype(np.int64))
        k = int(g.integers(0, seg.size + 1))
        ctx[r] = (seg[k - 1] + 1) if k > 0 else 0
        expect[r] = seg[:k].sum()
    stages = [("parent_lt", ctx)]
    np.testing.assert_array_equal(oracle.brute(vals, off, stages, "sum_i64")[0], expect)
    for strat in ("signal", "tagged"):
        np.testing.assert_array_equal(oracle.interp(vals, off, stages, "sum_i64", strategy=strat)["out"][0], expect)
    np.testing.assert_array_equal(oracle.brute_sharded(vals, off, stages, "sum_i64", threads=5)[0], expect)
    # node counts: survivors of region r at the aggregate = k_r
    kc = oracle.node_counts(vals, off, stages)
    np.testing.assert_array_equal(kc[:, 1], [np.count_nonzero(u[off[r]:off[r + 1]] < ctx[r]) for r in range(off.size - 1)])


# ------------------------------------------------- element-wise exit (f3)
def test_emit_matches_numpy_masks():
    """The element-wise exit emits (parent, value) of every
    surviving item in stream order: pinned to numpy masks -- region of each
    element by np.repeat over the lengths, survival by a numpy predicate."""
    lens = synth.lengths(700, "zipf", seed=2, zipf_max=300)
    lens[::5] = 0
    off = synth.offsets(lens, base=4)
    u = synth.values(int(off[-1]), "u32", seed=3)
    reg = np.repeat(np.arange(off.size - 1, dtype=np.uint32), lens)
    seg = u[off[0]:]
    v, r = oracle.emit(u, off, [])
    np.testing.assert_array_equal(v, seg)
    np.testing.assert_array_equal(r, reg)
    b = 1 << 31
    v, r = oracle.emit(u, off, [("lt_u32", b)])
    m = seg < b
    np.testing.assert_array_equal(v, seg[m])
    np.testing.assert_array_equal(r, reg[m])
    # a transform rewrites what is emitted: v' = a*v + c mod 2^32
    v, r = oracle.emit(u, off, [("affine_i32", 3, 7)])
    np.testing.assert_array_equal(v, (seg.astype(np.uint64) * 3 + 7).astype(np.uint32))


def test_emit_pair_by_construction():
    """Taxi stage 2: the pairs the oracle parses, verifies and
    swaps are exactly the well-formed ones the corpus generator wrote (its
    malformed variants -- ';', missing fields, 10-digit fields, a pair cut by
    the line end -- are dropped; "{{x,y}" yields its inner pair)."""
    b, off, exp = synth.taxi(300, seed=7)
    yx, r = oracle.emit_pair(b, off, synth.taxi_stages())
    np.testing.assert_array_equal(np.stack([r, yx[:, 0], yx[:, 1]], 1), exp)
    # without stage 1 every byte is tried: the same pairs (only '{' can start one)
    yx2, r2 = oracle.emit_pair(b, off, [])
    np.testing.assert_array_equal(np.stack([r2, yx2[:, 0], yx2[:, 1]], 1), exp)


# ------------------------------------------------------ fan-out (tree, f4)
def test_brute_split_partitions_the_survivors():
    """Tree topology (Fig. 1b): the two leaves' sums partition each
    region's survivors -- pinned to the numpy prefix identity of the masked
    values (child A: split op holds, child B: it does not) and to A + B = the
    linear pipeline's sum."""
    lens = synth.lengths(800, "zipf", seed=6, zipf_max=400)
    lens[::6] = 0
    off = synth.offsets(lens, base=3)
    vals = synth.values(int(off[-1]), "i32", seed=7)
    stages = [("hash_lt", 0x9E3779B1, 192)]
    a, b = oracle.brute_split(vals, off, stages, ("lt_u32", 1 << 31))
    u = vals.view(np.uint32).astype(np.uint64)
    keep = ((u * 0x9E3779B1) % (1 << 32)) >> 24 < 192
    A = np.where(keep & (u < (1 << 31)), vals.astype(np.int64), 0)
    B = np.where(keep & (u >= (1 << 31)), vals.astype(np.int64), 0)
    for arr, got in ((A, a), (B, b)):
        P = np.concatenate([[0], np.cumsum(arr)])
        np.testing.assert_array_equal(got, P[off[1:]] - P[off[:-1]])
    np.testing.assert_array_equal(a + b, oracle.brute(vals, off, stages, "sum_i64")[0])
