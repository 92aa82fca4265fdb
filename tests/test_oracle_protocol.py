"""Pins for the oracle's credit protocol (one edge), CPU only.

Each test names the passage it follows.  P = PAPER.md, S = SPEC.md lines.
"""
import os
import random

import pytest

import oracle
from oracle import BEGIN, END, Edge, OracleError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_fig2b_credits():
    """Fig. 2b caption P:281-291: one item before the first signal, two before the second."""
    e = Edge()
    for op, arg, exp in _rows("fig2b_credits.txt"):
        if op == "data":
            assert e.emit_data(int(arg)) == int(arg)
        else:
            assert e.emit_signal(BEGIN, 0) == int(exp)
    # receiver side of the same figure: 1 item, then signal, then 2 items, then signal
    assert e.admissible() == 1
    e.consume(1)
    assert e.next_signal() == (BEGIN, 0)
    assert e.admissible() == 2
    e.consume(2)
    assert e.next_signal() == (BEGIN, 0)
    assert e.state()["slen"] == 0


def test_emit_signal_examples_S141():
    """S empty |Q|=1 -> 1; one queued signal + 2 emitted since -> 2; S,Q empty -> 0."""
    e = Edge()
    e.emit_data(1)
    assert e.emit_signal(BEGIN, 0) == 1
    e.emit_data(2)
    assert e.emit_signal(END, 0) == 2
    assert Edge().emit_signal(BEGIN, 0) == 0


def test_admissible_examples_S151():
    """S:151-153 (rules 1, 2a, 2b of P:318-327)."""
    e = Edge()
    e.emit_data(5)
    assert e.admissible() == 5                       # rule (1): no signal queued
    e2 = Edge()
    e2.emit_data(3)
    e2.emit_signal(BEGIN, 0)                         # credit 3 (rule 1 at sender)
    e2.emit_data(2)
    assert e2.state()["head_credit"] == 3
    assert e2.admissible() == 3                      # rule (2b) transfer then (2a)
    st = e2.state()
    assert st["cur"] == 3 and st["head_credit"] == 0
    e3 = Edge()
    e3.emit_signal(BEGIN, 0)                         # credit 0
    assert e3.admissible() == 0
    assert e3.next_signal() == (BEGIN, 0)            # consumable now


def test_consume_examples_S161():
    """counter 3, consume 2 -> 1; S empty consume 4 -> counter 0; overdraw -> violation."""
    e = Edge()
    e.emit_data(3)
    e.emit_signal(END, 7)
    e.emit_data(1)
    assert e.admissible() == 3
    e.consume(2)
    assert e.state()["cur"] == 1
    with pytest.raises(OracleError, match="CreditViolation"):
        e.consume(2)
    f = Edge()
    f.emit_data(4)
    f.consume(4)
    assert f.state()["cur"] == 0


def test_next_signal_examples_S171():
    """head credit 0 -> dequeued; head credit 2 -> nothing, counter 2; S empty -> nothing."""
    e = Edge()
    e.emit_signal(BEGIN, 1)
    assert e.next_signal() == (BEGIN, 1)
    e2 = Edge()
    e2.emit_data(2)
    e2.emit_signal(END, 1)
    assert e2.next_signal() is None
    assert e2.state()["cur"] == 2
    assert Edge().next_signal() is None


def test_partial_enqueue_S89():
    """capacity 4: 3 -> 3; full -> 0; occupancy 2 + 5 -> 2."""
    assert Edge(qcap=4).emit_data(3) == 3
    e = Edge(qcap=4)
    e.emit_data(4)
    assert e.emit_data(1) == 0
    e2 = Edge(qcap=4)
    e2.emit_data(2)
    assert e2.emit_data(5) == 2


def test_signal_queue_full_S139():
    e = Edge(scap=2)
    e.emit_signal(BEGIN, 0)
    e.emit_signal(END, 0)
    with pytest.raises(OracleError, match="SignalQueueFull"):
        e.emit_signal(BEGIN, 1)


def test_enumerate_credits_S355():
    """parents of sizes 2 and 1 -> credits 0, 2, 0, 1."""
    rows = _rows("spec_enumerate_credits.txt")
    sizes = [int(x) for x in rows[0]]
    expect = [int(x) for x in rows[1]]
    e = Edge()
    got = []
    for r, n in enumerate(sizes):
        got.append(e.emit_signal(BEGIN, r))
        e.emit_data(n)
        got.append(e.emit_signal(END, r))
    assert got == expect


@pytest.mark.parametrize("seed", range(200))
def test_lemma1_random_schedules(seed):
    """Lemma 1 (proof P:788-812): a signal is received exactly when all
    items emitted before it have been consumed — i.e. the receiver's event sequence
    equals the merged single FIFO of the sender's emissions.  Also checks
    credit conservation and Claim 1 after every step."""
    rnd = random.Random(seed)
    qcap, scap = rnd.randint(1, 16), rnd.randint(1, 16)
    e = Edge(qcap, scap)
    merged = []          # sender's emission order: ("d", k) or ("s", id)
    got = []             # receiver's consumption order
    nd = ns = 0
    consumed = 0
    for _ in range(rnd.randint(20, 400)):
        act = rnd.random()
        if act < 0.4:
            k = rnd.randint(1, 4)
            n = e.emit_data(k)
            for _ in range(n):
                merged.append(("d", nd))
                nd += 1
        elif act < 0.55:
            if e.state()["slen"] < scap:
                e.emit_signal(BEGIN, ns)
                merged.append(("s", ns))
                ns += 1
        elif act < 0.85:
            a = e.admissible()
            if a:
                k = rnd.randint(1, a)
                e.consume(k)
                for _ in range(k):
                    got.append(("d", consumed))
                    consumed += 1
        else:
            while True:
                s = e.next_signal()
                if s is None:
                    break
                got.append(("s", s[1]))
        assert e.check(), "credit conservation / Claim 1 violated"
    # drain the receiver
    while True:
        a = e.admissible()
        if a:
            e.consume(a)
            for _ in range(a):
                got.append(("d", consumed))
                consumed += 1
            continue
        s = e.next_signal()
        if s is None:
            break
        got.append(("s", s[1]))
        assert e.check()
    assert got == merged
    st = e.state()
    assert st["qlen"] == 0 and st["slen"] == 0 and st["cur"] == 0


def test_back_to_back_signals_zero_credit():
    """Reading A4: back-to-back signals get credit 0 and are deliverable at once."""
    e = Edge()
    e.emit_data(2)
    assert e.emit_signal(END, 0) == 2
    assert e.emit_signal(BEGIN, 1) == 0
    assert e.emit_signal(END, 1) == 0
    e.consume(e.admissible())
    assert [e.next_signal() for _ in range(3)] == [(END, 0), (BEGIN, 1), (END, 1)]


def test_mix64_splitmix_vectors():
    """A19's finalizer is SplitMix64's; published seed-0 outputs (golden file)."""
    for st, out in _rows("splitmix64.txt"):
        assert oracle.mix64(int(st, 16)) == int(out, 16)


def _unmix64(z):
    """Inverse of the splitmix64 finalizer, written independently (xorshift and
    odd-multiplier inverses), so a mistyped constant in the oracle fails."""
    M = (1 << 64) - 1

    def inv_xorshift(y, s):
        x = y
        for _ in range(64 // s + 1):
            x = y ^ (x >> s)
        return x & M

    z = inv_xorshift(z, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M
    z = inv_xorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M
    return inv_xorshift(z, 30)


def test_mix64_bijection():
    rnd = random.Random(3)
    for _ in range(2000):
        x = rnd.getrandbits(64)
        assert _unmix64(oracle.mix64(x)) == x
