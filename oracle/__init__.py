"""CPU oracle for the region-based streaming hot path — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over ``oracle/oracle.c`` (plain C, built with
``-ffp-contract=off``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2006_07478_b200``) never imports it and
shares no code with it.

What it computes (citations: PAPER.md line ranges, section):

* :func:`brute` — the plain per-region fold (§4, Fig. 5):
  for each parent, getItem every element index, apply the stages, fold the
  survivors with begin/run/end.
* :func:`interp` — a sequential interpreter of the pipeline: queues, signal
  queues, credit rules (§3.1), two-phase firing (§3.2),
  fireability, ensembles <= w bounded by credit (§3.3),
  enumeration with Begin/End (§4), tagging.
* :class:`Edge` — one edge's protocol state, for the SPEC worked examples.
* :func:`node_counts` — items reaching each node per region, for the
  occupancy bound sum k / (w sum ceil(k/w)) (§5).

Pins: tests/test_oracle_*.py.  Functions without an independent pin say so in
DESIGN.md ("parity unpinned"); currently none.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# oracle-local op numbering (mirrors the enums at the top of oracle.c)
DTYPES = {"i32": 0, "u32": 1, "u8": 2, "f32": 3}
NP_DTYPES = {"i32": np.int32, "u32": np.uint32, "u8": np.uint8, "f32": np.float32}
FILTER, TRANSFORM = 2, 3
OPS = {"hash_lt": (FILTER, 1), "lt_u32": (FILTER, 2), "class": (FILTER, 3), "parent_lt": (FILTER, 4),
       "scale_f32": (TRANSFORM, 10), "affine_i32": (TRANSFORM, 11)}
AGGS = {"sum_i64": 1, "sum_f32": 2, "count_min_u32": 3, "count_xor64": 4}
STRATEGIES = {"signal": 0, "tagged": 1}
POLICIES = {"full_first": 0, "deepest_first": 1, "random": 2}
BEGIN, END = 1, 2
ERRORS = {0: "OK", -1: "CreditViolation", -2: "SignalQueueFull", -3: "LivelockDetected",
          -4: "UnmatchedEnd", -5: "InvalidArgument", -6: "InvariantViolation", -7: "NoMemory"}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2, no FP contraction) if stale."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB, _SRC])
    return _LIB


class _Stage(C.Structure):
    _fields_ = [("kind", C.c_int32), ("op", C.c_int32), ("p0", C.c_uint64), ("p1", C.c_uint64),
                ("table", C.c_void_p)]


class NodeStats(C.Structure):
    _fields_ = [("data_firings", C.c_uint64), ("full_firings", C.c_uint64),
                ("items", C.c_uint64), ("signal_firings", C.c_uint64)]


class Event(C.Structure):
    _fields_ = [("node", C.c_int32), ("type", C.c_int32), ("a", C.c_int64), ("b", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int, C.c_uint64
        L.or_brute.argtypes = [i32, vp, vp, i64, vp, i32, i32, vp, vp]
        L.or_brute_range.argtypes = [i32, vp, vp, i64, i64, vp, i32, i32, vp, vp]
        L.or_node_counts.argtypes = [i32, vp, vp, i64, vp, i32, vp]
        L.or_emit.argtypes = [i32, vp, vp, i64, vp, i32, vp, vp, i64]
        L.or_emit.restype = i64
        L.or_emit_pair.argtypes = [vp, vp, i64, vp, i32, vp, vp, i64]
        L.or_brute_split.argtypes = [i32, vp, vp, i64, vp, i32, vp, vp, vp]
        L.or_emit_pair.restype = i64
        L.or_interp.argtypes = [i32, vp, vp, i64, vp, i32, i32, i32, i64, i64, i64, i32, u64, i32,
                                vp, vp, vp, vp, i64, vp]
        L.or_mix64.argtypes = [u64]
        L.or_mix64.restype = u64
        L.or_edge_new.argtypes = [i64, i64]
        L.or_edge_new.restype = vp
        L.or_edge_free.argtypes = [vp]
        L.or_edge_emit_data.argtypes = [vp, i64]
        L.or_edge_emit_data.restype = i64
        L.or_edge_emit_signal.argtypes = [vp, i32, i64]
        L.or_edge_emit_signal.restype = i64
        L.or_edge_admissible.argtypes = [vp]
        L.or_edge_admissible.restype = i64
        L.or_edge_consume.argtypes = [vp, i64]
        L.or_edge_next_signal.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        L.or_edge_state.argtypes = [vp, vp]
        L.or_edge_check.argtypes = [vp]
        _lib = L
    return _lib


def _stages(spec):
    """Stage spec: list of tuples
    ("hash_lt", A, T) | ("lt_u32", bound) | ("class", 32-byte bitmap) |
    ("parent_lt", uint32 ctx[R]: keep iff v < ctx[parent]) |
    ("scale_f32", float) | ("affine_i32", a, b)."""
    arr = (_Stage * max(1, len(spec)))()
    keep = []
    for k, s in enumerate(spec):
        kind, op = OPS[s[0]]
        p0 = p1 = 0
        table = None
        if s[0] == "hash_lt":
            p0, p1 = int(s[1]) & 0xFFFFFFFF, int(s[2])
        elif s[0] == "lt_u32":
            p1 = int(s[1])
        elif s[0] == "class":
            buf = C.create_string_buffer(bytes(s[1]), 32)
            keep.append(buf)
            table = C.addressof(buf)
        elif s[0] == "parent_lt":
            ctx = np.ascontiguousarray(s[1], dtype=np.uint32)
            keep.append(ctx)
            table = ctx.ctypes.data
        elif s[0] == "scale_f32":
            p0 = struct.unpack("<I", struct.pack("<f", float(s[1])))[0]
        elif s[0] == "affine_i32":
            p0, p1 = int(s[1]) & 0xFFFFFFFF, int(s[2]) & 0xFFFFFFFF
        arr[k] = _Stage(kind, op, p0, p1, table)
    return arr, keep


def _dtype_name(elems: np.ndarray) -> str:
    for k, v in NP_DTYPES.items():
        if elems.dtype == v:
            return k
    raise OracleError(f"unsupported element dtype {elems.dtype}")


def _out_arrays(agg: str, R: int):
    if agg == "sum_i64":
        return np.zeros(R, np.int64), None
    if agg == "sum_f32":
        return np.zeros(R, np.float64), None
    if agg == "count_min_u32":
        return np.zeros(R, np.uint32), np.zeros(R, np.uint32)
    if agg == "count_xor64":
        return np.zeros(R, np.uint64), np.zeros(R, np.uint64)
    raise OracleError(agg)


def _ptr(a):
    return None if a is None else a.ctypes.data


def _prep(elems, offsets):
    elems = np.ascontiguousarray(elems)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    if offsets.ndim != 1 or offsets.size < 1:
        raise OracleError("offsets must be 1-D with R+1 entries")
    return elems, offsets


def brute(elems, offsets, stages, agg):
    """Plain per-region fold.  Returns (out0, out1-or-None)."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    o0, o1 = _out_arrays(agg, R)
    rc = lib().or_brute(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), R, C.addressof(st),
                        len(stages), AGGS[agg], _ptr(o0), _ptr(o1))
    if rc:
        raise OracleError(ERRORS.get(rc, rc))
    return o0, o1


def brute_split(elems, offsets, stages, split):
    """Fan-out (Fig. 1b): per region, the int64 sums of the
    survivors of `stages` that pass (child A) / fail (child B) the `split`
    FILTER op."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    sp, keep2 = _stages([split])
    a = np.zeros(R, np.int64)
    b = np.zeros(R, np.int64)
    rc = lib().or_brute_split(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), R, C.addressof(st),
                              len(stages), C.addressof(sp), _ptr(a), _ptr(b))
    if rc:
        raise OracleError(ERRORS.get(rc, rc))
    return a, b


def emit(elems, offsets, stages):
    """Element-wise exit: (values u32[n], regions
    u32[n]) of every item surviving the stages, in stream order."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    n = int(offsets[-1] - offsets[0]) if R else 0
    v = np.zeros(max(1, n), np.uint32)
    r = np.zeros(max(1, n), np.uint32)
    m = lib().or_emit(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), R, C.addressof(st), len(stages),
                      _ptr(v), _ptr(r), n)
    if m < 0:
        raise OracleError("bad arguments")
    return v[:m], r[:m]


def emit_pair(elems, offsets, stages):
    """Taxi stage 2: every byte surviving `stages` that starts a
    well-formed "{x,y}" inside its line is emitted as (line, y, x).  Returns
    (yx u32[n, 2], lines u32[n]) in stream order."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    n = int(offsets[-1] - offsets[0]) // 4 + 1 if R else 1
    yx = np.zeros((n, 2), np.uint32)
    r = np.zeros(n, np.uint32)
    m = lib().or_emit_pair(_ptr(elems), _ptr(offsets), R, C.addressof(st), len(stages), _ptr(yx), _ptr(r), n)
    if m < 0 or m > n:
        raise OracleError("bad arguments")
    return yx[:m], r[:m]


def brute_range(elems, offsets, r0, r1, stages, agg, o0, o1):
    """Evaluate regions [r0, r1) into preallocated outputs (for sharded baselines)."""
    st, keep = _stages(stages)
    rc = lib().or_brute_range(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), r0, r1,
                              C.addressof(st), len(stages), AGGS[agg], _ptr(o0), _ptr(o1))
    if rc:
        raise OracleError(ERRORS.get(rc, rc))


def brute_sharded(elems, offsets, stages, agg, threads=None):
    """The plain per-region fold of :func:`brute`, evaluated on `threads`
    contiguous region shards in parallel (regions are independent contexts,
    P:71-79; ctypes releases the GIL), for full-size parity checks."""
    import concurrent.futures as cf
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    o0, o1 = _out_arrays(agg, R)
    threads = threads or len(os.sched_getaffinity(0))
    # shard boundaries balanced by children
    n0, n1 = int(offsets[0]), int(offsets[-1])
    cuts = [0] + [int(np.searchsorted(offsets[:-1], n0 + (n1 - n0) * k // threads, side="left"))
                  for k in range(1, threads)] + [R]
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda k: brute_range(elems, offsets, cuts[k], cuts[k + 1], stages, agg, o0, o1)
                    if cuts[k + 1] > cuts[k] else None, range(threads)))
    return o0, o1


def node_counts(elems, offsets, stages):
    """kc[r, j] = items of region r consumed by node j+1 (j=0: first node after
    enumeration; j=len(stages): the aggregate)."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    kc = np.zeros((R, len(stages) + 1), np.int64)
    rc = lib().or_node_counts(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), R,
                              C.addressof(st), len(stages), _ptr(kc))
    if rc:
        raise OracleError(ERRORS.get(rc, rc))
    return kc


def occupancy_bound(kc: np.ndarray, w: int) -> np.ndarray:
    """Per-node upper bound on lane fraction under the signal strategy:
    sum_r k_r / (w * sum_r ceil(k_r / w))  (ensembles never span a region,
    P:370-381 §3.3, §5).  NaN where a node sees no items."""
    k = kc.astype(np.float64)
    ens = np.ceil(k / w).sum(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        return k.sum(axis=0) / (w * ens)


def interp(elems, offsets, stages, agg, strategy="signal", w=128, qcap=1024, scap=256,
           policy="full_first", seed=1, check=True, trace_cap=0):
    """Sequential pipeline interpreter.

    Returns dict(out=(out0, out1), stats=np.ndarray[n_nodes, 4]
    (data_firings, full_firings, items, signal_firings), trace=np.ndarray or None)."""
    elems, offsets = _prep(elems, offsets)
    R = offsets.size - 1
    st, keep = _stages(stages)
    o0, o1 = _out_arrays(agg, R)
    n_nodes = len(stages) + 2
    stats = (NodeStats * n_nodes)()
    tr = (Event * trace_cap)() if trace_cap else None
    tlen = C.c_int64(0)
    rc = lib().or_interp(DTYPES[_dtype_name(elems)], _ptr(elems), _ptr(offsets), R, C.addressof(st),
                         len(stages), AGGS[agg], STRATEGIES[strategy], w, qcap, scap,
                         POLICIES[policy], seed, int(check), _ptr(o0), _ptr(o1), C.addressof(stats),
                         C.addressof(tr) if tr is not None else None, trace_cap, C.byref(tlen))
    if rc:
        raise OracleError(ERRORS.get(rc, rc))
    S = np.array([[s.data_firings, s.full_firings, s.items, s.signal_firings] for s in stats],
                 dtype=np.int64)
    trace = None
    if tr is not None:
        if tlen.value > trace_cap:
            raise OracleError("trace buffer too small")
        trace = np.array([(e.node, e.type, e.a, e.b) for e in tr[:tlen.value]], dtype=np.int64)
    return {"out": (o0, o1), "stats": S, "trace": trace}


def mix64(z: int) -> int:
    return int(lib().or_mix64(z & 0xFFFFFFFFFFFFFFFF))


class Edge:
    """One edge's data queue + signal queue with the credit protocol."""

    def __init__(self, qcap=1024, scap=256):
        self.h = lib().or_edge_new(qcap, scap)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_edge_free(self.h)
            self.h = None

    def emit_data(self, n=1) -> int:
        return int(lib().or_edge_emit_data(self.h, n))

    def emit_signal(self, kind=BEGIN, r=0) -> int:
        c = int(lib().or_edge_emit_signal(self.h, kind, r))
        if c < 0:
            raise OracleError(ERRORS[c])
        return c

    def admissible(self) -> int:
        return int(lib().or_edge_admissible(self.h))

    def consume(self, n) -> None:
        rc = lib().or_edge_consume(self.h, n)
        if rc:
            raise OracleError(ERRORS[rc])

    def next_signal(self):
        k, r = C.c_int(0), C.c_int64(0)
        if lib().or_edge_next_signal(self.h, C.byref(k), C.byref(r)):
            return (k.value, r.value)
        return None

    def state(self) -> dict:
        st = np.zeros(5, np.int64)
        lib().or_edge_state(self.h, st.ctypes.data)
        return {"qlen": int(st[0]), "slen": int(st[1]), "cur": int(st[2]), "sent": int(st[3]),
                "head_credit": int(st[4])}

    def check(self) -> bool:
        return lib().or_edge_check(self.h) == 0
