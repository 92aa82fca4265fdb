"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/rs.h declares, the Python enums match the header, and
argument / topology errors are reported synchronously before any launch."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rs.h")


@pytest.fixture(scope="module")
def rs():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2006_07478_b200 as rs
    return rs


def _declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(rs_\w+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(rs):
    decl = _declared_functions()
    assert len(decl) >= 10
    out = subprocess.check_output(["nm", "-D", "--defined-only", rs.LIB_PATH]).decode()
    exported = set(re.findall(r" T (rs_\w+)", out))
    missing = [d for d in decl if d not in exported]
    assert not missing, missing
    assert sorted(rs.EXPORTS) == sorted(decl)


def test_enums_match_header(rs):
    src = open(HEADER).read()

    def val(name):
        return int(re.search(rf"\b{name}\s*=\s*(-?\d+)", src).group(1))
    for k, v in rs.OPS.items():
        name = "RS_OP_" + k.upper()
        assert val(name) == v, name
    assert val("RS_NODE_ENUMERATE") == rs.RS_NODE_ENUMERATE
    assert val("RS_NODE_AGGREGATE") == rs.RS_NODE_AGGREGATE
    assert val("RS_STRATEGY_TAGGED") == rs.STRATEGIES["tagged"]
    assert val("RS_STRATEGY_AUTO") == rs.STRATEGIES["auto"]
    assert val("RS_F32") == rs.DTYPES["f32"]
    assert val("RS_ERR_PROTOCOL") == rs.RS_ERR_PROTOCOL


def test_no_oracle_linkage(rs):
    """The product library shares no code with the oracle."""
    out = subprocess.check_output(["nm", "-D", rs.LIB_PATH]).decode()
    assert "or_" not in " ".join(re.findall(r" [TU] (\w+)", out)).replace("for_", "")
    src = open(os.path.join(ROOT, "paper_2006_07478_b200", "csrc", "rs.cu")).read()
    assert "oracle" not in src.lower().replace("cpu oracle", "")


def test_topology_errors(rs):
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline([("hash_lt", 3, 300)], "sum_i64")
    assert e.value.status == rs.RS_ERR_INVALID_ARG
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline([], "count_min_u32", elem="i32")
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline([("hash_lt", 3, 1)] * 5, "sum_i64")
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline([], "sum_i64", queue_cap=100)
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline([], "sum_i64", simd_width=256)
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    # raw node lists: AGGREGATE first / ENUMERATE missing / nested ENUMERATE
    L = rs.lib()
    for kinds in ([4, 2, 1], [2, 4], [1, 1, 4], [1, 4, 4]):
        nodes = (rs.rs_node * len(kinds))()
        for i, k in enumerate(kinds):
            nodes[i] = rs.rs_node(k, 20 if k == 4 else (1 if k == 2 else 0), 3, 100, None)
        h = C.c_void_p()
        st = L.rs_pipeline_create(nodes, len(kinds), 0, None, C.byref(h))
        assert st == rs.RS_ERR_INVALID_TOPOLOGY, kinds
        assert not h.value


def test_run_argument_errors_before_launch(rs):
    p = rs.Pipeline([("hash_lt", 3, 192)], "sum_i64")
    ws = p.workspace_bytes(1000, 100000)
    assert ws > 0
    L = rs.lib()
    agg = rs.rs_aggregates(0x1000, None)
    # negative region count
    assert L.rs_pipeline_run(p.h, 0x1000, 10, 0x1000, -1, None, agg, 0x1000, ws, None) == rs.RS_ERR_INVALID_ARG
    # R = 0 is a no-op
    assert L.rs_pipeline_run(p.h, None, 0, 0x1000, 0, None, agg, None, 0, None) == rs.RS_OK
    # misaligned elements
    assert L.rs_pipeline_run(p.h, 0x1004, 10, 0x1000, 1, None, agg, 0x1000, ws, None) == rs.RS_ERR_INVALID_ARG
    # workspace too small
    assert L.rs_pipeline_run(p.h, 0x1000, 10, 0x1000, 1, None, agg, 0x1000, 16, None) == rs.RS_ERR_WORKSPACE
    # null output
    bad = rs.rs_aggregates(None, None)
    assert L.rs_pipeline_run(p.h, 0x1000, 10, 0x1000, 1, None, bad, 0x1000, ws, None) == rs.RS_ERR_INVALID_ARG
    assert "NULL" in L.rs_last_error().decode()


def test_status_strings(rs):
    assert rs.status_name(rs.RS_OK) == "RS_OK"
    assert rs.status_name(rs.RS_ERR_PROTOCOL) == "RS_ERR_PROTOCOL"


def test_binding_fails_loudly_without_library(rs, tmp_path, monkeypatch):
    monkeypatch.setattr(rs, "_lib", None)
    monkeypatch.setattr(rs, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        rs.lib()


def test_auto_strategy_host_side(rs):
    """RS_STRATEGY_AUTO creates on the host, reports AUTO before
    any run, and sizes its workspace for either strategy (no GPU needed)."""
    import synth
    p = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy="auto")
    assert p.last_strategy() == "auto"
    # (AUTO's two kernels share one chunk table of 8192-child chunks)
    s = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy="signal", chunk=8192)
    t = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy="tagged", chunk=8192)
    for R, N in ((10, 1000), (1 << 20, 1 << 24)):
        assert p.workspace_bytes(R, N) == max(s.workspace_bytes(R, N), t.workspace_bytes(R, N))
    assert s.last_strategy() == "signal" and t.last_strategy() == "tagged"


def test_context_strategy_host_side(rs):
    """RS_STRATEGY_CONTEXT is built for 4-byte elements; other
    combinations, and the removed flag 8, fail at create time (no GPU needed)."""
    import synth
    p = rs.Pipeline(synth.sweep_stages(3), "sum_i64", strategy="context")
    assert p.last_strategy() == "context"
    assert p.workspace_bytes(100, 10000) > 0
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline(synth.text_stages(), "count_xor64", strategy="context")
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
    with pytest.raises(rs.RSError) as e:
        rs.Pipeline(synth.sweep_stages(2), "sum_i64", strategy="context", flags=rs.RS_FLAG_RESERVED8)
    assert e.value.status == rs.RS_ERR_UNSUPPORTED
