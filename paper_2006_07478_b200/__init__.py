"""Python binding of the region-streaming C ABI (include/rs.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of ``csrc/rs.cu`` (loaded from ``lib/librs.so``).  PyTorch supplies
device memory and streams; nothing here computes any part of the method and
there is no CPU fallback — if the shared library is missing, importing the
binding raises.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

_HERE = os.path.dirname(os.path.abspath(__file__))
# RS_LIB may point at another build of the same library (A/B measurements)
LIB_PATH = os.environ.get("RS_LIB") or os.path.join(_HERE, "lib", "librs.so")

# rs.h enumerations (kept in sync with include/rs.h by tests/test_abi.py)
RS_OK, RS_ERR_INVALID_ARG, RS_ERR_INVALID_TOPOLOGY, RS_ERR_UNSUPPORTED = 0, -1, -2, -3
RS_ERR_WORKSPACE, RS_ERR_CUDA, RS_ERR_PROTOCOL, RS_ERR_NCCL = -4, -5, -6, -7
RS_NODE_ENUMERATE, RS_NODE_FILTER, RS_NODE_TRANSFORM, RS_NODE_AGGREGATE, RS_NODE_EMIT, RS_NODE_SPLIT = 1, 2, 3, 4, 5, 6
OPS = {"none": 0, "hash_lt": 1, "lt_u32": 2, "class": 3, "parent_lt": 4, "scale_f32": 10, "affine_i32": 11,
       "sum_i64": 20, "sum_f32": 21, "count_min_u32": 22, "count_xor64": 23, "emit_value": 24, "emit_pair": 25, "sum_i64_drops": 27}
DTYPES = {"i32": 0, "u32": 1, "u8": 2, "f32": 3}
STRATEGIES = {"signal": 0, "tagged": 1, "auto": 2, "context": 3, "hybrid": 4}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
RS_FLAG_STATS, RS_FLAG_VALIDATE, RS_FLAG_TIMING, RS_FLAG_RESERVED8, RS_FLAG_PROFILE, RS_FLAG_UNFUSED = 1, 2, 4, 8, 16, 32
RS_FLAG_TRACE = 64
RS_FLAG_SHORT_OFF, RS_FLAG_SHORT_ON = 128, 256
TRACE_ENSEMBLE, TRACE_BEGIN, TRACE_END = 1, 2, 3

EXPORTS = ["rs_config_default", "rs_pipeline_create", "rs_pipeline_workspace_bytes", "rs_pipeline_run",
           "rs_pipeline_run_host", "rs_pipeline_run_emit", "rs_pipeline_stats", "rs_pipeline_profile", "rs_pipeline_check",
           "rs_pipeline_kernel_times",
           "rs_pipeline_launches", "rs_pipeline_last_strategy",
           "rs_pipeline_geometry", "rs_pipeline_set_trace", "rs_pipeline_destroy", "rs_status_string",
           "rs_last_error", "rs_comm_unique_id", "rs_comm_init", "rs_gather_aggregates", "rs_comm_barrier",
           "rs_comm_destroy", "rs_ipc_export", "rs_ipc_open", "rs_ipc_close"]


class RSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{status_name(status)}: {msg}")
        self.status = status


class rs_node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("op", C.c_int32), ("p0", C.c_uint64), ("p1", C.c_uint64),
                ("table", C.c_void_p)]


class rs_config(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("simd_width", C.c_uint32), ("queue_cap", C.c_uint32),
                ("signal_cap", C.c_uint32), ("grid", C.c_int32), ("chunk", C.c_uint32),
                ("flags", C.c_uint32), ("q0_stage", C.c_uint32), ("auto_min_len", C.c_uint32),
                ("tag_from", C.c_uint32)]


class rs_node_stats(C.Structure):
    _fields_ = [("data_firings", C.c_uint64), ("full_firings", C.c_uint64), ("items", C.c_uint64),
                ("signal_firings", C.c_uint64)]


class rs_aggregates(C.Structure):
    _fields_ = [("v0", C.c_void_p), ("v1", C.c_void_p)]


_lib = None


def lib():
    """Load lib/librs.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.rs_config_default.argtypes = [vp]
        L.rs_pipeline_create.argtypes = [vp, i32, i32, vp, C.POINTER(vp)]
        L.rs_pipeline_workspace_bytes.argtypes = [vp, i64, i64, C.POINTER(C.c_size_t)]
        L.rs_pipeline_run.argtypes = [vp, vp, i64, vp, i64, vp, rs_aggregates, vp, C.c_size_t, vp]
        L.rs_pipeline_run_host.argtypes = [vp, vp, i64, vp, i64, vp, rs_aggregates, vp]
        L.rs_pipeline_run_emit.argtypes = [vp, vp, i64, vp, i64, vp, vp, vp, C.c_uint64, vp, vp, C.c_size_t, vp]
        L.rs_pipeline_run_emit.restype = i32
        L.rs_pipeline_stats.argtypes = [vp, vp, i32, vp]
        L.rs_pipeline_check.argtypes = [vp, vp, C.POINTER(C.c_int32)]
        L.rs_pipeline_profile.argtypes = [vp, vp, vp]
        L.rs_pipeline_profile.restype = i32
        L.rs_pipeline_kernel_times.argtypes = [vp, vp, vp]
        L.rs_pipeline_kernel_times.restype = i32
        L.rs_pipeline_launches.argtypes = [vp]
        L.rs_pipeline_launches.restype = i32
        L.rs_pipeline_last_strategy.argtypes = [vp, C.POINTER(C.c_int32)]
        L.rs_pipeline_geometry.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.rs_pipeline_set_trace.argtypes = [vp, vp, C.c_uint64]
        L.rs_pipeline_set_trace.restype = i32
        L.rs_comm_unique_id.argtypes = [vp]
        L.rs_comm_init.argtypes = [vp, i32, i32, C.POINTER(vp)]
        L.rs_gather_aggregates.argtypes = [vp, C.c_int32, rs_aggregates, i64, vp, rs_aggregates, i32, vp]
        L.rs_comm_barrier.argtypes = [vp, vp]
        L.rs_comm_destroy.argtypes = [vp]
        L.rs_comm_destroy.restype = None
        L.rs_ipc_export.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        L.rs_ipc_open.argtypes = [vp, C.POINTER(vp)]
        L.rs_ipc_close.argtypes = [vp]
        for name in ("rs_comm_unique_id", "rs_comm_init", "rs_gather_aggregates", "rs_comm_barrier", "rs_ipc_export",
                     "rs_ipc_open", "rs_ipc_close"):
            getattr(L, name).restype = i32
        L.rs_pipeline_destroy.argtypes = [vp]
        L.rs_pipeline_destroy.restype = None
        L.rs_status_string.argtypes = [i32]
        L.rs_status_string.restype = C.c_char_p
        L.rs_last_error.restype = C.c_char_p
        for name in ("rs_config_default", "rs_pipeline_create", "rs_pipeline_workspace_bytes", "rs_pipeline_run",
                     "rs_pipeline_run_host", "rs_pipeline_run_emit", "rs_pipeline_stats", "rs_pipeline_check", "rs_pipeline_geometry",
                     "rs_pipeline_last_strategy"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def status_name(s: int) -> str:
    return lib().rs_status_string(s).decode()


def _check(s: int):
    if s != RS_OK:
        raise RSError(s, lib().rs_last_error().decode())


def _node(spec) -> tuple:
    """Stage spec tuple -> (kind, op, p0, p1, table bytes or None)."""
    name = spec[0]
    if name == "hash_lt":
        return RS_NODE_FILTER, OPS[name], int(spec[1]) & 0xFFFFFFFF, int(spec[2]), None
    if name == "lt_u32":
        return RS_NODE_FILTER, OPS[name], 0, int(spec[1]), None
    if name == "class":
        return RS_NODE_FILTER, OPS[name], 0, 0, bytes(spec[1])
    if name == "parent_lt":                  # ("parent_lt",): contexts are passed to run(parent_ctx=...)
        return RS_NODE_FILTER, OPS[name], 0, 0, None
    if name == "scale_f32":
        return RS_NODE_TRANSFORM, OPS[name], struct.unpack("<I", struct.pack("<f", float(spec[1])))[0], 0, None
    if name == "affine_i32":
        return RS_NODE_TRANSFORM, OPS[name], int(spec[1]) & 0xFFFFFFFF, int(spec[2]) & 0xFFFFFFFF, None
    raise ValueError(f"unknown stage {name}")


AGG_ELEM = {"split_sum_i64": "i32", "sum_i64_drops": "i32", "sum_i64": "i32", "sum_f32": "f32", "count_min_u32": "u32", "count_xor64": "u8", "emit_value": "i32",
            "emit_pair": "u8"}


class Pipeline:
    """rs_pipeline handle.  ``stages``: list of stage tuples (see _node);
    ``agg``: aggregate op name.  Node list = [ENUMERATE] + stages + [AGGREGATE]."""

    def __init__(self, stages, agg, elem=None, strategy="signal", queue_cap=0, signal_cap=0, grid=0,
                 chunk=0, flags=RS_FLAG_STATS, simd_width=128, q0_stage=0, auto_min_len=0, tag_from=0, split=None):
        """agg "split_sum_i64" builds a tree (RS_NODE_SPLIT): `split` is the
        FILTER-op tuple that routes an item to child A (v0) or child B (v1)."""
        L = lib()
        self.stages = list(stages)
        self.agg = agg
        self.elem = elem or AGG_ELEM[agg]
        tree = agg == "split_sum_i64"
        nodes = (rs_node * (len(self.stages) + (4 if tree else 2)))()
        self._tables = []
        nodes[0] = rs_node(RS_NODE_ENUMERATE, 0, 0, 0, None)
        for i, s in enumerate(self.stages):
            kind, op, p0, p1, table = _node(s)
            tp = None
            if table is not None:
                buf = C.create_string_buffer(table, 32)
                self._tables.append(buf)
                tp = C.addressof(buf)
            nodes[i + 1] = rs_node(kind, op, p0, p1, tp)
        if tree:
            kind, op, p0, p1, _ = _node(split)
            nodes[len(self.stages) + 1] = rs_node(RS_NODE_SPLIT, op, p0, p1, None)
            nodes[-2] = rs_node(RS_NODE_AGGREGATE, OPS["sum_i64"], 0, 0, None)
            nodes[-1] = rs_node(RS_NODE_AGGREGATE, OPS["sum_i64"], 0, 0, None)
        else:
            nodes[-1] = rs_node(RS_NODE_EMIT if agg.startswith("emit") else RS_NODE_AGGREGATE, OPS[agg], 0, 0, None)
        cfg = rs_config()
        L.rs_config_default(C.byref(cfg))
        cfg.strategy = STRATEGIES[strategy]
        cfg.simd_width = simd_width
        if queue_cap:
            cfg.queue_cap = queue_cap
        if signal_cap:
            cfg.signal_cap = signal_cap
        cfg.grid = grid
        cfg.chunk = chunk
        cfg.flags = flags
        cfg.q0_stage = q0_stage
        cfg.auto_min_len = auto_min_len
        cfg.tag_from = tag_from
        h = C.c_void_p()
        _check(L.rs_pipeline_create(nodes, len(nodes), DTYPES[self.elem], C.byref(cfg), C.byref(h)))
        self.h = h
        self.n_nodes = len(nodes)
        self.strategy = strategy

    def close(self):
        if getattr(self, "h", None):
            lib().rs_pipeline_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_strategy(self) -> str:
        """Strategy the last run used ("signal"/"tagged"; "auto" before the first run)."""
        v = C.c_int32()
        _check(lib().rs_pipeline_last_strategy(self.h, C.byref(v)))
        return STRATEGY_NAMES[v.value]

    def workspace_bytes(self, n_regions: int, n_elems: int) -> int:
        b = C.c_size_t()
        _check(lib().rs_pipeline_workspace_bytes(self.h, n_regions, n_elems, C.byref(b)))
        return b.value

    # -- torch-tensor conveniences (torch is plumbing: memory + streams) --
    def alloc_outputs(self, n_regions: int, device="cuda"):
        import torch
        if self.agg == "sum_i64":
            return torch.empty(n_regions, dtype=torch.int64, device=device), None
        if self.agg in ("split_sum_i64", "sum_i64_drops"):
            return (torch.empty(n_regions, dtype=torch.int64, device=device),
                    torch.empty(n_regions, dtype=torch.int64, device=device))
        if self.agg == "sum_f32":
            return torch.empty(n_regions, dtype=torch.float32, device=device), None
        if self.agg == "count_min_u32":
            return (torch.empty(n_regions, dtype=torch.int32, device=device),
                    torch.empty(n_regions, dtype=torch.int32, device=device))
        return (torch.empty(n_regions, dtype=torch.int64, device=device),
                torch.empty(n_regions, dtype=torch.int64, device=device))

    def alloc_workspace(self, n_regions: int, n_elems: int, device="cuda"):
        import torch
        return torch.empty(self.workspace_bytes(n_regions, n_elems) + 256, dtype=torch.uint8, device=device)

    def run(self, elems, offsets, out, workspace, stream=None, parent_ctx=None):
        """elems: 1-D device tensor; offsets: int64 device tensor [R+1];
        out: (v0, v1-or-None) device tensors; workspace: uint8 device tensor;
        parent_ctx: uint32 (int32 view) device tensor [R] for PARENT_LT nodes.
        Asynchronous on `stream` (default: torch's current stream)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        R = offsets.numel() - 1
        ws_ptr = (workspace.data_ptr() + 255) & ~255
        ws_bytes = workspace.numel() - (ws_ptr - workspace.data_ptr())
        agg = rs_aggregates(out[0].data_ptr(), out[1].data_ptr() if out[1] is not None else None)
        _check(lib().rs_pipeline_run(self.h, elems.data_ptr() if elems.numel() else None, elems.numel(),
                                     offsets.data_ptr(), R, parent_ctx.data_ptr() if parent_ctx is not None else None,
                                     agg, ws_ptr, ws_bytes, C.c_void_p(stream.cuda_stream)))

    def run_emit(self, elems, offsets, values, regions, count, workspace, stream=None, parent_ctx=None):
        """EMIT pipelines: every surviving item -> values[k] (int32/uint32
        tensor), regions[k] (int32 tensor), k < count[0] (int64 device tensor)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        R = offsets.numel() - 1
        ws_ptr = (workspace.data_ptr() + 255) & ~255
        ws_bytes = workspace.numel() - (ws_ptr - workspace.data_ptr())
        _check(lib().rs_pipeline_run_emit(self.h, elems.data_ptr() if elems.numel() else None, elems.numel(),
                                          offsets.data_ptr(), R,
                                          parent_ctx.data_ptr() if parent_ctx is not None else None,
                                          values.data_ptr(), regions.data_ptr(),
                                          min(values.numel() // (2 if self.agg == "emit_pair" else 1), regions.numel()),
                                          count.data_ptr(), ws_ptr, ws_bytes, C.c_void_p(stream.cuda_stream)))

    def run_raw(self, elems_ptr, n_elems, offsets_ptr, n_regions, out0_ptr, out1_ptr, ws_ptr, ws_bytes, stream_ptr,
                ctx_ptr=None):
        agg = rs_aggregates(out0_ptr, out1_ptr)
        _check(lib().rs_pipeline_run(self.h, elems_ptr, n_elems, offsets_ptr, n_regions, ctx_ptr, agg, ws_ptr,
                                     ws_bytes, C.c_void_p(stream_ptr)))

    def run_host(self, elems, offsets, out0, out1=None, stream=None, parent_ctx=None):
        """Host (numpy or pinned CPU tensor) in, host out; synchronous."""
        import torch

        def ptr(a):
            if a is None:
                return None
            return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data
        n = elems.numel() if isinstance(elems, torch.Tensor) else elems.size
        R = (offsets.numel() if isinstance(offsets, torch.Tensor) else offsets.size) - 1
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        agg = rs_aggregates(ptr(out0), ptr(out1))
        _check(lib().rs_pipeline_run_host(self.h, ptr(elems) if n else None, n, ptr(offsets), R, ptr(parent_ctx), agg,
                                          C.c_void_p(s)))

    def stats(self, stream=None):
        import numpy as np
        import torch
        st = (rs_node_stats * self.n_nodes)()
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(lib().rs_pipeline_stats(self.h, st, self.n_nodes, C.c_void_p(s)))
        return np.array([[x.data_firings, x.full_firings, x.items, x.signal_firings] for x in st], dtype=np.int64)

    def check(self, stream=None):
        import torch
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        code = C.c_int32(0)
        _check(lib().rs_pipeline_check(self.h, C.c_void_p(s), C.byref(code)))
        return code.value

    def profile(self, stream=None):
        """Per-node cycle counters of the last RS_FLAG_PROFILE run (see rs.h)."""
        import torch
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        buf = (C.c_uint64 * 16)()
        _check(lib().rs_pipeline_profile(self.h, buf, C.c_void_p(s)))
        return list(buf)

    def kernel_times(self, stream=None):
        """(prepass, pipeline, fixup) device ms of the last run (RS_FLAG_TIMING)."""
        import torch
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        ms = (C.c_float * 3)()
        _check(lib().rs_pipeline_kernel_times(self.h, ms, C.c_void_p(s)))
        return [ms[0], ms[1], ms[2]]

    def set_trace(self, buf):
        """RS_FLAG_TRACE: attach a device uint8/int32 tensor as the event buffer (rs.h)."""
        self._trace = buf
        _check(lib().rs_pipeline_set_trace(self.h, buf.data_ptr() if buf is not None else None,
                                           buf.numel() * buf.element_size() if buf is not None else 0))

    def read_trace(self):
        """Events of the last traced run as a uint32 array [n, 8] (see rs.h);
        raises if the buffer overflowed."""
        import numpy as np
        w = self._trace.cpu().numpy().view(np.uint32)
        n = int(w[0])
        cap = (w.size - 8) // 8
        if n > cap:
            raise RuntimeError(f"trace buffer overflow: {n} events, capacity {cap}")
        return w[8:8 + 8 * n].reshape(n, 8).copy()

    def launches(self) -> int:
        return int(lib().rs_pipeline_launches(self.h))

    def geometry(self):
        g, w, c = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().rs_pipeline_geometry(self.h, C.byref(g), C.byref(w), C.byref(c)))
        return {"grid": g.value, "warps_per_cta": w.value, "chunk": c.value}


# ------------------------------------------------------------- multi-GPU (rs.h)
class Comm:
    """rs_comm handle: NCCL communicator of the C ABI (the aggregate gather)."""

    def __init__(self, uid: bytes, rank: int, world: int):
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(lib().rs_comm_init(buf, rank, world, C.byref(h)))
        self.h, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().rs_comm_unique_id(buf))
        return buf.raw

    def gather(self, agg, local, bounds, root_out, root=0, stream=None):
        """rs_gather_aggregates: local = (v0, v1-or-None) device tensors of this
        rank's regions; bounds = world+1 region bases; root_out read on `root`."""
        import torch
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        base = (C.c_int64 * len(bounds))(*[int(b) for b in bounds])
        loc = rs_aggregates(local[0].data_ptr(), local[1].data_ptr() if local[1] is not None else None)
        ro = rs_aggregates(root_out[0].data_ptr() if root_out is not None else None,
                           root_out[1].data_ptr() if root_out is not None and root_out[1] is not None else None)
        n = int(bounds[self.rank + 1] - bounds[self.rank])
        _check(lib().rs_gather_aggregates(self.h, OPS[agg], loc, n, base, ro, root, C.c_void_p(s)))

    def barrier(self, stream=None):
        import torch
        s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(lib().rs_comm_barrier(self.h, C.c_void_p(s)))

    def close(self):
        if getattr(self, "h", None):
            lib().rs_comm_destroy(self.h)
            self.h = None


def ipc_export(ptr: int):
    """(64-byte handle of the allocation holding ptr, ptr's offset in it)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    _check(lib().rs_ipc_export(C.c_void_p(ptr), buf, C.byref(off)))
    return buf.raw, int(off.value)


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    _check(lib().rs_ipc_open(C.create_string_buffer(bytes(handle), 64), C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int):
    _check(lib().rs_ipc_close(C.c_void_p(ptr)))
