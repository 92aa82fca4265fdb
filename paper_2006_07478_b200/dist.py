"""Multi-GPU plumbing: whole-region partition and the aggregate gather.

Regions are independent contexts (`begin()` resets node
state per region), so a stream partitioned by whole regions needs no
exchange while it is processed; the only collective is assembling the
per-region aggregates on rank 0 (BASELINE north star: "per-region aggregates
are assembled with an NCCL gather").  The collective itself is the C ABI's
(include/rs.h): ``rs_gather_aggregates`` (grouped NCCL send/recv at exact
offsets) or the peer-memory path (``rs_ipc_*``: rank 0's output buffer mapped
into every rank, the kernels store each region's aggregate there over NVLink
as it completes).  torch.distributed only carries the 128-byte NCCL id and
the 64-byte IPC handles between the processes, and the host barriers; nothing
here computes any part of the method.
"""
from __future__ import annotations


def partition(offsets, world: int):
    """Contiguous region ranges balanced by children: rank k owns regions
    [bounds[k], bounds[k+1]) with bounds[k] = first region whose start is
    >= off[0] + k*N/world.  `offsets` is an int64 tensor or
    ndarray of R+1 entries; returns a Python list of world+1 region indices.
    The imbalance is at most one region."""
    import numpy as np
    try:
        import torch
        if isinstance(offsets, torch.Tensor):
            off = offsets.detach()
            R = off.numel() - 1
            n0, n1 = int(off[0].item()), int(off[-1].item())
            targets = torch.tensor([n0 + (n1 - n0) * k // world for k in range(1, world)],
                                   dtype=off.dtype, device=off.device)
            mids = torch.searchsorted(off[:-1].contiguous(), targets, right=False).tolist() if R else []
            return [0] + [int(m) for m in mids] + [R]
    except ImportError:
        pass
    off = np.asarray(offsets)
    R = off.size - 1
    n0, n1 = int(off[0]), int(off[-1])
    mids = [int(np.searchsorted(off[:-1], n0 + (n1 - n0) * k // world, side="left")) for k in range(1, world)]
    return [0] + mids + [R]


def gather_aggregates(local, bounds, dst: int = 0, group=None):
    """Host-plumbing gather for CPU tests (gloo): `local` (this rank's
    aggregates, regions bounds[rank] .. bounds[rank+1]) assembled into one
    dense tensor on `dst` (None elsewhere).  GPU runs use the C ABI instead
    (RankComm.gather / the peer-memory path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [bounds[k + 1] - bounds[k] for k in range(world)]
    assert local.numel() == sizes[rank], "local shard size does not match the partition"
    m = max(sizes) if sizes else 0
    buf = torch.zeros(m, dtype=local.dtype)
    buf[: local.numel()] = local.cpu()
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst, group=group)
        return torch.cat([parts[k][: sizes[k]] for k in range(world)])
    dist.gather(buf, None, dst=dst, group=group)
    return None


def rank_comm(group=None):
    """The C ABI's NCCL communicator over this process group: rank 0 creates
    the unique id, torch.distributed passes it to the others."""
    import torch.distributed as dist

    import paper_2006_07478_b200 as rs
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [rs.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return rs.Comm(box[0], rank, world)


class RootOutputs:
    """Rank 0's dense output arrays (R_total regions) and every rank's device
    address of them: rank 0 uses its own buffers, the other ranks map them with
    CUDA IPC (rs_ipc_export / rs_ipc_open), so ``ptr(k, rank_base)`` is where
    this rank's pipeline stores the aggregates of its first region."""

    def __init__(self, pipeline, r_total, device, group=None):
        import torch.distributed as dist

        import paper_2006_07478_b200 as rs
        self.rank = dist.get_rank(group)
        self.bytes = {"sum_i64": (8, 0), "sum_f32": (4, 0), "count_min_u32": (4, 4),
                      "count_xor64": (8, 8)}[pipeline.agg]
        self.out = pipeline.alloc_outputs(r_total, device) if self.rank == 0 else None
        handles = [None, None]
        if self.rank == 0:
            handles = [rs.ipc_export(t.data_ptr()) if t is not None else None for t in self.out]
        box = [handles]
        dist.broadcast_object_list(box, src=0, group=group)
        self.mapped = []
        self.base = []
        for h, t in zip(box[0], self.out or (None, None)):
            if h is None:
                self.base.append(None)
                continue
            if self.rank == 0:
                self.base.append(t.data_ptr())
            else:
                m = rs.ipc_open(h[0])
                self.mapped.append(m)
                self.base.append(m + h[1])

    def ptrs(self, first_region):
        """(v0, v1) device addresses of region `first_region` in rank 0's arrays."""
        return tuple(None if b is None else b + first_region * nb for b, nb in zip(self.base, self.bytes))

    def close(self):
        import paper_2006_07478_b200 as rs
        for m in self.mapped:
            rs.ipc_close(m)
        self.mapped = []
