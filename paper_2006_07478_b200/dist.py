"""Multi-GPU plumbing: whole-region partition and the aggregate gather.

Regions are independent contexts (`begin()` resets node
state per region), so a stream partitioned by whole regions needs no
exchange while it is processed; the only collective is assembling the
per-region aggregates on rank 0 (BASELINE north star: "per-region aggregates
are assembled with an NCCL gather").  torch.distributed supplies the process
group (NCCL on GPUs, gloo on CPU for the tests); nothing here computes any
part of the method.
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
    """Gather per-region aggregates of every rank into one dense array on `dst`.

    `local`: 1-D tensor of this rank's aggregates (regions bounds[rank] ..
    bounds[rank+1]); `bounds`: the partition (world+1 entries).  Returns the
    assembled tensor on `dst` (None elsewhere).  Shards are padded to the
    largest one so a single collective moves everything."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [bounds[k + 1] - bounds[k] for k in range(world)]
    assert local.numel() == sizes[rank], "local shard size does not match the partition"
    m = max(sizes) if sizes else 0
    # gloo moves host tensors (CPU tests, the 1-GPU functional run); NCCL device ones
    dev = local.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.zeros(m, dtype=local.dtype, device=dev)
    buf[: local.numel()] = local.to(dev)
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst, group=group)
        return torch.cat([parts[k][: sizes[k]] for k in range(world)])
    dist.gather(buf, None, dst=dst, group=group)
    return None
