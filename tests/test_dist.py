"""Multi-GPU host logic on CPU (gloo, world_size 2): whole-region partition and
the aggregate gather.  Per-shard aggregates come from the oracle (the CUDA
kernels need a GPU); what is tested is that sharding by whole regions and
gathering reproduces the unsharded result (regions are independent contexts,
P:71-79) and that the partition is balanced by children."""
import os
import socket

import numpy as np
import pytest

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_balanced_and_covering():
    from paper_2006_07478_b200.dist import partition
    lens = synth.lengths(20000, "zipf", seed=3, zipf_max=4096)
    off = synth.offsets(lens, base=11)
    for world in (1, 2, 3, 8):
        b = partition(off, world)
        assert b[0] == 0 and b[-1] == off.size - 1 and all(x <= y for x, y in zip(b, b[1:]))
        n = off[-1] - off[0]
        for k in range(world):
            kids = off[b[k + 1]] - off[b[k]]
            assert abs(kids - n / world) <= 4096 + 1     # imbalance <= the largest region
    # empty regions and a single region
    assert partition(np.array([5, 5, 5], np.int64), 2)[-1] == 2
    assert partition(np.array([0, 100], np.int64), 4) == [0, 1, 1, 1, 1]


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2006_07478_b200.dist import gather_aggregates, partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lens = synth.lengths(5000, "zipf", seed=7, zipf_max=512)
    off = synth.offsets(lens)
    vals = synth.values(int(off[-1]), "i32", seed=8)
    stages = synth.sweep_stages(3)
    b = partition(off, world)
    mine = oracle.brute(vals, off[b[rank]:b[rank + 1] + 1], stages, "sum_i64")[0]
    full = gather_aggregates(torch.from_numpy(mine), b, dst=0)
    if rank == 0:
        ref = oracle.brute(vals, off, stages, "sum_i64")[0]
        np.save(result_path, np.array([int(np.array_equal(full.numpy(), ref)), full.numel()]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_gather(tmp_path):
    import torch.multiprocessing as mp
    path = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    ok, n = np.load(path)
    assert ok == 1 and n == 5000
