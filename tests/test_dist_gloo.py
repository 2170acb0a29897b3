"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU host logic.

Only one GPU exists in this build's environment, so the N > 1 path is covered
here on the CPU: the 1D owner cut every rank computes without communication
(gc_partition_bounds, the rule the intersection kernels apply to their task
list) and the ncclUniqueId broadcast that joins libgc contexts into one NCCL
communicator (init_distributed).  The GPU side of the split is covered by the
loopback partitions in test_parity_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _costs(seed=0, n=100_000):
    rng = np.random.default_rng(seed)
    # power-law-ish per-item costs with zeros, like per-in-edge suffix costs
    c = (rng.pareto(1.2, size=n) * 3).astype(np.int64)
    c[rng.random(n) < 0.2] = 0
    return np.concatenate([[0], np.cumsum(c)]), c


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1708_06866_b200 import gc
    # 1) identical cut points on every rank, no communication needed
    pref, cost = _costs()
    b = gc.partition_bounds(pref, world)
    t = torch.from_numpy(b)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    same = all(torch.equal(g, gathered[0]) for g in gathered)
    # 2) unique-id broadcast into every rank's context (fake context: no GPU here)
    class FakeCtx:
        def comm_init(self, uid, nranks, r):
            self.args = (uid, nranks, r)
    gc_nccl = gc.nccl_unique_id
    gc.nccl_unique_id = lambda: bytes(range(128))      # NCCL needs no network for the test
    try:
        ctx = FakeCtx()
        gc.init_distributed(ctx)
    finally:
        gc.nccl_unique_id = gc_nccl
    uid, nranks, r = ctx.args
    results[rank] = (same, b.tolist(), uid == bytes(range(128)), nranks, r)
    dist.barrier()
    dist.destroy_process_group()


def test_partition_and_uid_broadcast_world2(gc_lib_path):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    pref, cost = _costs()
    total = int(pref[-1])
    for rank in range(world):
        same, b, uid_ok, nranks, r = results[rank]
        assert same and uid_ok and nranks == world and r == rank
    b = results[0][1]
    assert b[0] == 0 and b[-1] == len(cost)
    # balanced: each owner's cost within one item of total / world
    for r in range(world):
        part = int(cost[b[r]:b[r + 1]].sum())
        assert abs(part - total / world) <= cost.max() + 1


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 64])
def test_partition_bounds_rule(gc_lib_path, parts):
    """Single-process check of the owner rule against its definition."""
    from paper_1708_06866_b200 import gc
    pref, cost = _costs(seed=parts)
    b = gc.partition_bounds(pref, parts)
    total = pref[-1]
    owner = np.minimum((pref[:-1] * parts) // total, parts - 1)   # trailing zero-cost items: last owner
    for r in range(parts):
        assert np.all(owner[b[r]:b[r + 1]] == r)
    assert b[0] == 0 and b[-1] == len(cost) and np.all(np.diff(b) >= 0)
    # zero total: everything goes to owner 0
    z = gc.partition_bounds(np.zeros(11, dtype=np.int64), parts)
    assert z[0] == 0 and np.all(z[1:] == 10)
