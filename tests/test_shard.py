"""Sharded DDM (paper_1807_04180_b200/shard.py) on the CPU: the block
ownership and halo lists, and the halo exchange itself over gloo with world_size 2
and 4 (fake engines whose payloads identify subdomain and step). The GPU engine
under the same driver: tests/test_gpu_shard.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1807_04180_b200.shard import ShardPlan, exchange, rank_grid

_NB8 = [(+1, 0), (-1, 0), (0, +1), (0, -1), (+1, +1), (-1, +1), (+1, -1), (-1, -1)]


@pytest.mark.parametrize("n1,n2,world", [(4, 4, 2), (16, 16, 8), (8, 8, 4), (16, 16, 3), (2, 2, 4)])
def test_plan_partitions_and_halos_are_symmetric(n1, n2, world):
    plans = [ShardPlan(n1, n2, world, r) for r in range(world)]
    owned = sorted(t for p in plans for t in p.mine)
    assert owned == list(range(n1 * n2))  # a partition
    pr, pc = rank_grid(world, n1, n2)
    assert pr * pc == world
    for p in plans:
        for r, ts in p.send.items():
            assert plans[r].recv[p.rank] == ts  # what I send is what it expects
        # exactly the subdomains of other ranks in my subdomains' 8-neighbourhood
        need = set()
        for t in p.mine:
            i, j = t % n1, t // n1
            for di, dj in _NB8:
                if 0 <= i + di < n1 and 0 <= j + dj < n2:
                    u = (j + dj) * n1 + i + di
                    if p.owner[u] != p.rank:
                        need.add(u)
        assert need == {u for ts in p.recv.values() for u in ts}


def test_config4_on_8_gpus_layout():
    p = ShardPlan(16, 16, 8, 0)
    assert (p.pr, p.pc) in ((4, 2), (2, 4))
    assert len(p.mine) == 32
    assert sum(len(v) for v in p.send.values()) <= 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n1 = n2 = 6
    nw = 7
    plan = ShardPlan(n1, n2, world, rank)

    def payload(t, s):
        return (np.arange(nw) + 1000 * t + 1j * s).astype(np.complex128)

    got = {}
    for s in range(1, 4):
        def pack(ts):
            assert all(plan.owner[t] == rank for t in ts)
            return np.stack([payload(t, s) for t in ts]), np.array([t % 2 for t in ts], np.int32)

        def unpack(ts, buf, flags):
            for k, t in enumerate(ts):
                got[(t, s)] = bool(np.array_equal(buf[k], payload(t, s)) and flags[k] == t % 2)
        exchange(plan, pack, unpack, s, nw, dist)
    expect = {(t, s) for ts in plan.recv.values() for t in ts for s in range(1, 4)}
    out[rank] = (set(got) == expect) and all(got.values())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_over_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
