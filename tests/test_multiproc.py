"""N>1 path on CPU (gloo, world_size 2): bench.py runs one replica of the DDM
per rank (the path has no data-path collective at N>1 -- "replicas only",
DESIGN.md) with a barrier and a max-over-ranks timing reduction. This drives
those same helpers over two processes, each rank doing its own oracle DDM
replica."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import bench
    import pyoracle
    from paper_1807_04180_b200.problems import small
    w, r, _ = bench.dist_setup()
    prob = small(40, 2, 2, 4.0, 4, 8, source=("point", 0.3 + 0.1 * r, 0.6))
    o = pyoracle.OracleEngine(prob)
    bench.barrier(w)
    z = o.precondition(prob.source_f(), 3)
    t = float(1.0 + r)  # stand-in per-rank time
    tmax = bench.allreduce_max(t, w)
    out[r] = (tmax, float(np.linalg.norm(z)))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_rank, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == 2.0  # max over ranks
    assert out[0][1] > 0 and out[1][1] > 0 and out[0][1] != out[1][1]  # independent replicas
