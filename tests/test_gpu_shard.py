"""The sharded DDM (shard.py) with the CUDA engine: two ranks over gloo,
each an engine solving its block of subdomains, exchanging the block-boundary
solutions and zero flags after every step (hddm_halo_pack / _unpack) and summing their
assembled fields -- against the single engine solving everything. The box has one
GPU, so both ranks share cuda:0; their kernels never wait on one another (every
exchange is host-staged between steps), so this is a correctness test of the
multi-rank path, not a measurement."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(name):
    from paper_1807_04180_b200.problems import small
    if name == "2x2":
        return small(40, 2, 2, 4.0, 4, 8, source=("gaussian", 0.41, 0.63, 0.05)), 4
    return small(48, 4, 4, 3.0, 2, 6, source=("point", 0.2, 0.7)), 7


def _rank(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from paper_1807_04180_b200.engine import DdmStats
    from paper_1807_04180_b200.shard import ShardedDdm
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob, K = _case(name)
    sh = ShardedDdm(prob, device=0)
    f = prob.source_f()
    res = {}
    for k in (1, 2, K):
        st = DdmStats()
        z = sh.precondition(f, k, st)
        res[k] = (z, st.solves, st.skipped)
    from paper_1807_04180_b200.engine import FgmresOptions
    ps = DdmStats()
    x, fr = sh.fgmres(f, FgmresOptions(1e-8, 40, 30), K, ps)
    sh.close()
    if rank == 0:
        out["res"] = {k: (v[0].tobytes(), v[1], v[2]) for k, v in res.items()}
        out["mine"] = len(sh.plan.mine)
        out["fg"] = (x.tobytes(), fr.iters, fr.converged, list(fr.history), ps.solves, ps.skipped)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["2x2", "4x4"])
def test_sharded_precondition_matches_single_engine(name):
    from paper_1807_04180_b200.engine import DdmEngine, DdmStats
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(2, _free_port(), name, out), nprocs=2, join=True)
    prob, K = _case(name)
    f = prob.source_f()
    from paper_1807_04180_b200.engine import FgmresOptions
    with DdmEngine(prob) as e:
        for k, (zb, solves, skipped) in out["res"].items():
            st = DdmStats()
            z1 = e.precondition(f, k, st)
            z = np.frombuffer(zb, np.complex128)
            assert np.linalg.norm(z - z1) <= 1e-12 * np.linalg.norm(z1), k
            assert (solves, skipped) == (st.solves, st.skipped), k
        # FGMRES(30) over the sharded preconditioner: same iterations, x, history, counts
        ps = DdmStats()
        x1, r1 = e.fgmres(f, FgmresOptions(1e-8, 40, 30), K, ps)
        xb, iters, conv, hist, solves, skipped = out["fg"]
        x = np.frombuffer(xb, np.complex128)
        assert (iters, conv) == (r1.iters, r1.converged)
        assert np.linalg.norm(x - x1) <= 1e-10 * np.linalg.norm(x1)
        np.testing.assert_allclose(hist, r1.history, rtol=1e-6, atol=1e-13)
        assert (solves, skipped) == (ps.solves, ps.skipped)
    assert out["mine"] == prob.n1 * prob.n2 // 2
