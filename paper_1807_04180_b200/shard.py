"""Sharded DDM preconditioner over torch.distributed.

One engine per rank (one GPU per rank in production) solves a rectangular block of the
n1 x n2 subdomain grid (``ShardPlan``). A DDM step is local except for its inputs from
neighbouring subdomains: the transfers of step s read the step s-1 solutions of the
edge neighbours and the step s-2 solutions of the corner neighbours (ddm.cpp:174-214,
transfer.cpp:64-88), and the zero flags of both. So after every step each rank sends
the solutions and flags of its block-boundary subdomains to the ranks whose
subdomains border them, and receives theirs (``hddm_halo_pack`` / ``_unpack``); the
blend-accumulate is local into a full-size field that the ranks sum at the end
(``all_reduce``), which is precondition(r, K) (ddm.cpp:280-287) distributed.

The halo payloads are staged through host memory here, so the same code runs over
gloo (the CPU tests and the one-GPU box, where two ranks share a device) and NCCL.
Per step a rank sends at most 8 neighbour blocks' worth of boundary subdomains: at
config 4 on 8 GPUs (4 x 2 blocks of 4 x 8 subdomains) ~20 subdomain vectors of 0.6 MB.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

_NB8 = [(+1, 0), (-1, 0), (0, +1), (0, -1), (+1, +1), (-1, +1), (+1, -1), (-1, -1)]


def rank_grid(world: int, n1: int, n2: int) -> Tuple[int, int]:
    """pr x pc = world ranks over the n1 x n2 subdomains, as square as the grid allows."""
    best = None
    for pr in range(1, world + 1):
        if world % pr:
            continue
        pc = world // pr
        if pr > n1 or pc > n2:
            continue
        score = abs(math.log((n1 / pr) / (n2 / pc)))
        if best is None or score < best[0]:
            best = (score, pr, pc)
    if best is None:
        raise ValueError(f"{world} ranks cannot split a {n1} x {n2} subdomain grid")
    return best[1], best[2]


@dataclass
class ShardPlan:
    """Block ownership of the subdomains and the per-step halo lists of one rank."""
    n1: int
    n2: int
    world: int
    rank: int
    pr: int = 0
    pc: int = 0
    owner: List[int] = field(default_factory=list)
    mine: List[int] = field(default_factory=list)
    send: Dict[int, List[int]] = field(default_factory=dict)  # rank -> my subdomains it reads
    recv: Dict[int, List[int]] = field(default_factory=dict)  # rank -> its subdomains I read

    def __post_init__(self):
        self.pr, self.pc = rank_grid(self.world, self.n1, self.n2)
        n1, n2 = self.n1, self.n2
        self.owner = [((t // n1) * self.pc // n2) * self.pr + (t % n1) * self.pr // n1
                      for t in range(n1 * n2)]
        self.mine = [t for t in range(n1 * n2) if self.owner[t] == self.rank]
        send: Dict[int, set] = {}
        recv: Dict[int, set] = {}
        for t in self.mine:
            i, j = t % n1, t // n1
            for di, dj in _NB8:
                si, sj = i + di, j + dj
                if not (0 <= si < n1 and 0 <= sj < n2):
                    continue
                u = sj * n1 + si
                o = self.owner[u]
                if o != self.rank:
                    send.setdefault(o, set()).add(t)  # o's subdomain u reads my t
                    recv.setdefault(o, set()).add(u)  # my t reads o's u
        self.send = {r: sorted(v) for r, v in sorted(send.items())}
        self.recv = {r: sorted(v) for r, v in sorted(recv.items())}

    def owned_mask(self) -> np.ndarray:
        return np.array([1 if o == self.rank else 0 for o in self.owner], np.int32)


def exchange(plan: ShardPlan, pack, unpack, tag: int, nw: int, dist=None):
    """One halo exchange: pack(ts) -> (buf [n, nw] complex, flags [n]) for each
    neighbour rank, non-blocking point-to-point sends and receives in both directions,
    then unpack(ts, buf, flags) of everything received."""
    import torch
    if dist is None:
        import torch.distributed as dist
    reqs, keep = [], []
    for r, ts in plan.send.items():
        buf, flags = pack(ts)
        b = torch.from_numpy(np.ascontiguousarray(buf, np.complex128).view(np.float64))
        f = torch.from_numpy(np.ascontiguousarray(flags, np.int32))
        keep.append((b, f))
        reqs.append(dist.isend(b, dst=r, tag=2 * tag))
        reqs.append(dist.isend(f, dst=r, tag=2 * tag + 1))
    recvs = {}
    for r, ts in plan.recv.items():
        b = torch.empty((len(ts), 2 * nw), dtype=torch.float64)
        f = torch.empty(len(ts), dtype=torch.int32)
        recvs[r] = (b, f)
        reqs.append(dist.irecv(b, src=r, tag=2 * tag))
        reqs.append(dist.irecv(f, src=r, tag=2 * tag + 1))
    for q in reqs:
        q.wait()
    for r, ts in plan.recv.items():
        b, f = recvs[r]
        unpack(ts, b.numpy().view(np.complex128), f.numpy())


class ShardedDdm:
    """precondition(r, K) of a 2-D problem sharded over the ranks of the default
    torch.distributed group (DdmEngine surface; one engine per rank)."""

    def __init__(self, prob, device: int = 0, engine=None):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.prob = prob
        self.plan = ShardPlan(prob.n1, prob.n2, self.world, self.rank)
        if engine is None:
            from .engine import DdmEngine
            engine = DdmEngine(prob, device=device)
        self.eng = engine
        self.eng.set_owned(self.plan.owned_mask())
        nx, ny = self.eng.window_dims()
        self.nw = nx * ny
        self._tag = 0

    def close(self):
        self.eng.close()

    def precondition(self, r, ksteps: int, stats=None) -> np.ndarray:
        """z = M(r): K sweeps with a halo exchange after each, then the sum of the
        ranks' assembled fields. stats (DdmStats) accumulates solves / skips over all
        ranks."""
        import torch
        from .engine import DdmStats
        e = self.eng
        e.precondition_begin(r)
        for s in range(1, ksteps + 1):
            e.step(s)
            self._tag += 1
            exchange(self.plan, lambda ts: e.halo_pack(s, ts),
                     lambda ts, b, f: e.halo_unpack(s, ts, b, f), self._tag, self.nw, self.dist)
        st = DdmStats()
        z = e.precondition_end(st)
        zt = torch.from_numpy(z.view(np.float64).copy())
        self.dist.all_reduce(zt)
        cnt = torch.tensor([st.solves, st.skipped], dtype=torch.int64)
        self.dist.all_reduce(cnt)
        if stats is not None:
            stats.solves += int(cnt[0])
            stats.skipped += int(cnt[1])
        return zt.numpy().view(np.complex128)

    def fgmres(self, b, opt, ksteps: int, pstats=None):
        """fgmres(A = apply_global, M = the sharded precondition(K)) as cli.cpp:210-228
        wires it: every rank runs the engine's device FGMRES on identical vectors; its
        host-driven cycles call back after every step (halo exchange) and after every
        preconditioner application (all_reduce of the assembled fields). Returns
        (x, FgmresResult) on every rank; pstats accumulates solves / skips of all ranks."""
        import torch
        from .engine import DdmStats
        e = self.eng

        def hook(stage, s):
            if stage == 1:
                self._tag += 1
                exchange(self.plan, lambda ts: e.halo_pack(s, ts),
                         lambda ts, bb, f: e.halo_unpack(s, ts, bb, f), self._tag, self.nw, self.dist)
            else:
                a = torch.from_numpy(e.assembled().view(np.float64).copy())
                self.dist.all_reduce(a)
                e.assembled(a.numpy().view(np.complex128))

        st = DdmStats()
        e.set_step_hook(hook)
        try:
            x, res = e.fgmres(b, opt, ksteps, st)
        finally:
            e.set_step_hook(None)
        cnt = torch.tensor([st.solves, st.skipped], dtype=torch.int64)
        self.dist.all_reduce(cnt)
        if pstats is not None:
            pstats.solves += int(cnt[0])
            pstats.skipped += int(cnt[1])
        return x, res

