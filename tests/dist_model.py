"""CPU model of the multi-rank exchange protocol of csrc/dist.cu (test only).

Each rank of a torch.distributed (gloo) group owns Omega_k = [lo, hi) with its
F, H and out-columns; pushes to other ranks' rows go to an
outbox G; an exchange ships the non-zero outbox entries and merges them
(PAPER.md:223-226, 274-277).  SYNC exchanges after every pass and reduces the
pass totals globally (same passes as one process); ASYNC runs `m` local passes
with the local threshold rule, then a round where rank k ships its outbox only
if s_k > r_k / K (eq. send) and the round's all-reduce of
r_k + s_k decides termination (in-flight mass is zero inside a round).

Plain numpy on purpose: it models the protocol, not the kernels.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _allreduce(x: float, op=dist.ReduceOp.SUM) -> float:
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=op)
    return float(t.item())


def _exchange(G, bounds, rank, world, F, lo):
    """Ship non-zero outbox entries to their owners, merge the received ones."""
    payload = {}
    for q in range(world):
        if q == rank:
            continue
        a, b = int(bounds[q]), int(bounds[q + 1])
        idx = np.nonzero(G[a:b])[0]
        payload[q] = (idx.astype(np.int64), G[a:b][idx].copy())
        G[a:b] = 0.0
    gathered = [None] * world
    dist.all_gather_object(gathered, payload)
    recv_mass, sent = 0.0, sum(len(v[0]) for v in payload.values())
    for q in range(world):
        if q == rank:
            continue
        idx, val = gathered[q][rank]
        np.add.at(F, idx, val)
        recv_mass += float(np.abs(val).sum())
    return sent, recv_mass


class RankModel:
    def __init__(self, rank, world, bounds, cp, ri, b_local, n, d=0.85, alpha=1.5, f=0.05):
        self.rank, self.world, self.bounds, self.n, self.d = rank, world, bounds, n, d
        self.lo, self.hi = int(bounds[rank]), int(bounds[rank + 1])
        self.cp, self.ri = np.asarray(cp), np.asarray(ri)
        self.F = np.array(b_local, dtype=np.float64)
        self.H = np.zeros_like(self.F)
        self.G = np.zeros(n)
        self.alpha, self.f = alpha, f
        self.deg = np.diff(self.cp)
        self.T = _allreduce(float(np.abs(self.F).max()) if len(self.F) else 0.0, dist.ReduceOp.MAX) / alpha
        self.log = []           # (T, frontier) per pass (global in SYNC, local in ASYNC)
        self.exchanged = 0

    def _pass(self):
        """Snapshot pass on the owned range: select, take, push (local -> F, remote -> G)."""
        S = np.nonzero(np.abs(self.F) > self.T)[0]
        s = self.F[S].copy()
        self.F[S] = 0.0
        self.H[S] += s
        for i, si in zip(S, s):
            a, b = self.cp[i], self.cp[i + 1]
            if b == a:
                continue
            w = si * (self.d / float(b - a))
            rows = self.ri[a:b]
            loc = (rows >= self.lo) & (rows < self.hi)
            np.add.at(self.F, rows[loc] - self.lo, w)
            np.add.at(self.G, rows[~loc], w)
        return len(S)

    def run_sync(self, target, max_passes=100000):
        for _ in range(max_passes):
            r = _allreduce(float(np.abs(self.F).sum()))
            if r < target:
                return r
            cnt = _allreduce(float(self._pass()))
            self.log.append((self.T, int(cnt)))
            sent, _ = _exchange(self.G, self.bounds, self.rank, self.world, self.F, self.lo)
            self.exchanged += sent
            if cnt <= self.f * self.n:
                self.T /= self.alpha
        raise RuntimeError("no convergence")

    def run_async(self, target, m=4, max_rounds=100000):
        nl = self.hi - self.lo
        for _ in range(max_rounds):
            for _ in range(m):
                cnt = self._pass()
                self.log.append((self.T, cnt))
                if cnt <= self.f * nl:
                    self.T /= self.alpha
            s_k = float(np.abs(self.G).sum())
            r_k = float(np.abs(self.F).sum())
            send = s_k > r_k / self.world or (r_k == 0.0 and s_k > 0.0)
            if send:
                sent, _ = _exchange(self.G, self.bounds, self.rank, self.world, self.F, self.lo)
                self.exchanged += sent
                s_k = 0.0
            else:
                _exchange(np.zeros_like(self.G), self.bounds, self.rank, self.world, self.F, self.lo)
            R = _allreduce(float(np.abs(self.F).sum()) + s_k)
            if R < target:
                sent, _ = _exchange(self.G, self.bounds, self.rank, self.world, self.F, self.lo)
                self.exchanged += sent
                return R
        raise RuntimeError("no convergence")
