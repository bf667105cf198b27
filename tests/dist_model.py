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


# ------------------------------------------------------------------ P2P model --
# DI_EXCHANGE_P2P (csrc/p2p.cu) as a protocol model: every rank owns a window in
# POSIX shared memory (header: head/tail/acked/board per peer and the quiesce
# epoch; one inbox ring per peer), ranks run rounds at their own pace (merge what
# has arrived, local passes, board, send rule with records written straight into
# the receiver's ring and the head published after them), and gloo collectives
# appear only in the quiesce-then-reduce confirmation and at the start of a run.

class P2PWindow:
    """Header + per-peer rings over one shared-memory block (the device window)."""

    def __init__(self, shm, world, cap):
        W = world
        self.shm, self.cap = shm, cap
        buf, off = shm.buf, 0

        def view(dtype, count):
            nonlocal off
            a = np.ndarray((count,), dtype=dtype, buffer=buf, offset=off)
            off += a.nbytes
            return a
        self.head = view(np.uint64, W)
        self.tail = view(np.uint64, W)
        self.acked = view(np.float64, W)
        self.board = view(np.float64, W)
        self.quiesce = view(np.uint64, 1)
        self.rows = [view(np.int64, cap) for _ in range(W)]
        self.vals = [view(np.float64, cap) for _ in range(W)]

    @staticmethod
    def nbytes(world, cap):
        return 8 * (4 * world + 1) + 16 * cap * world


class P2PRank(RankModel):
    def __init__(self, rank, world, bounds, cp, ri, b_local, n, key, **kw):
        from multiprocessing import shared_memory
        super().__init__(rank, world, bounds, cp, ri, b_local, n, **kw)
        self.cap = 2 * n + 64
        self.collectives = 0
        size = P2PWindow.nbytes(world, self.cap)
        self._mine = shared_memory.SharedMemory(name=f"{key}_{rank}", create=True, size=size)
        self.win = P2PWindow(self._mine, world, self.cap)
        self.win.head[:] = 0
        self.win.tail[:] = 0
        self.win.acked[:] = 0.0
        self.win.board[:] = np.inf
        self.win.quiesce[:] = 0
        dist.barrier()
        self._peers = [shared_memory.SharedMemory(name=f"{key}_{q}") if q != rank else None for q in range(world)]
        self.peer = [P2PWindow(s, world, self.cap) if s is not None else self.win for s in self._peers]
        self.head_out = np.zeros(world, dtype=np.uint64)
        self.tail_in = np.zeros(world, dtype=np.uint64)
        self.sent = np.zeros(world)
        self.merged = np.zeros(world)
        self.epoch = 0
        self.confirms = 0

    def close(self):
        dist.barrier()
        for s in self._peers:
            if s is not None:
                s.close()
        self._mine.close()
        dist.barrier()
        self._mine.unlink()

    def _coll(self, x):
        self.collectives += 1
        return _allreduce(x)

    def _merge(self):
        for q in range(self.world):
            if q == self.rank:
                continue
            h = int(self.win.head[q])                 # snapshot (acquire)
            t = int(self.tail_in[q])
            if h == t:
                continue
            pos = np.arange(t, h) % self.cap
            rows, vals = self.win.rows[q][pos].copy(), self.win.vals[q][pos].copy()
            np.add.at(self.F, rows, vals)
            self.tail_in[q] = h
            self.merged[q] += float(np.abs(vals).sum())
            self.peer[q].acked[self.rank] = self.merged[q]     # into the sender's header
            self.peer[q].tail[self.rank] = h

    def _send(self, mask):
        for q in range(self.world):
            if q == self.rank or not (mask >> q) & 1:
                continue
            a, b = int(self.bounds[q]), int(self.bounds[q + 1])
            idx = np.nonzero(self.G[a:b])[0]
            if len(idx) == 0:
                continue
            ring = self.peer[q]
            pos = (int(self.head_out[q]) + np.arange(len(idx))) % self.cap
            ring.rows[self.rank][pos] = idx
            ring.vals[self.rank][pos] = self.G[a:b][idx]
            self.sent[q] += float(np.abs(self.G[a:b][idx]).sum())
            self.exchanged += len(idx)
            self.G[a:b][idx] = 0.0
            self.head_out[q] += len(idx)
            ring.head[self.rank] = self.head_out[q]           # published after the records

    def _board(self):
        inflight = sum(self.sent[q] - self.win.acked[q] for q in range(self.world) if q != self.rank)
        v = float(np.abs(self.F).sum()) + float(np.abs(self.G).sum()) + max(inflight, 0.0)
        for q in range(self.world):
            self.peer[q].board[self.rank] = v

    def _confirm(self, my_oop):
        self.confirms += 1
        everyone = sum(1 << q for q in range(self.world) if q != self.rank)
        self._merge()
        self._coll(0.0)                # every publish of the round loops done
        self._merge()
        self._coll(0.0)                # every ring consumed
        self._send(everyone)
        self._coll(0.0)                # flushes published
        self._merge()
        self.collectives += 1
        t = torch.tensor([float(np.abs(self.F).sum()), 1.0 if my_oop else 0.0], dtype=torch.float64)
        dist.all_reduce(t)
        self.epoch += 1
        return float(t[0]), float(t[1]) > 0

    def run_p2p(self, target, m=4, max_rounds=20000, delay=None):
        import time
        nl = self.hi - self.lo
        R = self._coll(float(np.abs(self.F).sum()))
        if R < target:
            return R
        for rnd in range(max_rounds):
            self._merge()
            for _ in range(m):
                cnt = self._pass()
                self.log.append((self.T, cnt))
                if cnt <= self.f * nl:
                    self.T /= self.alpha
            if delay:
                time.sleep(delay(rnd))
            self._board()
            s_k = float(np.abs(self.G).sum())
            r_k = float(np.abs(self.F).sum())
            oop = rnd + 1 >= max_rounds
            if int(self.win.quiesce[0]) > self.epoch or float(self.win.board.sum()) < target or oop:
                if int(self.win.quiesce[0]) <= self.epoch:
                    for q in range(self.world):
                        self.peer[q].quiesce[0] = self.epoch + 1
                R, any_oop = self._confirm(oop)
                if R < target:
                    return R
                if any_oop:
                    raise RuntimeError("no convergence")
                self._board()
                continue
            if s_k > r_k / self.world or (r_k == 0.0 and s_k > 0.0):
                mask = 0
                for q in range(self.world):
                    if q == self.rank:
                        continue
                    used = int(self.head_out[q]) - int(self.win.tail[q])
                    if self.cap - used >= self.bounds[q + 1] - self.bounds[q]:
                        mask |= 1 << q
                self._send(mask)
        raise RuntimeError("no convergence")
