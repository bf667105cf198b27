"""Host-side helpers of the multi-GPU path (one rank per GPU).

Partition (reading R10), CSC sharding, communicator ids.
Only argument marshalling and setup arithmetic on integer arrays live here;
the passes, the outbox compaction, the exchange and the merge run in
libditer.so (csrc/dist.cu).

    bounds = partition_bounds(col_ptr, K, cost="out")      # Cost-Balanced ranges
    bounds = partition_bounds_measured(col_ptr, K, bounds, work)   # re-balanced by a pilot solve's work
    cp, ri, v, b = shard_csc(col_ptr, row_idx, values, b, bounds, rank)
    cid = loopback_comm_id("test")    # K contexts of one process on one GPU (tests)
    cid = shm_comm_id("job42")        # K processes of one host, host-side collectives (tests)
    cid = nccl_comm_id(process_group) # one GPU per rank (rank 0 creates, broadcast)
"""
from __future__ import annotations

import numpy as np

from . import di_get_unique_id, di_partition_cb

LOOP_TAG = b"DILOOP01"
SHM_TAG = b"DISHM001"


def in_degree(row_idx, n: int) -> np.ndarray:
    return np.bincount(np.asarray(row_idx), minlength=n).astype(np.int64)


def partition_bounds(col_ptr, K: int, cost: str = "out", row_idx=None) -> np.ndarray:
    """Contiguous edge-balanced ranges omega_0..omega_K.

    cost="out": balance sum of #out_n (the paper's Cost-Balanced partition);
    cost="inout": balance #out_n + #in_n (still contiguous and balanced by edge
    count; SURVEY.md §8e shows it lifts the work-balance bound on Zipf-over-id
    graphs from 0.50 to 0.71 at K = 8); cost="inhalf" / "in/<m>": #out_n + floor(#in_n / m).
    """
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    n = len(col_ptr) - 1
    if cost == "out":
        prefix = col_ptr
    elif cost in ("inout", "inhalf") or cost.startswith("in/"):
        if row_idx is None:
            raise ValueError(f"cost='{cost}' needs row_idx")
        indeg = in_degree(row_idx, n)
        div = 2 if cost == "inhalf" else int(cost[3:]) if cost.startswith("in/") else 1
        indeg = indeg // div
        prefix = col_ptr + np.concatenate([[0], np.cumsum(indeg)])
    else:
        raise ValueError(cost)
    return di_partition_cb(prefix, K)


def partition_bounds_measured(col_ptr, K: int, prev_bounds, prev_work) -> np.ndarray:
    """Ranges re-balanced by MEASURED work (the paper's dynamic adaptation of the sets
    Omega_k, PAPER.md:178-184 and :523-543 / reading R22, applied between two solves instead of between
    rounds -- DI_EXCHANGE_P2P fixes its outbox slots at create, so it cannot move
    boundaries mid-run).

    prev_work[k] = diffusion work rank k did on prev_bounds in a pilot solve (pushes:
    di_stats edges + remote_pushes).  Each node's cost becomes #out_n x (work per
    stored edge of the rank that held it), i.e. the pilot's work spread over the rank's
    columns in proportion to their out-degree, and the Cost-Balanced split (R10) is
    taken over that cost.  Integer arithmetic on a fixed-point density so that every
    rank derives the same bounds from the same gathered numbers."""
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    prev_bounds = np.asarray(prev_bounds, dtype=np.int64)
    work = np.asarray(prev_work, dtype=np.float64)
    Kp = len(prev_bounds) - 1
    if len(work) != Kp or Kp < 1 or np.any(work < 0) or work.sum() <= 0:
        raise ValueError("prev_work needs one non-negative entry per previous range")
    stored = (col_ptr[prev_bounds[1:]] - col_ptr[prev_bounds[:-1]]).astype(np.float64)
    dens = work / np.maximum(stored, 1.0)
    dens = dens / dens.max()
    q = np.maximum(1, np.rint(dens * 4096.0)).astype(np.int64)     # fixed-point work per stored edge
    prefix = np.empty_like(col_ptr)
    base = 0
    for k in range(Kp):
        lo, hi = int(prev_bounds[k]), int(prev_bounds[k + 1])
        prefix[lo:hi + 1] = base + (col_ptr[lo:hi + 1] - col_ptr[lo]) * q[k]
        base = int(prefix[hi])
    return di_partition_cb(prefix, K)


def remote_fraction(row_idx_local, lo: int, hi: int) -> float:
    """Share of a rank's stored edges whose row lies outside its range [lo, hi)."""
    ri = np.asarray(row_idx_local)
    if ri.size == 0:
        return 0.0
    out = 0
    for a in range(0, ri.size, 1 << 26):                      # chunked: no N-sized temporaries
        c = ri[a:a + (1 << 26)]
        out += int(np.count_nonzero((c < lo) | (c >= hi)))
    return out / ri.size


def pushes_performed(stats: dict, rho: float, remote_push: int) -> float:
    """Pushes a rank executed in a solve, from its di_stats.  di_stats.edges counts every
    edge of a diffused node (the metric's E_p); with remote edges delivered as H
    increments (DI_REMOTE_INCREMENT) the passes push only the local ones and the
    increments are counted in remote_pushes, so the work is edges x (1 - rho) +
    remote_pushes with rho the rank's static remote-edge share (selection does not
    depend on where an edge leads).  Per-diffusion mode pushes every edge in the pass."""
    if remote_push:
        return stats["edges"] * (1.0 - rho) + stats["remote_pushes"]
    return float(stats["edges"])


def shard_csc(col_ptr, row_idx, values, b, bounds, rank: int):
    """Columns [lo, hi) of the global CSC: local col_ptr (from 0), GLOBAL row ids."""
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    e0, e1 = int(col_ptr[lo]), int(col_ptr[hi])
    cp = col_ptr[lo:hi + 1] - e0
    ri = np.asarray(row_idx)[e0:e1]
    v = None if values is None else np.asarray(values)[e0:e1]
    bb = None if b is None else np.asarray(b)[lo:hi]
    return cp, ri, v, bb


def loopback_comm_id(key: str) -> bytes:
    """Communicator id of the in-process loopback fabric (K ranks = K threads, one GPU)."""
    raw = LOOP_TAG + key.encode()[:120]
    return raw + b"\0" * (128 - len(raw))


def shm_comm_id(name: str) -> bytes:
    """Communicator id of the cross-process shared-memory fabric: K processes on one
    host (one GPU or several) with host-side collectives; their DI_EXCHANGE_P2P windows
    are mapped with CUDA IPC (tests: IPC between processes on one GPU, where NCCL
    refuses two ranks per device).  `name` must be unique per group."""
    raw = SHM_TAG + name.encode()[:100]
    return raw + b"\0" * (128 - len(raw))


def nccl_comm_id(group=None) -> bytes:
    """ncclUniqueId made by rank 0 and broadcast over a torch process group."""
    import torch.distributed as dist
    obj = [di_get_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
