"""Host-side helpers of the multi-GPU path (one rank per GPU).

Partition (reading R10), CSC sharding, communicator ids.
Only argument marshalling and setup arithmetic on integer arrays live here;
the passes, the outbox compaction, the exchange and the merge run in
libditer.so (csrc/dist.cu).

    bounds = partition_bounds(col_ptr, K, cost="out")      # Cost-Balanced ranges
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
