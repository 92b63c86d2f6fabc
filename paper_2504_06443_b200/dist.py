"""Row-panel sharding across GPUs (north star "Multi-GPU sharding").

Row panels are independent and write disjoint rows of C, so the only exchange step is one broadcast
of B (NCCL over NVLink on a multi-GPU box). Partition: contiguous panel ranges [p_r, p_{r+1}) such
that each rank's weight (default: nnz, as the north star prescribes) is about total / R; rank r starts
at the first panel p whose exclusive weight prefix W_p >= r * W_total / R, the last rank ends at P,
ranks may be empty when R > P. Contiguous ranges keep B-row locality for the L2.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Shard:
    rank: int
    p0: int          # first panel (inclusive)
    p1: int          # last panel (exclusive)
    row0: int        # first row = p0 * tm
    nrows: int       # rows owned (last panel may be ragged)


def panel_weights(row_ptr: np.ndarray, tm: int = 16, weight: str = "nnz") -> np.ndarray:
    """Weight per panel from row_ptr alone: 'nnz' (north star) or 'rows' (uniform)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    M = rp.shape[0] - 1
    P = (M + tm - 1) // tm
    idx = np.minimum(np.arange(P + 1, dtype=np.int64) * tm, M)
    if weight == "nnz":
        return np.diff(rp[idx])
    if weight == "rows":
        return np.diff(idx)
    raise ValueError(weight)


def shard_plan(row_ptr: np.ndarray, world: int, tm: int = 16, weight="nnz") -> list[Shard]:
    """Contiguous panel ranges with ~equal weight per rank (deterministic). `weight` is 'nnz' (north star),
    'rows', or an explicit per-panel weight array (e.g. HRPB blocks per panel from a GPU build: the cost-model
    option of SURVEY §8(e), which tracks gathered bytes on low-alpha matrices)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    rp = np.asarray(row_ptr, dtype=np.int64)
    M = rp.shape[0] - 1
    if isinstance(weight, str):
        w = panel_weights(rp, tm, weight)
    else:
        w = np.asarray(weight, dtype=np.int64)
        if w.shape[0] != (M + tm - 1) // tm:
            raise ValueError("one weight per panel expected")
    P = w.shape[0]
    W = np.zeros(P + 1, dtype=np.int64)
    W[1:] = np.cumsum(w)
    total = int(W[-1])
    starts = []
    for r in range(world):
        target = (r * total) // world if total > 0 else (r * P) // world
        key = W[:P] if total > 0 else np.arange(P)
        starts.append(int(np.searchsorted(key, target, side="left")) if r > 0 else 0)
    starts.append(P)
    for r in range(1, world + 1):  # monotone
        starts[r] = max(starts[r], starts[r - 1])
    shards = []
    for r in range(world):
        p0, p1 = starts[r], starts[r + 1]
        row0 = min(p0 * tm, M)
        shards.append(Shard(r, p0, p1, row0, min(p1 * tm, M) - row0))
    return shards


def slice_rows(row_ptr, col_idx, vals, shard: Shard):
    """CSR rows of one shard with a rebased row_ptr (views of col_idx / vals, no copy)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    a, b = int(rp[shard.row0]), int(rp[shard.row0 + shard.nrows])
    rp_local = rp[shard.row0:shard.row0 + shard.nrows + 1] - a
    return rp_local, col_idx[a:b], vals[a:b]


def broadcast_B(B, group=None, src: int = 0):
    """The only collective of the path: B from rank `src` to every rank (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    dist.broadcast(B, src=src, group=group)
    return B


def sharded_spmm(row_ptr, col_idx, vals, M: int, K: int, B, rank: int, world: int, tm: int = 16,
                 compute=None, group=None):
    """Row-panel-sharded C = A.B. Each rank builds and multiplies its own slab; returns (shard, C_local).

    `compute(rp_local, ci, v, nrows, K, B)` defaults to the CUDA path (hrpb_build + hrpb_spmm through the
    C ABI); B must already be replicated (see broadcast_B).
    """
    shard = shard_plan(row_ptr, world, tm)[rank]
    rp_l, ci_l, v_l = slice_rows(row_ptr, col_idx, vals, shard)
    if compute is None:
        compute = _cuda_compute
    return shard, compute(rp_l, ci_l, v_l, shard.nrows, K, B)


def _cuda_compute(rp_l, ci_l, v_l, nrows, K, B):
    import torch
    from . import hrpb as hp
    dev = B.device
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)
    A = hp.build(t(rp_l), t(ci_l), t(v_l), nrows, K)
    return hp.spmm(A, B)


# ------------------------------------------------------------------ NEXT-3: B row-sharded, peer gathers
def b_row_shards(K: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Row sharding of B for hrpb_spmm_sharded: rows_per_shard = ceil(K / world) and every
    rank's [row0, row1) (the last ranks may hold fewer rows, or none when world > K). The kernel takes exactly
    ceil(K / rows_per_shard) shards, so ranks past that count hold no rows and are not in the shard table."""
    if world < 1:
        raise ValueError("world must be >= 1")
    rps = max(1, -(-K // world))
    return rps, [(min(r * rps, K), min((r + 1) * rps, K)) for r in range(world)]


def peer_shards(B_local, K: int, group=None):
    """Every rank holds its B row shard (rows b_row_shards(K, world)[1][rank], CUDA, contiguous); returns the shard
    table for hrpb_spmm_sharded: this rank's own tensor and every other rank's shard mapped into this process by
    CUDA IPC (device memory of the peer GPU, read over NVLink by the SpMM's gathers; peer access is enabled by the
    library per device pair). One all_gather of IPC handles is the only exchange (no B replica, no broadcast).
    Needs one process per GPU on one node with every GPU visible (torchrun's default)."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rps, rows = b_row_shards(K, world)
    nsh = -(-K // rps) if K > 0 else 1
    if tuple(B_local.shape[:1]) != (rows[rank][1] - rows[rank][0],):
        raise ValueError(f"rank {rank} must hold {rows[rank][1] - rows[rank][0]} rows of B")
    mine = reduce_tensor(B_local) if B_local.numel() else None
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    shards = []
    for r in range(nsh):
        if r == rank:
            shards.append(B_local)
        else:
            fn, args = handles[r]
            shards.append(fn(*args))
    return rps, shards
