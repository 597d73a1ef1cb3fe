"""Multi-GPU plumbing of the column-sharded evaluation.

One process per GPU (torchrun), the CDS replicated on every rank, the Q columns of W
split into contiguous shards. Y[:, c] depends only on W[:, c] (executor.cpp:119-129,
SURVEY F8), so the data path needs no collective. ``torch.distributed`` is used for the
barrier, the max-over-ranks of timings, the replication check and, only when a caller
wants the full Y on every rank, an all-gather of the column shards.
"""
from __future__ import annotations

import hashlib

import numpy as np

from .cds import CDS


def column_shard(q: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [c0, c1) of the q columns for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_shard: bad rank/world")
    return q * rank // world, q * (rank + 1) // world


def cds_fingerprint(cds: CDS) -> str:
    """Content hash of a CDS; equal on every rank iff the replicated CDS is identical."""
    h = hashlib.sha256()
    for name in ("perm", "start", "end", "lchild", "rchild", "sranks", "participating", "near_pairs", "far_pairs",
                 "v_order", "dptr", "bptr", "vptr", "dgen", "bgen", "vgen"):
        h.update(np.ascontiguousarray(getattr(cds, name)).tobytes())
    return h.hexdigest()


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def check_replicated(cds: CDS) -> None:
    """Raise if the CDS differs between ranks (all ranks must build/load the same one)."""
    import torch.distributed as dist

    if not dist.is_initialized():
        return
    mine = cds_fingerprint(cds)
    every = [None] * dist.get_world_size()
    dist.all_gather_object(every, mine)
    if any(f != mine for f in every):
        raise RuntimeError("CDS differs between ranks: the column-sharded evaluation needs a replicated CDS")


def gather_columns(y_local: np.ndarray, q_total: int) -> np.ndarray:
    """All-gather the ranks' column shards (n x q_r, Fortran) into the full n x q Y."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    n = y_local.shape[0]
    widths = [column_shard(q_total, world, r) for r in range(world)]
    qmax = max(c1 - c0 for c0, c1 in widths)
    buf = torch.zeros((qmax, n), dtype=torch.float64)
    c0, c1 = widths[rank]
    buf[: c1 - c0] = torch.from_numpy(np.ascontiguousarray(y_local.T))
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    y = np.empty((n, q_total), dtype=np.float64, order="F")
    for r, (a, b) in enumerate(widths):
        y[:, a:b] = parts[r][: b - a].numpy().T
    return y
