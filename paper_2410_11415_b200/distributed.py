"""Batch sharding across the GPUs of one box.

Batch rows are independent in forward and backward (engine.py:219-220;
pinned by the reference's test_engine.py:72-86), so the path shards with no
data-path collective: rank r of N evaluates rows [r*B/N, (r+1)*B/N) with the
circuit plan replicated, and results are collected with one all_gather
(NCCL over NVLink on GPUs, gloo in the CPU tests). Nothing here depends on
CUDA; the evaluation callable is injected.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank` (first `batch % world` ranks
    take one extra row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local, world: int, group=None):
    """All-gather per-rank row blocks (torch tensors [b_r, C], b_r may differ
    by one) and concatenate them in rank order on every rank."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = local.shape[1:]
    pad = max(sizes)
    buf = torch.zeros((pad, *width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def sharded_eval(evaluate, weights: np.ndarray, world: int, rank: int, group=None):
    """Evaluate this rank's shard with `evaluate(rows) -> (outputs, grads)`
    (numpy in, numpy out) and all-gather both to full [B, ...] arrays."""
    import torch

    lo, hi = shard_bounds(weights.shape[0], world, rank)
    out, grad = evaluate(weights[lo:hi])
    out_all = gather_rows(torch.from_numpy(np.ascontiguousarray(out)), world, group)
    grad_all = gather_rows(torch.from_numpy(np.ascontiguousarray(grad)), world, group)
    return out_all.numpy(), grad_all.numpy()
