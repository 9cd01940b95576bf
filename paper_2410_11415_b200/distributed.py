"""Batch sharding across the GPUs of one box.

Batch rows are independent in forward and backward (engine.py:219-220;
pinned by the reference's test_engine.py:72-86), so the path shards with no
data-path collective: rank r of N evaluates rows [r*B/N, (r+1)*B/N) with the
circuit plan replicated on every GPU, and the per-rank outputs [b_r, R] and
input gradients [b_r, K] are collected with one all-gather each (NCCL over
NVLink between GPUs; gloo in the CPU tests).

``ShardedPass`` is the device path: one CUDA-graph-captured forward+backward
of this rank's rows, followed by the two all-gathers of device tensors into
[B, R] / [B, K] device buffers, all stream-ordered (bench.py's multi-GPU arm
and tests/test_distributed_gpu.py). ``gather_rows`` / ``sharded_eval`` are
the host-level helpers (numpy in / out) used by the CPU tests.
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


def _comm_device(group=None):
    """Device the collective runs on: the current CUDA device for NCCL (it
    rejects host tensors), the host for gloo."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_rows(local, world: int, group=None, sizes=None, out=None):
    """All-gather per-rank row blocks (tensors [b_r, C...]) in rank order.

    `sizes` (the per-rank row counts, e.g. from shard_bounds) avoids a count
    exchange; without it the counts are all-gathered first. The exchange
    runs on the backend's device (CUDA for NCCL, host for gloo) and the
    result comes back on `local`'s device, in `out` when given ([sum b_r,
    C...]). Blocks may differ in length: they are padded to the longest."""
    import torch
    import torch.distributed as dist

    if world == 1:
        if out is not None:
            out.copy_(local)
            return out
        return local
    dev = _comm_device(group)
    if sizes is None:
        n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
        parts = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(parts, n, group=group)
        sizes = [int(s.item()) for s in parts]
    sizes = [int(s) for s in sizes]
    if len(sizes) != world or sizes[dist.get_rank(group)] != local.shape[0]:
        raise ValueError(f"row counts {sizes} do not match this rank's {local.shape[0]} rows")
    width = tuple(local.shape[1:])
    pad = max(sizes)
    send = local if local.device == dev else local.to(dev)
    if send.shape[0] != pad or not send.is_contiguous():
        buf = torch.zeros((pad, *width), dtype=local.dtype, device=dev)
        buf[: local.shape[0]] = send
        send = buf
    total = sum(sizes)
    even = all(s == pad for s in sizes)
    if out is not None and tuple(out.shape) != (total, *width):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {(total, *width)}")
    if dev.type == "cuda":
        # one flat receive buffer (NCCL all_gather_into_tensor)
        if even and out is not None and out.device == dev and out.is_contiguous():
            recv = out
        else:
            recv = torch.empty((world * pad, *width), dtype=local.dtype, device=dev)
        dist.all_gather_into_tensor(recv, send, group=group)
        parts = [recv[r * pad:r * pad + s] for r, s in enumerate(sizes)]
    else:
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        parts = [p[:s] for p, s in zip(parts, sizes)]
    if out is None:
        res = parts[0] if len(parts) == 1 else torch.cat(parts, dim=0)
        return res.to(local.device) if res.device != local.device else res
    if not (even and parts[0].data_ptr() == out.data_ptr()):
        o = 0
        for p, s in zip(parts, sizes):
            out[o:o + s].copy_(p)
            o += s
    return out


def sharded_eval(evaluate, weights: np.ndarray, world: int, rank: int, group=None):
    """Evaluate this rank's shard with `evaluate(rows) -> (outputs, grads)`
    (numpy in, numpy out) and all-gather both to full [B, ...] arrays."""
    import torch

    lo, hi = shard_bounds(weights.shape[0], world, rank)
    sizes = [b - a for a, b in (shard_bounds(weights.shape[0], world, r) for r in range(world))]
    out, grad = evaluate(weights[lo:hi])
    out_all = gather_rows(torch.from_numpy(np.ascontiguousarray(out)), world, group, sizes)
    grad_all = gather_rows(torch.from_numpy(np.ascontiguousarray(grad)), world, group, sizes)
    return out_all.cpu().numpy(), grad_all.cpu().numpy()


class ShardedPass:
    """This rank's share of a global batch on its GPU: a captured forward +
    backward of rows shard_bounds(global_batch, world, rank) (engine
    DevicePlan.capture), then the all-gathers of outputs and input gradients
    into ``outputs`` [B, R] and ``grads`` [B, K] (device tensors, every rank).

        sp = ShardedPass(tc, 1024, np.float32, KLAY_LOG, world, rank)
        sp.weights.copy_(w_all[sp.lo:sp.hi])   # this rank's rows, on device
        sp.step()                              # replay + 2 all-gathers
    """

    def __init__(self, tc, global_batch: int, dtype, semiring: int, world: int, rank: int,
                 epsilon: float = 0.0, group=None, device=None, gather: bool = True):
        import torch

        from .engine import device_plan

        if global_batch < world:
            raise ValueError(f"global batch {global_batch} < {world} ranks")
        self.world, self.rank, self.group, self.gather = world, rank, group, gather
        self.global_batch = global_batch
        self.lo, self.hi = shard_bounds(global_batch, world, rank)
        self.sizes = [b - a for a, b in (shard_bounds(global_batch, world, r) for r in range(world))]
        self.plan = device_plan(tc, device)
        self.cap = self.plan.capture(self.hi - self.lo, dtype, semiring, epsilon=epsilon,
                                     backward=True)
        self.weights = self.cap.weights
        dev = self.plan.device
        tdt = self.cap.outputs.dtype
        self.outputs = torch.empty((global_batch, self.plan.num_roots), dtype=tdt, device=dev)
        self.grads = torch.empty((global_batch, self.plan.num_inputs), dtype=tdt, device=dev)

    @property
    def local_batch(self) -> int:
        return self.hi - self.lo

    def step(self):
        """One forward+backward of this rank's rows, then the gathers."""
        self.cap.replay()
        if self.gather:
            gather_rows(self.cap.outputs, self.world, self.group, self.sizes, out=self.outputs)
            gather_rows(self.cap.grads, self.world, self.group, self.sizes, out=self.grads)
        return self.outputs, self.grads

    @property
    def gathered_bytes(self) -> int:
        """Bytes this rank receives per step (outputs + grads of the other ranks)."""
        other = self.global_batch - self.local_batch
        return other * (self.outputs.shape[1] + self.grads.shape[1]) * self.outputs.element_size()
