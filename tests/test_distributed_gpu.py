"""Two ranks through libklay: the batch-sharded device path (ShardedPass,
bench.py's multi-GPU arm) and the config E DDP training step.

The box has one GPU, so both ranks run on cuda:0 as separate processes with
the gloo backend (NCCL refuses two ranks on one device). Nothing waits on
another rank inside a kernel: each rank's graph is independent and only the
host-side collective couples them (B200_PROFILING.md). The sharded results
must equal the single-process evaluation of the whole batch bit for bit
(rows are independent: the reference's test_engine.py:72-86)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import CIRCUITS, load_case

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _weights(tc, B, seed=11):
    rng = np.random.default_rng(seed)
    return np.log(rng.uniform(0.05, 0.95, size=(B, tc.num_inputs)))


def _load(name):
    from paper_2410_11415_b200.tensorized import load_npz
    if name in ("B", "E"):
        return load_npz(os.path.join(CIRCUITS, f"{name}.npz"))
    return load_case(name)[0]


def _shard_worker(rank, world, port, name, B, dtype, result_dir):
    import torch
    import torch.distributed as dist

    from paper_2410_11415_b200 import _lib
    from paper_2410_11415_b200.distributed import ShardedPass

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tc = _load(name)
        w = _weights(tc, B)
        sp = ShardedPass(tc, B, dtype, _lib.KLAY_LOG, world, rank)
        sp.weights.copy_(torch.from_numpy(w[sp.lo:sp.hi].astype(dtype)))
        out, grad = sp.step()
        torch.cuda.synchronize()
        np.save(os.path.join(result_dir, f"out{rank}.npy"), out.cpu().numpy())
        np.save(os.path.join(result_dir, f"grad{rank}.npy"), grad.cpu().numpy())
        np.save(os.path.join(result_dir, f"rows{rank}.npy"), np.array([sp.lo, sp.hi]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,B,dtype", [("corpus_5", 7, np.float64), ("B", 256, np.float32),
                                          ("E", 129, np.float64)])
def test_two_rank_sharded_pass_matches_single_process(cuda, tmp_path, name, B, dtype):
    import torch

    from paper_2410_11415_b200 import _lib, engine
    world = 2
    mp.start_processes(_shard_worker, args=(world, _free_port(), name, B, dtype, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    tc = _load(name)
    w = _weights(tc, B)
    cap = engine.device_plan(tc, cuda).capture(B, dtype, _lib.KLAY_LOG, backward=True)
    cap.weights.copy_(torch.from_numpy(w.astype(dtype)))
    cap.replay()
    torch.cuda.synchronize()
    out, grad = cap.outputs.cpu().numpy(), cap.grads.cpu().numpy()
    rows = [tuple(np.load(tmp_path / f"rows{r}.npy")) for r in range(world)]
    assert rows == [(0, (B + 1) // 2), ((B + 1) // 2, B)]
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"out{r}.npy"), out, equal_nan=True)
        assert np.array_equal(np.load(tmp_path / f"grad{r}.npy"), grad, equal_nan=True)


def _ddp_worker(rank, world, port, B, result_dir):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "examples"))
    import mnist_addition as ma

    from paper_2410_11415_b200 import CircuitModule
    from paper_2410_11415_b200.distributed import shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tc = _load("E")
        circuit = CircuitModule(tc, "log", device=dev)
        torch.manual_seed(0)
        mlp = torch.nn.parallel.DistributedDataParallel(ma.DigitMLP().to(dev, torch.float64))
        pos, neg = ma.slot_index(tc)
        images, labels = ma.make_batch(B, torch.Generator().manual_seed(5), dev, torch.float64)
        lo, hi = shard_bounds(B, world, rank)
        opt = torch.optim.SGD(mlp.parameters(), lr=0.01)
        loss = ma.train_step(mlp, circuit, opt, images[lo:hi], labels[lo:hi], pos, neg)
        # SGD already stepped: report the post-step parameters and the grads
        grads = [p.grad.detach().cpu().numpy() for p in mlp.parameters()]
        params = [p.detach().cpu().numpy() for p in mlp.parameters()]
        np.savez(os.path.join(result_dir, f"ddp{rank}.npz"), loss=loss.cpu().numpy(),
                 **{f"g{i}": g for i, g in enumerate(grads)},
                 **{f"p{i}": p for i, p in enumerate(params)})
    finally:
        dist.destroy_process_group()


def test_two_rank_ddp_training_step_matches_full_batch(cuda, tmp_path):
    """Config E under DDP (2 ranks x 16 rows): the all-reduced MLP gradients
    and the updated parameters equal the single-process step on all 32
    rows (fp64; only the reduction order of the mean differs)."""
    import sys

    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "examples"))
    import mnist_addition as ma

    from paper_2410_11415_b200 import CircuitModule
    world, B = 2, 32
    mp.start_processes(_ddp_worker, args=(world, _free_port(), B, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    tc = _load("E")
    circuit = CircuitModule(tc, "log", device=cuda)
    torch.manual_seed(0)
    mlp = ma.DigitMLP().to(cuda, torch.float64)
    pos, neg = ma.slot_index(tc)
    images, labels = ma.make_batch(B, torch.Generator().manual_seed(5), cuda, torch.float64)
    opt = torch.optim.SGD(mlp.parameters(), lr=0.01)
    ma.train_step(mlp, circuit, opt, images, labels, pos, neg)
    ref_g = [p.grad.detach().cpu().numpy() for p in mlp.parameters()]
    ref_p = [p.detach().cpu().numpy() for p in mlp.parameters()]
    for r in range(world):
        got = np.load(tmp_path / f"ddp{r}.npz")
        for i, (g, p) in enumerate(zip(ref_g, ref_p)):
            scale = max(np.abs(g).max(), 1e-300)
            assert np.abs(got[f"g{i}"] - g).max() <= 1e-12 * scale, (r, i)
            assert np.allclose(got[f"p{i}"], p, rtol=1e-12, atol=1e-15), (r, i)
