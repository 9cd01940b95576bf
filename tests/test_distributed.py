"""Multi-process (world_size 2, gloo, CPU) coverage of the batch-sharded path:
each rank evaluates its rows (here with the CPU oracle standing in for the
device evaluation) and the all-gathered result equals the single-process
evaluation of the whole batch, bit for bit (rows are independent)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import load_case


def test_shard_bounds_cover_batch():
    from paper_2410_11415_b200.distributed import shard_bounds
    for B in (1, 2, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            ranges = [shard_bounds(B, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, result_dir):
    import torch.distributed as dist

    from oracle import engine_port as oracle
    from paper_2410_11415_b200.distributed import sharded_eval

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tc, gold = load_case(name)
        rng = np.random.default_rng(11)
        w = np.log(rng.uniform(0.05, 0.95, size=(7, tc.num_inputs)))

        def evaluate(rows):
            out, tr = oracle.forward(tc, rows, "log")
            return out, oracle.backward(tc, tr, "log")

        out, grad = sharded_eval(evaluate, w, world, rank)
        np.save(os.path.join(result_dir, f"out{rank}.npy"), out)
        np.save(os.path.join(result_dir, f"grad{rank}.npy"), grad)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["fig_pair_merge", "corpus_5"])
def test_two_rank_gloo_sharding_matches_single_process(tmp_path, name):
    from oracle import engine_port as oracle
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    tc, _ = load_case(name)
    rng = np.random.default_rng(11)
    w = np.log(rng.uniform(0.05, 0.95, size=(7, tc.num_inputs)))
    out, tr = oracle.forward(tc, w, "log")
    grad = oracle.backward(tc, tr, "log")
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"out{r}.npy"), out)
        assert np.array_equal(np.load(tmp_path / f"grad{r}.npy"), grad)


def _gather_worker(rank, world, port, result_dir):
    import torch
    import torch.distributed as dist

    from paper_2410_11415_b200.distributed import gather_rows, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 11
        sizes = [b - a for a, b in (shard_bounds(B, world, r) for r in range(world))]
        lo, hi = shard_bounds(B, world, rank)
        full = torch.arange(B * 3, dtype=torch.float64).reshape(B, 3)
        out = torch.full((B, 3), -1.0, dtype=torch.float64)
        got = gather_rows(full[lo:hi], world, sizes=sizes, out=out)
        assert got is out
        assert torch.equal(out, full)
        got2 = gather_rows(full[lo:hi].clone(), world)  # counts exchanged
        assert torch.equal(got2, full)
        try:
            gather_rows(full[lo:hi], world, sizes=[B, 0, 0][:world])
            bad = False
        except ValueError:
            bad = True
        np.save(os.path.join(result_dir, f"ok{rank}.npy"), np.array([bad]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_rows_uneven_into_out(tmp_path):
    """gather_rows with precomputed shard sizes (bench.py / ShardedPass) and
    a preallocated output, uneven shards (6 + 5 rows), and a size mismatch
    raising ValueError on the rank whose count disagrees."""
    world = 2
    mp.start_processes(_gather_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    assert bool(np.load(tmp_path / "ok1.npy")[0])
