"""Neurosymbolic training step on MNIST-addition-shaped inputs (SURVEY §8(d)
config E): a random-init MLP classifies each digit image, its log-softmax
feeds the semantic-loss circuit (2-digit addition, 199 roots) evaluated on
the B200 path in the log semiring (fp64), loss = -log P(sum = label).

    python examples/mnist_addition.py [--steps 5] [--batch 128]
    torchrun --nproc-per-node N examples/mnist_addition.py   # DDP, NCCL grad all-reduce

Synthetic data (N(0,1) images, random digits); no dataset download.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_11415_b200 import CircuitModule, load_npz  # noqa: E402

NDIGITS = 2
NPOS = 2 * NDIGITS


def slot_index(tc):
    """Per (position, digit): slot of literal x[p,d] and of its negation
    (variable p*10+d+1, see tools/gen_circuits.py mnist_addition)."""
    pos = torch.empty(NPOS, 10, dtype=torch.long)
    neg = torch.empty(NPOS, 10, dtype=torch.long)
    for lit, slot in tc.input_map.items():
        p, d = divmod(lit.variable - 1, 10)
        (pos if lit.positive else neg)[p, d] = slot
    return pos, neg


class DigitMLP(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.net = torch.nn.Sequential(torch.nn.Flatten(), torch.nn.Linear(784, 256),
                                       torch.nn.ReLU(), torch.nn.Linear(256, 10))

    def forward(self, x):  # [B, NPOS, 28, 28] -> [B, NPOS, 10] log-probabilities
        B = x.shape[0]
        return torch.log_softmax(self.net(x.reshape(B * NPOS, 28, 28)), -1).reshape(B, NPOS, 10)


def circuit_weights(logp, pos, neg, K):
    """Log-weights of the circuit inputs: x[p,d] -> log p(d | image p), not x -> log 1."""
    B = logp.shape[0]
    w = torch.zeros(B, K, dtype=logp.dtype, device=logp.device)
    w = w.index_put((torch.arange(B, device=logp.device)[:, None], pos.reshape(1, -1).expand(B, -1).to(logp.device)),
                    logp.reshape(B, -1))
    return w


def make_batch(B, gen, device, dtype):
    digits = torch.randint(0, 10, (B, NPOS), generator=gen)
    images = torch.randn(B, NPOS, 28, 28, generator=gen, dtype=dtype)
    a = digits[:, 1] * 10 + digits[:, 0]
    b = digits[:, 3] * 10 + digits[:, 2]
    return images.to(device), (a + b).to(device)


def train_step(mlp, circuit, opt, images, labels, pos, neg):
    opt.zero_grad(set_to_none=True)
    w = circuit_weights(mlp(images), pos, neg, circuit.num_inputs)
    roots = circuit(w)                                   # [B, 199] log-WMC per sum
    loss = -roots[torch.arange(len(labels), device=roots.device), labels].mean()
    loss.backward()                                      # circuit backward on B200, then MLP
    opt.step()
    return loss.detach()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=128, help="per GPU")
    args = ap.parse_args()
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    tc = load_npz(os.path.join(ROOT, "data", "circuits", "E.npz"))
    circuit = CircuitModule(tc, "log", device=dev)
    mlp = DigitMLP().to(dev, torch.float64)
    if world > 1:
        mlp = torch.nn.parallel.DistributedDataParallel(mlp, device_ids=[local])
    opt = torch.optim.SGD(mlp.parameters(), lr=0.1)
    pos, neg = slot_index(tc)
    gen = torch.Generator().manual_seed(1000 + rank)
    for step in range(args.steps):
        images, labels = make_batch(args.batch, gen, dev, torch.float64)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        loss = train_step(mlp, circuit, opt, images, labels, pos, neg)
        torch.cuda.synchronize()
        if rank == 0:
            print(f"step {step} loss {loss.item():.6f} {1e3 * (time.perf_counter() - t0):.2f} ms")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
