"""Torch surface (CircuitModule / KlayFunction) and the config E training
step: autograd gradients equal the reference backward with seed =
grad_output (fp64 rel 1e-12; fp32 elementwise vs fp64 within max(1e-5 rel,
2x the reference's own fp32 error), conftest.fp32_close)."""

import numpy as np
import pytest

from conftest import fp32_close, load_case, load_config, rel_close

pytestmark = pytest.mark.gpu


def test_module_forward_backward_matches_oracle(cuda):
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import CircuitModule
    for name in ("fig_pair_merge", "constants", "corpus_5"):
        tc, gold = load_case(name)
        lw = np.log(gold["w_real"])
        for dt, rtol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
            layer = CircuitModule(tc, "log")
            w = torch.tensor(lw, dtype=dt, device=cuda, requires_grad=True)
            roots = layer(w)
            seed = torch.tensor(gold["seed"], dtype=dt, device=cuda)
            (roots * seed).sum().backward()
            if dt == torch.float64:
                rel_close(roots.detach().cpu().numpy(), gold["log_out"], rtol)
                rel_close(w.grad.cpu().numpy(), gold["log_grad_seed"], rtol, rtol)
            else:  # elementwise vs the reference's own fp32 run (oracle, bit-identical)
                with np.errstate(all="ignore"):
                    o32, t32 = oracle.forward(tc, lw.astype(np.float32), "log")
                    g32 = oracle.backward(tc, t32, "log", gold["seed"].astype(np.float32))
                fp32_close(roots.detach().cpu().numpy(), gold["log_out"], o32)
                fp32_close(w.grad.cpu().numpy(), gold["log_grad_seed"], g32)
        layer = CircuitModule(tc, "real")
        w = torch.tensor(gold["w_real"], dtype=torch.float64, device=cuda, requires_grad=True)
        layer(w).sum().backward()
        assert np.array_equal(w.grad.cpu().numpy(), gold["real_grad"])
        out = CircuitModule(tc, "bool")(torch.tensor(gold["w_bool"], device=cuda))
        assert np.array_equal(out.cpu().numpy(), gold["bool_out"])
        _ = oracle


def test_module_gradcheck_small(cuda):
    import torch
    from paper_2410_11415_b200 import CircuitModule
    tc, gold = load_case("fig_main")
    layer = CircuitModule(tc, "log")
    w = torch.tensor(np.log(gold["w_real"][:2]), dtype=torch.float64, device=cuda,
                     requires_grad=True)
    assert torch.autograd.gradcheck(layer, (w,), eps=1e-6, atol=1e-7, rtol=1e-5)


def test_mnist_addition_training_step(cuda):
    """Config E: one training step; the circuit's input gradient equals the
    oracle's backward with seed = -onehot(label)/B, and the loss decreases
    over a few SGD steps on a fixed batch."""
    import os
    import sys
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "examples"))
    import mnist_addition as ma
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import CircuitModule
    tc, gold = load_config("E")
    circuit = CircuitModule(tc, "log")
    torch.manual_seed(0)
    mlp = ma.DigitMLP().to(cuda, torch.float64)
    pos, neg = ma.slot_index(tc)
    gen = torch.Generator().manual_seed(5)
    images, labels = ma.make_batch(16, gen, cuda, torch.float64)
    w = ma.circuit_weights(mlp(images), pos, neg, tc.num_inputs).detach().requires_grad_(True)
    roots = circuit(w)
    loss = -roots[torch.arange(16, device=cuda), labels].mean()
    loss.backward()
    out, tr = oracle.forward(tc, w.detach().cpu().numpy(), "log")
    seed = np.zeros((16, tc.num_roots))
    seed[np.arange(16), labels.cpu().numpy()] = -1.0 / 16
    rel_close(roots.detach().cpu().numpy(), out, 1e-12)
    rel_close(w.grad.cpu().numpy(), oracle.backward(tc, tr, "log", seed), 1e-12, 1e-12)
    opt = torch.optim.SGD(mlp.parameters(), lr=0.01)
    losses = [ma.train_step(mlp, circuit, opt, images, labels, pos, neg).item() for _ in range(4)]
    assert all(b < a for a, b in zip(losses, losses[1:])), losses
