"""Generate golden vectors by running the REFERENCE engine in this container.

    python tools/gen_golden.py            # small cases + configs A-D

The reference (``/root/reference/pkg/src/laycirc``) is importable only here;
its outputs are frozen into ``tests/golden/`` so the GPU box (which has no
``/root/reference``) can check the CUDA path and the oracle against them.

Per case ``<name>``:
  tests/golden/circuits/<name>.npz   tensorized circuit (paper_2410_11415_b200.tensorized.save_npz)
  tests/golden/<name>.npz            weights + reference results:
     w_real [B,K] fp64    real-domain rows (some with exact zeros)
     w_bool [B,K] fp64    0/1 rows
     seed   [B,R] fp64    random backward seed
     real_out/real_grad, real_grad_seed          forward_real + backward
     log_out/log_grad, log_grad_seed             forward_log(to_log) + backward
     logeps_out/logeps_grad                      epsilon = 1e-3
     real32_out/real32_grad, log32_out/log32_grad  dtype=np.float32
     bool_out, maxprod_out                       evaluate_semiring
Config circuits (A-D) are read from data/circuits/ (tools/gen_circuits.py).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, ROOT)

import laycirc  # noqa: E402
from laycirc import (  # noqa: E402
    Circuit, Literal, WeightAssignment, backward, evaluate_semiring,
    forward_log, forward_real, layerize, tensorize,
)
from laycirc.bench import rng_for  # noqa: E402
import conftest as refconf  # noqa: E402  (reference test fixtures)

from paper_2410_11415_b200.tensorized import load_npz, save_npz  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def small_cases():
    cases = {}
    cases["fig_main"] = [refconf.build_fig_main()]
    cases["fig_second"] = [refconf.build_fig_second()]
    cases["fig_pair_merge"] = [refconf.build_fig_main(), refconf.build_fig_second()]
    cases["fig_dup_roots"] = [refconf.build_fig_main(), refconf.build_fig_main()]
    cases["single_leaf"] = [refconf.build_single_leaf()]
    cases["tautology"] = [refconf.build_tautology()]
    unsat = Circuit(num_vars=1)
    unsat.set_roots([unsat.add_false()])
    taut = Circuit(num_vars=1)
    taut.set_roots([taut.add_true()])
    cases["constants"] = [refconf.build_fig_main(), unsat, taut]
    c = Circuit(num_vars=3)
    kids = [c.add_leaf(Literal(v)) for v in (1, 2, 3)]
    c.set_roots([c.add_and(kids)])
    cases["and3"] = [c]
    c = Circuit(num_vars=3)
    kids = [c.add_and([c.add_leaf(Literal(v)), c.add_leaf(Literal(v, False))]) for v in (1, 2, 3)]
    c.set_roots([c.add_or(kids)])
    cases["sum3"] = [c]
    c = Circuit(num_vars=2)
    x = c.add_leaf(Literal(1))
    y = c.add_leaf(Literal(2))
    c.set_roots([c.add_or([c.add_and([x, y]), c.add_and([x, x])])])
    cases["dup_child"] = [c]
    for i, circ in enumerate(refconf.compiled_corpus(count=6, seed=321)):
        cases[f"corpus_{i}"] = [circ]
    # wide fan-in / long segments: the random-NNF generator (root fan-in = width)
    cases["rnnf_small"] = [laycirc.bench.gen_random_nnf(12, 300, 4, 3, 5)]
    cases["rnnf_wide"] = [laycirc.bench.gen_random_nnf(8, 3000, 3, 40, 7)]
    return {k: tensorize(layerize(v)) for k, v in cases.items()}


def weights_for(tc, rng, batch):
    K = tc.num_inputs
    w = rng.uniform(0.05, 0.95, size=(batch, K))
    # rows 1 and 2 carry exact zeros: -inf in the log domain, zero-safe
    # product adjoints in the real domain
    if batch >= 3 and K >= 1:
        w[1, rng.integers(0, K, size=max(1, K // 8))] = 0.0
        w[2, rng.integers(0, K, size=max(1, K // 3))] = 0.0
    if batch >= 4:
        w[3, :] = 0.0  # everything zero: all -inf segments everywhere
    wb = rng.integers(0, 2, size=(batch, K)).astype(np.float64)
    seed = rng.uniform(-1.0, 1.0, size=(batch, tc.num_roots))
    return w, wb, seed


def run_reference(tc, w, wb, seed, eps=1e-3, with_grads=True):
    res = {"w_real": w, "w_bool": wb, "seed": seed}
    W = WeightAssignment(w)
    tr = forward_real(tc, W)
    res["real_out"] = tr.outputs
    if with_grads:
        res["real_grad"] = backward(tc, tr)
        res["real_grad_seed"] = backward(tc, tr, seed)
    L = W.to_log()
    tr = forward_log(tc, L)
    res["log_out"] = tr.outputs
    if with_grads:
        res["log_grad"] = backward(tc, tr)
        res["log_grad_seed"] = backward(tc, tr, seed)
    tr = forward_log(tc, L, epsilon=eps)
    res["logeps_out"] = tr.outputs
    if with_grads:
        res["logeps_grad"] = backward(tc, tr)
    tr = forward_real(tc, W, dtype=np.float32)
    res["real32_out"] = tr.outputs
    if with_grads:
        res["real32_grad"] = backward(tc, tr)
    tr = forward_log(tc, L, dtype=np.float32)
    res["log32_out"] = tr.outputs
    if with_grads:
        res["log32_grad"] = backward(tc, tr)
    res["bool_out"] = evaluate_semiring(tc, WeightAssignment(wb), "bool")
    res["maxprod_out"] = evaluate_semiring(tc, W, "maxprod")
    return res


def main(argv):
    os.makedirs(os.path.join(GOLD, "circuits"), exist_ok=True)
    rng = rng_for(20241015)
    if "small" in argv or not argv:
        for name, tc in small_cases().items():
            save_npz(tc, os.path.join(GOLD, "circuits", f"{name}.npz"))
            w, wb, seed = weights_for(tc, rng, 6)
            np.savez_compressed(os.path.join(GOLD, f"{name}.npz"), **run_reference(tc, w, wb, seed))
            print("golden", name, tc.num_inputs, [l.width for l in tc.layers], flush=True)
    for cfg in ("A", "B", "C", "D", "E", "Cp"):
        if argv and cfg not in argv:
            continue
        path = os.path.join(ROOT, "data", "circuits", f"{cfg}.npz")
        if not os.path.exists(path):
            print("skip", cfg, "(no circuit)")
            continue
        tc = load_npz(path)
        w, wb, seed = weights_for(tc, rng, 8)
        np.savez_compressed(os.path.join(GOLD, f"cfg{cfg}.npz"), **run_reference(tc, w, wb, seed))
        print("golden config", cfg, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
