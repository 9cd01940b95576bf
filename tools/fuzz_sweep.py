"""Long random-circuit sweep against the CPU oracle (GPU box; not part of
the test suite): many seeds of tests/test_fuzz_gpu.random_circuit with random
shapes and batch sizes, real fp64 bit-exact and log fp64 rel 1e-12, values,
gradients and every trace layer.
    python tools/fuzz_sweep.py [n_seeds] [first_seed]"""
import os
import sys

import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from conftest import rel_close  # noqa: E402
from oracle import engine_port as oracle  # noqa: E402
from paper_2410_11415_b200 import _lib, device_plan  # noqa: E402
from paper_2410_11415_b200.engine import _NodeValues  # noqa: E402
from test_fuzz_gpu import random_circuit  # noqa: E402

warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
first = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
dev = torch.device("cuda", 0)
bad = done = 0
for seed in range(first, first + n):
    rng = np.random.default_rng(seed)
    K = int(rng.integers(4, 120)) * 2
    L = int(rng.integers(2, 16))
    try:
        tc = random_circuit(seed, K=K, L=L, wmax=int(rng.integers(8, 3000)), grow=int(rng.integers(1, 4)))
    except ValueError:  # widths too narrow for the drawn shape
        continue
    done += 1
    plan = device_plan(tc)
    B = int(rng.integers(1, 300))
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    w[rng.uniform(size=w.shape) < 0.04] = 0.0
    try:
        x = torch.tensor(w, dtype=torch.float64, device=dev)
        out, vals = plan.forward(x, _lib.KLAY_REAL, np.float64)
        g = plan.backward(vals, B, _lib.KLAY_REAL, np.float64)
        ref, tr = oracle.forward(tc, w, "real")
        assert np.array_equal(out.cpu().numpy(), ref, equal_nan=True), "real out"
        np.testing.assert_array_equal(g.cpu().numpy(), oracle.backward(tc, tr, "real"))
        with np.errstate(divide="ignore"):
            lw = np.log(w)
        x = torch.tensor(lw, dtype=torch.float64, device=dev)
        out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
        g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
        with np.errstate(all="ignore"):
            ref, tr = oracle.forward(tc, lw, "log")
            gref = oracle.backward(tc, tr, "log")
        rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
        rel_close(g.cpu().numpy(), gref, 1e-12, 1e-12)
        nv = _NodeValues(plan, vals, B)
        for l in range(len(tr)):
            rel_close(nv[l], tr[l], 1e-12, 1e-12)
    except AssertionError as e:
        bad += 1
        print(f"seed {seed}: K={K} L={L} B={B} schedule={plan.schedule}: {str(e)[:300]}")
print(f"fuzz sweep: {done - bad} / {done} circuits ok ({n - done} seeds drew no valid shape)")
