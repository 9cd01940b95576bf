"""Long random-circuit sweep against the CPU oracle (GPU box; not part of
the test suite): many seeds of tests/test_fuzz_gpu.random_circuit with random
shapes and batch sizes, real fp64 bit-exact and log fp64 rel 1e-12, values,
gradients and every trace layer.

A log fp64 gradient that misses rel 1e-12 is re-judged against the same
oracle run in x87 extended precision (np.longdouble): when the GPU result is
no further from it than the reference-order numpy fp64 result is (x 2), the
miss is the circuit's conditioning, counted apart from the failures
(tools/fuzz_conditioning.py prints the numbers for single seeds).
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
from test_fuzz_gpu import sweep_case  # noqa: E402

warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
first = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
dev = torch.device("cuda", 0)
bad = done = cond = 0


def max_rel(a, ref):
    e = np.abs(a - ref)
    m = np.isfinite(e)
    return float((e[m] / (np.abs(ref[m]) + 1e-300)).max()) if m.any() else 0.0


for seed in range(first, first + n):
    case = sweep_case(seed)
    if case is None:  # widths too narrow for the drawn shape
        continue
    tc, B, w = case
    done += 1
    plan = device_plan(tc)
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
        gg = g.cpu().numpy()
        try:
            rel_close(gg, gref, 1e-12, 1e-12)
        except AssertionError:
            with np.errstate(all="ignore"):
                _, trx = oracle.forward(tc, lw.astype(np.longdouble), "log")
                gx = oracle.backward(tc, trx, "log").astype(np.float64)
            e_gpu, e_ref = max_rel(gg, gx), max_rel(gref, gx)
            if e_gpu > 2 * e_ref + 1e-12:
                raise
            cond += 1
            print(f"seed {seed}: B={B}: log fp64 gradient beyond 1e-12 of the reference, ill-conditioned: "
                  f"vs extended precision gpu {e_gpu:.2e}, reference fp64 {e_ref:.2e}")
        nv = _NodeValues(plan, vals, B)
        for l in range(len(tr)):
            rel_close(nv[l], tr[l], 1e-12, 1e-12)
    except AssertionError as e:
        bad += 1
        print(f"seed {seed}: B={B} schedule={plan.schedule}: {str(e)[:300]}")
print(f"fuzz sweep: {done - bad} / {done} circuits ok, {cond} of them with an ill-conditioned log fp64 "
      f"gradient ({n - done} seeds drew no valid shape)")
