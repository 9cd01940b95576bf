"""Worst fp32 error of the log semiring vs the fp64 reference goldens
(roots: relative; grads: relative to the grad scale, as the tests measure)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402

from conftest import load_config  # noqa: E402
from paper_2410_11415_b200 import engine as k  # noqa: E402

for name in ("A", "B", "C", "D", "E", "Cp"):
    tc, gold = load_config(name)
    if "log_out" not in gold:
        continue
    W = k.WeightAssignment(gold["w_real"])
    tr = k.forward_log(tc, W.to_log(), dtype=np.float32)
    o, ro = tr.outputs.astype(np.float64), gold["log_out"]
    fin = np.isfinite(ro)
    rel = np.max(np.abs(o[fin] - ro[fin]) / np.maximum(np.abs(ro[fin]), 1e-300)) if fin.any() else 0
    msg = f"{name}: roots max rel {rel:.2e}"
    if "log_grad" in gold:
        g = k.backward(tc, tr).astype(np.float64)
        rg = gold["log_grad"]
        f2 = np.isfinite(rg)
        scale = np.abs(rg[f2]).max()
        err = np.abs(g[f2] - rg[f2]) / (np.abs(rg[f2]) + scale)
        msg += f"; grads max err/(|g|+scale) {err.max():.2e}"
    print(msg)
