"""Localize alias-path mismatches: per-layer forward trace and gradient of a
config vs the oracle (log fp64, epsilon 0). python tools/dbg_alias.py A"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import CONFIGS, load_case, load_config  # noqa: E402
from oracle import engine_port as oracle  # noqa: E402
from paper_2410_11415_b200 import _lib, device_plan  # noqa: E402
from paper_2410_11415_b200.engine import _NodeValues  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "A"
tc, gold = (load_config if name in CONFIGS else load_case)(name)
w = gold["w_real"]
with np.errstate(divide="ignore"):
    lw = np.log(w)
dev = torch.device("cuda", 0)
plan = device_plan(tc, dev)
B = lw.shape[0]
x = torch.tensor(lw, dtype=torch.float64, device=dev)
out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64).cpu().numpy()
with np.errstate(all="ignore"):
    ref, tr = oracle.forward(tc, lw, "log")
    gref = oracle.backward(tc, tr, "log")


def bad(a, b):
    fin = np.isfinite(b)
    d = np.zeros(a.shape, bool)
    d |= np.isnan(a) != np.isnan(b)
    d[fin] |= np.abs(a[fin] - b[fin]) > 1e-9 * np.maximum(np.abs(b[fin]), 1e-300)
    d[~fin & ~np.isnan(b)] |= a[~fin & ~np.isnan(b)] != b[~fin & ~np.isnan(b)]
    return d


print("roots bad:", bad(out.cpu().numpy(), ref).sum(), "grad bad:", bad(g, gref).sum(), "of", g.size)
nv = _NodeValues(plan, vals, B)
for l in range(len(tr)):
    d = bad(nv[l], tr[l])
    if d.any():
        print("trace layer", l, "bad", d.sum(), "of", d.size, "first", np.argwhere(d)[:3].tolist())
        break
else:
    print("trace ok")
# adjoint per layer is internal; report the worst grad columns
if bad(g, gref).any():
    cols = np.nonzero(bad(g, gref).any(0))[0]
    print("bad grad columns", cols[:10], "example", g[0, cols[:3]], gref[0, cols[:3]])
