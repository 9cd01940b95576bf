"""Re-run single tools/fuzz_sweep.py seeds and print the worst errors:
    python tools/fuzz_one.py seed [seed ...]"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from oracle import engine_port as oracle  # noqa: E402
from paper_2410_11415_b200 import _lib, device_plan  # noqa: E402
from test_fuzz_gpu import sweep_case  # noqa: E402

warnings.simplefilter("ignore")
dev = torch.device("cuda", 0)


def worst(got, ref):
    fin = np.isfinite(ref)
    err = np.abs(got[fin] - ref[fin])
    scale = np.abs(ref[fin]).max() if fin.any() else 1
    rel = err / np.maximum(np.abs(ref[fin]), 1e-300)
    bad = err > 1e-12 * np.abs(ref[fin]) + 1e-12 * scale
    nanmis = int((np.isnan(got) != np.isnan(ref)).sum())
    return f"max rel {rel.max():.3e} bad {int(bad.sum())}/{bad.size} nan-mismatch {nanmis}"


for seed in map(int, sys.argv[1:]):
    tc, B, w = sweep_case(seed)
    plan = device_plan(tc)
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw, dtype=torch.float64, device=dev)
    for retain in (True, "full"):
        out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64, retain=retain)
        g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
        with np.errstate(all="ignore"):
            ref, tr = oracle.forward(tc, lw, "log")
            gref = oracle.backward(tc, tr, "log")
        print(f"seed {seed} B={B} widths={[l.width for l in tc.layers]} retain={retain} "
              f"out: {worst(out.cpu().numpy(), ref)}; grad: {worst(g.cpu().numpy(), gref)}")
