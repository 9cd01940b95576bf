"""Conditioning check for fuzz seeds whose log fp64 gradients miss the 1e-12
bar: compares the GPU gradients (saved by tools/fuzz_dump.py on the box) and
the reference-order numpy fp64 oracle against the same oracle run in x87
extended precision (np.longdouble). If both fp64 results are equally far from
the extended-precision one, the miss is the circuit's conditioning, not the
kernel. CPU only; test infrastructure (imports oracle/).
    python tools/fuzz_conditioning.py 50502 50661 50992"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import engine_port as oracle  # noqa: E402
from test_fuzz_gpu import sweep_case  # noqa: E402

warnings.simplefilter("ignore")


def rel(a, ref):
    e = np.abs(a - ref)
    m = np.isfinite(e)
    return float((e[m] / (np.abs(ref[m]) + 1e-300)).max())


for seed in map(int, sys.argv[1:]):
    tc, B, w = sweep_case(seed)
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    gpu = np.load(os.path.join(ROOT, "gpurun_out", f"fz_{seed}.npz"))["g"]
    _, tr = oracle.forward(tc, lw, "log")
    g64 = oracle.backward(tc, tr, "log")
    _, trx = oracle.forward(tc, lw.astype(np.longdouble), "log")
    gx = oracle.backward(tc, trx, "log").astype(np.float64)
    print(f"seed {seed}: max rel err vs extended precision: gpu {rel(gpu, gx):.2e}, "
          f"reference-order numpy fp64 {rel(g64, gx):.2e}; gpu vs numpy fp64 {rel(gpu, g64):.2e}")
