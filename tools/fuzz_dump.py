"""Save the GPU log fp64 gradients of fuzz seeds (for offline comparison with
a long-double oracle run): python tools/fuzz_dump.py seed ... -> gpurun_out/fz_<seed>.npz"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2410_11415_b200 import _lib, device_plan  # noqa: E402
from test_fuzz_gpu import sweep_case  # noqa: E402

warnings.simplefilter("ignore")
for seed in map(int, sys.argv[1:]):
    tc, B, w = sweep_case(seed)
    plan = device_plan(tc)
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw, dtype=torch.float64, device=torch.device("cuda", 0))
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    np.savez(os.path.join(ROOT, "gpurun_out", f"fz_{seed}.npz"), out=out.cpu().numpy(), g=g.cpu().numpy())
