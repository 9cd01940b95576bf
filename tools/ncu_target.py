"""Minimal driver for ncu captures (GPU box): plan + N fwd+bwd steps of the
benchmark workload (config C, log fp32, B=1024), nothing else.
    python tools/ncu_target.py [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_11415_b200 import _lib, engine  # noqa: E402
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
tc = load_npz(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "data", "circuits", "C.npz"))
dev = torch.device("cuda", 0)
plan = engine.device_plan(tc, dev)
B = 1024
w = torch.from_numpy(np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs)))
                     .astype(np.float32)).to(dev)
vals = plan.alloc_values(B, np.float32)
work = plan.workspace(B, np.float32)
for _ in range(steps):
    plan.forward(w, _lib.KLAY_LOG, np.float32, values=vals)
    plan.backward(vals, B, _lib.KLAY_LOG, np.float32, workspace=work)
torch.cuda.synchronize()
print("ok")
