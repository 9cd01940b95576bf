"""Minimal driver for ncu captures (GPU box): plan + N fwd+bwd steps of the
benchmark workload (config C, log fp32, B=1024; or another config), nothing else.
    python tools/ncu_target.py [steps] [config] [batch] [dtype]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_11415_b200 import _lib, engine  # noqa: E402
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = sys.argv[2] if len(sys.argv) > 2 else "C"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
dt = np.dtype(sys.argv[4]) if len(sys.argv) > 4 else np.dtype(np.float32)
tc = load_npz(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "data", "circuits", f"{cfg}.npz"))
dev = torch.device("cuda", 0)
plan = engine.device_plan(tc, dev)
w = torch.from_numpy(np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs)))
                     .astype(dt)).to(dev)
vals = plan.alloc_values(B, dt)
work = plan.workspace(B, dt)
for _ in range(steps):
    plan.forward(w, _lib.KLAY_LOG, dt, values=vals)
    plan.backward(vals, B, _lib.KLAY_LOG, dt, workspace=work)
torch.cuda.synchronize()
print("ok")
