"""Per-layer timing of the persistent tail (KLAY_TAIL_TRACE=1 globaltimer
stamps) on config C: python tools/tail_trace.py [B]"""
import os
import sys

os.environ["KLAY_TAIL_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_11415_b200 import _lib, engine  # noqa: E402
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device("cuda", 0)
tc = load_npz("data/circuits/C.npz")
plan = engine.device_plan(tc, dev)
dt = np.float32
w = torch.from_numpy(np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs))).astype(dt)).to(dev)
for _ in range(3):
    out, vals = plan.forward(w, _lib.KLAY_LOG, dt)
    plan.backward(vals, B, _lib.KLAY_LOG, dt)
torch.cuda.synchronize()
widths = [l.width for l in tc.layers]
edges = [len(l.sources) for l in tc.layers]
print("layer widths (last 50):", widths[-50:])
print("layer edges  (last 50):", edges[-50:])
