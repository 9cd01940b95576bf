"""In-graph time per launch class (bench.time_classes) for any config:
    python tools/class_breakdown.py B float64 256 [log|real]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2410_11415_b200 import _lib, engine  # noqa: E402
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

cfg, dt, B = sys.argv[1], np.dtype(sys.argv[2]).type, int(sys.argv[3])
sr = {"log": _lib.KLAY_LOG, "real": _lib.KLAY_REAL}[sys.argv[4] if len(sys.argv) > 4 else "log"]
tc = load_npz(os.path.join("data", "circuits", f"{cfg}.npz"))
dev = torch.device("cuda", 0)
plan = engine.device_plan(tc, dev)
cap = plan.capture(B, dt, sr, backward=True)
w = np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs))
cap.weights.copy_(torch.from_numpy(np.log(w) if sr == _lib.KLAY_LOG else w))
for _ in range(3):
    cap.replay()
ms = bench._timed_replays(cap.replay, 20, dev)
lib = _lib.load()


def step():
    plan.forward(cap.weights, sr, dt, retain=True, values=cap.values, outputs=cap.outputs, workspace=cap._fw)
    plan.backward(cap.values, B, sr, dt, grads=cap.grads, workspace=cap._bw)


ct = bench.time_classes(lib, step, iters=20)
s = 8 if dt == np.float64 else 4
print(f"{cfg} {np.dtype(dt).name} B={B}: step {ms:.4f} ms = {B / ms * 1e3:.0f} evals/s; "
      f"schedule {plan.schedule}")
for c, t in ct.items():
    print(f"  {c:12s} {t['launches']:3d} launches {t['ms']:.4f} ms")
