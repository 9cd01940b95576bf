"""Device-timed evals/s of the non-headline configs (bench.measure_config),
one line per config: python tools/extra_configs.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.argv = sys.argv[:1]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
cases = [("A", "real", np.float64, 1, False), ("B", "log", np.float64, 256, True),
         ("D", "bool", np.float32, 4096, False), ("D", "bool_packed", "u1", 4096, False),
         ("D", "real", np.float32, 4096, False), ("E", "log", np.float64, 128, True),
         ("Cp", "log", np.float32, 1024, True)]
for name, sr, dt, B, bwd in cases:
    r = bench.measure_config(name, sr, dt, B, bwd, dev, iters=5 if name == "Cp" else 20)
    print(f"{name:3s} {sr:12s} B={B:5d} {r['evals_per_s']:12.0f} evals/s  frac {r.get('roofline_frac', 0) or 0:.3f}")
