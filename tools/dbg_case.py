"""Debug helper (GPU box): run one golden case's real / log fwd+bwd and report
parity; use with KLAY_SYNC_DEBUG=1 to locate a failing launch.
    python tools/dbg_case.py <small-case | cfgA..cfgD> [real|log] [f64|f32]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_case, load_config  # noqa: E402
import paper_2410_11415_b200 as k  # noqa: E402

name = sys.argv[1]
dom = sys.argv[2] if len(sys.argv) > 2 else "real"
dt = np.float32 if len(sys.argv) > 3 and sys.argv[3] == "f32" else np.float64
tc, gold = load_config(name[3:]) if name.startswith("cfg") else load_case(name)
rows = [0, 4, 5, 6, 7] if "nozero" in sys.argv else slice(None)
W = k.WeightAssignment(gold["w_real"][rows])
tr = k.forward_real(tc, W, dtype=dt) if dom == "real" else k.forward_log(tc, W.to_log(), dtype=dt)
print("fwd ok", flush=True)
g = k.backward(tc, tr)
ref = gold[("real" if dom == "real" else "log") + ("32" if dt == np.float32 else "") + "_grad"]
print("bwd ok; max abs err", float(np.nanmax(np.abs(g - ref[rows]))))
