import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2410_11415_b200 import _lib, engine
from paper_2410_11415_b200.tensorized import load_npz
tc = load_npz("data/circuits/C.npz")
dev = torch.device("cuda", 0)
plan = engine.device_plan(tc, dev)
B=1024
w = torch.from_numpy(np.log(np.random.default_rng(0).uniform(0.05,0.95,(B,tc.num_inputs))).astype(np.float32)).to(dev)
vals = plan.alloc_values(B, np.float32); work = plan.workspace(B, np.float32)
for _ in range(2):
    plan.forward(w, _lib.KLAY_LOG, np.float32, values=vals)
    plan.backward(vals, B, _lib.KLAY_LOG, np.float32, workspace=work)
torch.cuda.synchronize()
print("ok")
