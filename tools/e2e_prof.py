"""Where engine.gradient's host-side time goes (GPU box): config C, log fp32,
B = 1024, the bench's e2e call, stage by stage.
    python tools/e2e_prof.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_11415_b200 import engine  # noqa: E402
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

tc = load_npz(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "circuits", "C.npz"))
B = 1024
rows = np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs))).astype(np.float32)


def api():
    return engine.gradient(tc, engine.WeightAssignment(rows, "log"), log_domain=True, dtype=np.float32)


for _ in range(3):
    api()
torch.cuda.synchronize()


def t(f, n=40):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


plan = engine.device_plan(tc)
cap = plan._grad_pass[1]
W = engine.WeightAssignment(rows, "log")
stream = torch.cuda.current_stream(plan.device)


def rep():
    cap.replay()
    stream.synchronize()


print(f"gradient() total          {t(api):8.1f} us")
print(f"WeightAssignment(rows)    {t(lambda: engine.WeightAssignment(rows, 'log')):8.1f} us")
print(f"to_log + check_shapes     {t(lambda: engine._check_shapes(tc, W.to_log())):8.1f} us")
print(f"device_plan lookup        {t(lambda: engine.device_plan(tc)):8.1f} us")
print(f"copy-in (torch copy_)     {t(lambda: cap.h_weights.copy_(torch.from_numpy(np.ascontiguousarray(W.values)))):8.1f} us")
print(f"replay + sync             {t(rep):8.1f} us")
print(f"copy-out (2 clones)       {t(lambda: (cap.h_out.clone().numpy(), cap.h_grad.clone().numpy())):8.1f} us")
cap2 = plan.capture(B, np.float32, 1, epsilon=0.0, backward=True, seeded=False, host_io=False)


def rep2():
    cap2.replay()
    stream.synchronize()


print(f"device-only graph + sync  {t(rep2):8.1f} us")
