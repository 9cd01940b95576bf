import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_11415_b200 import engine
from paper_2410_11415_b200.tensorized import load_npz
tc = load_npz("data/circuits/C.npz")
B = 1024
w = np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs))).astype(np.float32)
W = engine.WeightAssignment(w, "log")
for _ in range(3): engine.gradient(tc, W, log_domain=True, dtype=np.float32)
torch.cuda.synchronize()
def t(f, n=30):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
print("gradient total us", t(lambda: engine.gradient(tc, W, log_domain=True, dtype=np.float32)))
cap = list(engine._PASS_CACHE.values())[0]
stream = torch.cuda.current_stream()
def rep():
    cap.replay(); stream.synchronize()
print("replay+sync us", t(rep))
print("to_log us", t(lambda: W.to_log()))
print("device_plan us", t(lambda: engine.device_plan(tc)))
print("check_shapes us", t(lambda: engine._check_shapes(tc, W)))
def copyin():
    cap.h_weights.numpy()[...] = W.values
print("copyin us", t(copyin))
print("copyout us", t(lambda: (cap.h_out.numpy().copy(), cap.h_grad.numpy().copy())))
# device-only graph (no host io)
plan = engine.device_plan(tc)
cap2 = plan.capture(B, np.float32, 1, epsilon=0.0, backward=True, seeded=False, host_io=False)
def rep2():
    cap2.replay(); stream.synchronize()
print("device graph replay+sync us", t(rep2))
# line-by-line timing of engine.gradient's body
import collections
acc = collections.defaultdict(float)
N = 30
for _ in range(N):
    t0 = time.perf_counter()
    w2 = W.to_log()
    engine._check_shapes(tc, w2)
    dt = engine._resolve_dtype(np.float32)
    plan = engine.device_plan(tc)
    key = (id(plan), B, np.dtype(dt).str, 1, 0.0, False)
    cap = engine._PASS_CACHE.get(key)
    t1 = time.perf_counter()
    stream = torch.cuda.current_stream(plan.device)
    t2 = time.perf_counter()
    cap.h_weights.numpy()[...] = w2.values
    t3 = time.perf_counter()
    cap.replay()
    t4 = time.perf_counter()
    stream.synchronize()
    t5 = time.perf_counter()
    r = cap.h_out.numpy().copy(), cap.h_grad.numpy().copy()
    t6 = time.perf_counter()
    for k, a, b in (("pre", t0, t1), ("stream", t1, t2), ("copyin", t2, t3), ("replay", t3, t4),
                    ("sync", t4, t5), ("copyout", t5, t6)):
        acc[k] += (b - a) / N * 1e6
print({k: round(v, 1) for k, v in acc.items()}, "dtype", W.values.dtype)
# host copy variants
wt = torch.from_numpy(W.values)
hw = cap.h_weights
def c_np():
    hw.numpy()[...] = W.values
def c_torch():
    hw.copy_(wt)
print("copyin numpy us", t(c_np, 200), "torch us", t(c_torch, 200), "threads", torch.get_num_threads())
ho, hg = cap.h_out, cap.h_grad
def o_np():
    return ho.numpy().copy(), hg.numpy().copy()
def o_torch():
    return ho.clone().numpy(), hg.clone().numpy()
def o_empty():
    a = np.empty(hg.shape, np.float32); a[...] = hg.numpy(); b = np.empty(ho.shape, np.float32); b[...] = ho.numpy(); return b, a
print("copyout numpy us", t(o_np, 200), "torch us", t(o_torch, 200), "empty+assign", t(o_empty, 200))
