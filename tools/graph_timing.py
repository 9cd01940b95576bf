import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2410_11415_b200 import _lib, engine
from paper_2410_11415_b200.tensorized import load_npz
dev = torch.device("cuda", 0)
for name, B, dt in (("C", 1024, np.float32), ("B", 256, np.float64), ("A", 1, np.float64), ("E", 128, np.float64)):
    tc = load_npz(f"data/circuits/{name}.npz")
    plan = engine.device_plan(tc, dev)
    code = _lib.KLAY_LOG
    w = torch.from_numpy(np.log(np.random.default_rng(0).uniform(0.05, 0.95, (B, tc.num_inputs))).astype(dt)).to(dev)
    vals = plan.alloc_values(B, dt); work = plan.workspace(B, dt); fw = plan.forward_workspace(B, dt)
    out = torch.empty((B, tc.num_roots), dtype=w.dtype, device=dev); g = torch.empty((B, tc.num_inputs), dtype=w.dtype, device=dev)
    def step():
        plan.forward(w, code, dt, values=vals, outputs=out, workspace=fw)
        plan.backward(vals, B, code, dt, grads=g, workspace=work)
    for _ in range(3): step()
    torch.cuda.synchronize()
    def timeit(fn, n=50):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    t_stream = timeit(step)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    graph.replay(); torch.cuda.synchronize()
    t_graph = timeit(graph.replay)
    ref = g.clone(); graph.replay(); torch.cuda.synchronize()
    step(); torch.cuda.synchronize()
    print(name, B, f"stream {t_stream:.3f} ms graph {t_graph:.3f} ms", "same" if torch.equal(ref, g) else "DIFF", flush=True)
