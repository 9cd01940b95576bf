"""Per-launch timing of one fwd+bwd step (CUDA events around every kernel,
libklay profiler) with achieved GB/s against the algorithmic bytes of
SURVEY §8(d). Usage (GPU box):
    python tools/profile_layers.py [--config C] [--batch 1024] [--dtype f32] [--domain log]
"""

import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import layer_bytes, load_peaks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--domain", default="log")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2410_11415_b200 import _lib, engine
    from paper_2410_11415_b200.tensorized import load_npz
    tc = load_npz(os.path.join(ROOT, "data", "circuits", f"{args.config}.npz"))
    dt = np.float32 if args.dtype == "f32" else np.float64
    s = 4 if dt == np.float32 else 8
    B = args.batch
    dev = torch.device("cuda", 0)
    plan = engine.device_plan(tc, dev)
    lib = _lib.load()
    code = _lib.KLAY_LOG if args.domain == "log" else _lib.KLAY_REAL
    rng = np.random.default_rng(0)
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    if args.domain == "log":
        w = np.log(w)
    wd = torch.from_numpy(w.astype(dt)).to(dev)
    vals = plan.alloc_values(B, dt)
    work = plan.workspace(B, dt)
    for _ in range(3):
        plan.forward(wd, code, dt, values=vals)
        plan.backward(vals, B, code, dt, workspace=work)
    torch.cuda.synchronize()
    cap = 4 * len(tc.layers) + 16
    acc = {}
    for _ in range(args.reps):
        lib.klay_profiler_begin()
        plan.forward(wd, code, dt, values=vals)
        plan.backward(vals, B, code, dt, workspace=work)
        kinds = (ctypes.c_int32 * cap)()
        layers = (ctypes.c_int32 * cap)()
        tms = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        lib.klay_profiler_end(cap, kinds, layers, tms, ctypes.byref(n))
        for i in range(n.value):
            acc.setdefault((kinds[i], layers[i]), []).append(tms[i])
    fwd_b, bwd_b = layer_bytes(tc, s, B, args.domain)
    peak, _ = load_peaks()
    widths = [tc.num_inputs] + [l.width for l in tc.layers]
    tot = {k: [0, 0] for k in range(8)}
    micro_l = min([l for (k, l) in acc if k == 6], default=len(tc.layers) + 1)
    microb_l = min([l for (k, l) in acc if k == 7], default=len(tc.layers) + 1)
    print(f"{'kind':>4} {'l':>3} {'op':>4} {'Wprev':>6} {'W':>6} {'E':>7} {'us':>9} {'GB/s':>8} {'frac':>6}")
    for (k, l), ts in sorted(acc.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        t = float(np.median(ts))
        b = fwd_b.get(l, 0) if k == 0 else (bwd_b.get(l, 0) if k == 1 else 0)
        tot[k][0] += t
        tot[k][1] += b
        if k in (0, 1):
            op = tc.layers[l - 1].op
            gbs = b / (t / 1e3) / 1e9
            print(f"{k:>4} {l:>3} {op:>4} {widths[l-1]:>6} {widths[l]:>6} "
                  f"{len(tc.layers[l-1].sources):>7} {t*1e3:>9.1f} {gbs:>8.0f} {gbs/peak:>6.3f}")
        elif k in (4, 5, 6, 7):
            top = micro_l if k == 4 else (microb_l if k == 5 else len(tc.layers) + 1)
            layers = range(l, top)
            b = sum((bwd_b if k in (5, 7) else fwd_b)[i] for i in layers)
            tot[k][1] += b
            gbs = b / (t / 1e3) / 1e9
            print(f"{k:>4} {l:>3} tail({len(layers)} layers) {t*1e3:>9.1f} us {gbs:>8.0f} GB/s")
        else:
            print(f"{k:>4} {l:>3} boundary {t*1e3:>9.1f} us")
    for k, name in ((0, "fwd"), (1, "bwd"), (2, "fwd-boundary"), (3, "bwd-boundary"),
                    (4, "fwd-tail"), (5, "bwd-tail"), (6, "fwd-micro-tail"), (7, "bwd-micro-tail")):
        t, b = tot[k]
        if t:
            print(f"{name}: {t:.3f} ms, {b/1e9:.3f} GB algorithmic, "
                  f"{b/(t/1e3)/1e9 if b else 0:.0f} GB/s")
    allms = sum(v[0] for v in tot.values())
    print(f"total kernel time {allms:.3f} ms per step (B={B})")


if __name__ == "__main__":
    main()
