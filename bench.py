"""Benchmark: circuit evaluations/s, forward+backward, log semiring.

Workload (BASELINE.json configs[2]): the 1,016,536-node
d-DNNF compiled from gen_3cnf(56, 128, seed 1) (data/circuits/C.npz), log
semiring fp32, 1024 batch rows per GPU (weak scaling), Philox(key=0) weights
p ~ U(0.05, 0.95) per literal. One step = forward (trace retained) +
backward (all-ones seed) over one batch; with N > 1 ranks each rank owns its
own 1024 rows and the root outputs are all-gathered over NCCL.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints ONE JSON line. `value` = device-timed evals/s with inputs
resident in HBM (CUDA events, max over ranks); `e2e` = the same metric
through the public API (engine.forward_log + engine.backward with host numpy
arrays; H2D of the weights and D2H of roots + grads inside the timed region);
`roofline` = the dominant kernel's algorithmic bytes / its event-timed
duration (per-launch CUDA events in a separate instrumented step);
`cpu_baseline` = the CPU oracle (numpy restatement of the reference engine)
on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "circuit evals/sec (fwd+bwd, log semiring) vs nodes; HBM roofline fraction"
CIRCUIT = os.path.join(ROOT, "data", "circuits", "C.npz")
WORKLOAD = "C: gen_3cnf(56,128,seed=1) -> compile_cnf -> layerize -> tensorize (1,016,536 nodes)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------

def _tail_from(tc):
    """First layer of libklay's persistent tail (klay.cu: longest suffix of
    layers with <= KLAY_TAIL_EDGES edges, at most 96 layers)."""
    lim = int(os.environ.get("KLAY_TAIL_EDGES", "256"))
    L = len(tc.layers)
    t = L
    while t > 0 and L - t < 96 and len(tc.layers[t - 1].sources) <= lim:
        t -= 1
    return t


def _micro_ok(tc, l, fwd):
    widths = [tc.num_inputs] + [x.width for x in tc.layers]
    wmax = 1280
    layer = tc.layers[l]
    W, Wp, E = widths[l + 1], widths[l], len(layer.sources)
    key = layer.segments if fwd else layer.sources
    fan = int(np.bincount(np.asarray(key), minlength=W if fwd else Wp).max())
    nodes = W if fwd else Wp
    return W <= wmax and Wp <= wmax and fan <= 129 and nodes + 1 + E <= 8192


def _micro_head(tc, fwd):
    """Layers in libklay's forward / backward micro head (klay.cu micro_head:
    the longest qualifying prefix of <= 256-node layers below every tail, at
    least two layers)."""
    lim = min(_micro_from(tc, fwd), _tail_from(tc))
    h = 0
    widths = [tc.num_inputs] + [x.width for x in tc.layers]
    while (h < lim and h < 64 and _micro_ok(tc, h, fwd)
           and widths[h + 1] <= 256 and widths[h] <= 256):
        h += 1
    return h if h >= 2 else 0


def _micro_from(tc, fwd):
    """First layer of libklay's forward / backward micro tail (klay.cu
    micro_suffix: longest suffix of <= 64 layers with widths <= 1280,
    fan-in / fan-out <= 129 and one layer's CSR <= 8192 ints; log semiring)."""
    L = len(tc.layers)
    m = L
    while m > 0 and L - m < 64 and _micro_ok(tc, m - 1, fwd):
        m -= 1
    return m


def _alias_bound(tc):
    """Nodes of layers >= this bound are never aliased (read by a tail)."""
    return min(_tail_from(tc), _micro_from(tc, True), _micro_from(tc, False))


_ALIAS_PLANS = {}


def alias_plan(tc):
    key = (id(tc), _alias_bound(tc))
    if key not in _ALIAS_PLANS:
        _ALIAS_PLANS[key] = _alias_plan(tc)
    return _ALIAS_PLANS[key]


def _alias_plan(tc):
    """Host restatement of libklay's unary-node aliases and adjoint routes
    (klay.cu build_aliases), for the byte model: per node layer, which nodes
    are aliased, their source row, and which adjoints are routed."""
    L = len(tc.layers)
    tail = _alias_bound(tc)
    hmax = max(_micro_head(tc, True), _micro_head(tc, False))
    lo = hmax + 2 if hmax else 1
    widths = [tc.num_inputs] + [l.width for l in tc.layers]
    rows = np.cumsum([0] + widths)
    child, npar, par, ali, srow = [], [], [], [], []
    for nl in range(L + 1):
        w = widths[nl]
        child.append(np.full(w, -1))
        npar.append(np.zeros(w, np.int64))
        par.append(np.full(w, -1))
        ali.append(np.zeros(w, bool))
        srow.append(rows[nl] + np.arange(w))
    for l, lay in enumerate(tc.layers):
        seg, src = np.asarray(lay.segments), np.asarray(lay.sources)
        fan = np.bincount(seg, minlength=lay.width)
        un = fan[seg] == 1
        child[l + 1][seg[un]] = src[un]
        npar[l] += np.bincount(src, minlength=widths[l])
        par[l][src] = seg
    is_sum = lambda nl: nl >= 1 and (nl - 1) % 2 == 1
    for nl in range(lo, min(L, tail)):
        m = child[nl] >= 0
        ali[nl] = m
        srow[nl][m] = srow[nl - 1][child[nl][m]]
    up = [np.where((npar[nl] == 1) & (par[nl] >= 0), par[nl], -1) for nl in range(L)]
    for nl in range(L):
        ok = up[nl] >= 0
        ok[ok] = ali[nl + 1][up[nl][ok]]
        up[nl] = np.where(ok, up[nl], -1)
    up.append(np.full(widths[L], -1))
    skip = [np.zeros(w, bool) for w in widths]
    top = [np.zeros(w, bool) for w in widths]
    masked_top = [np.zeros(w, bool) for w in widths]
    mask_src = [np.zeros(w, bool) for w in widths]
    for nl in range(L):
        for i in np.nonzero(up[nl] >= 0)[0]:
            if ali[nl][i] and up[nl - 1][child[nl][i]] == i:
                continue
            tl, t, masked, path = nl, i, False, [(nl, i)]
            while up[tl][t] >= 0:
                t = up[tl][t]
                tl += 1
                masked |= is_sum(tl)
                path.append((tl, t))
            if masked and (ali[nl][i] or nl == 0):
                continue
            for a, b in path[:-1]:
                skip[a][b] = True
            top[tl][t] = True
            masked_top[tl][t] = masked
            mask_src[nl][i] = masked
    return dict(widths=widths, ali=ali, srow=srow, skip=skip, masked_top=masked_top,
                mask_src=mask_src, tail=tail)


def survey_layer_bytes(tc, s, B, domain="log"):
    """SURVEY §8(d)'s algorithmic bytes per launch (the contract's figure):
      fwd_l = s*B*(W_{l-1} + W_l) + 4*(E_l + W_l + 1)
      bwd_l = c_l*s*B*(W_{l-1} + W_l) + 4*(2E_l + W_{l-1} + 1), c_l = 2 for
        log-sum and real-product layers (they read N_l and N_{l-1} besides
        the adjoints), 1 for pass-through layers.
    20.359 MB per evaluation at config C in fp32 (roofline 317.6 k evals/s)."""
    fwd, bwd = {}, {}
    prev = tc.num_inputs
    for l, layer in enumerate(tc.layers, start=1):
        W, E = layer.width, len(layer.sources)
        heavy = (layer.op != "prod") if domain == "log" else (layer.op == "prod")
        c = 2 if heavy else 1
        fwd[l] = s * B * (prev + W) + 4 * (E + W + 1)
        bwd[l] = c * s * B * (prev + W) + 4 * (2 * E + prev + 1)
        prev = W
    return fwd, bwd


def layer_bytes(tc, s, B, domain="log", alias=None):
    """Per-launch algorithmic bytes of every forward and backward layer kernel
    (rows of s*B bytes; index bytes at 4 per entry).

    Plain dataflow (reference order):
      fwd_l = rows(W_{l-1} + W_l) + 4*(E_l + W_l + 1)
      bwd_l = rows(2*W_{l-1} + W_l + P_l) + 4*(2E_l + W_{l-1} + 1): parent
        adjoints (W_l) in, child values (W_{l-1}) in, child adjoints out,
        plus P_l parent values: 0 for pass-through layers, W_l for real
        products, the non-unary parents for log sums (epsilon 0).
    With unary-node aliases and adjoint routes (log, epsilon 0,
    backward-only trace; klay.cu build_aliases, restated in alias_plan):
      fwd_l = rows(distinct operand rows of the computed nodes + computed
        nodes) + masks (s*B/32 bytes per route bottom) + indices
      bwd_l = rows(distinct parents of the computed children (adjoints)
        + their non-unary parents (values, log sums) + distinct own-value
        rows (log sums) + computed children) + masks of masked route tops
        (pass-through layers) + indices
    """
    if alias is None:
        alias = domain == "log"
    row = s * B
    mask = s * B / 32.0
    fwd, bwd = {}, {}
    ap = alias_plan(tc) if alias else None
    prev = tc.num_inputs
    for l, layer in enumerate(tc.layers, start=1):
        i = l - 1
        W, E = layer.width, len(layer.sources)
        seg, src = np.asarray(layer.segments), np.asarray(layer.sources)
        fan = np.bincount(seg, minlength=W)
        if ap is None:
            fwd[l] = row * (prev + W) + 4 * (E + W + 1)
            if domain == "log" and layer.op != "prod":
                P = int((fan > 1).sum())
                bwd[l] = row * (2 * prev + W + P) + 4 * (2 * E + prev + 1)
            elif domain != "log" and layer.op == "prod":
                bwd[l] = 2 * row * (prev + W) + 4 * (2 * E + prev + 1)
            else:
                bwd[l] = row * (prev + W) + 4 * (2 * E + prev + 1)
            prev = W
            continue
        ali_n, ali_c = ap["ali"][l], ap["ali"][i]
        src_rows = ap["srow"][i][src]
        comp = ~ali_n[seg]                      # edges of computed nodes
        n_comp = int((~ali_n).sum())
        fwd[l] = (row * (np.unique(src_rows[comp]).size + n_comp)
                  + mask * int(ap["mask_src"][l].sum()) + 4 * (int(comp.sum()) + 2 * n_comp + 1))
        kept = ~ap["skip"][i]
        ke = kept[src]                          # edges of computed children
        n_kept = int(kept.sum())
        adj = np.unique(seg[ke]).size
        if layer.op == "prod":
            bwd[l] = (row * (adj + n_kept) + mask * int(ap["masked_top"][i].sum())
                      + 4 * (2 * int(ke.sum()) + 2 * n_kept + 1))
        else:
            nonun = ke & (fan[seg] > 1)
            bwd[l] = (row * (adj + np.unique(seg[nonun]).size
                             + np.unique(ap["srow"][i][kept]).size + n_kept)
                      + 4 * (2 * int(ke.sum()) + 3 * n_kept + 1))
        prev = W
    return fwd, bwd


def bytes_per_eval(tc, s, B, alias=None, survey=False):
    fwd, bwd = survey_layer_bytes(tc, s, B) if survey else layer_bytes(tc, s, B, alias=alias)
    return (sum(fwd.values()) + sum(bwd.values())) / B


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU oracle timing (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------

_W_TC = None


def _worker_init(path):
    global _W_TC
    from paper_2410_11415_b200.tensorized import load_npz
    from oracle import engine_port as oracle
    _W_TC = load_npz(path)
    oracle.plans(_W_TC)


def _worker_run(args):
    """One bounded chunk: fwd (fp32, log, trace) + bwd on `rows` rows."""
    from oracle import engine_port as oracle
    seed, rows = args
    rng = np.random.Generator(np.random.Philox(key=seed))
    w = np.log(rng.uniform(0.05, 0.95, size=(rows, _W_TC.num_inputs))).astype(np.float32)
    t0 = time.perf_counter()
    _, tr = oracle.forward(_W_TC, w, "log")
    oracle.backward(_W_TC, tr, "log")
    return rows, time.perf_counter() - t0


def cpu_pool_size(per_worker_gb=1.0):
    n = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available / 2 ** 30
        n = max(1, min(n, int(avail * 0.6 / per_worker_gb)))
    except Exception:
        pass
    return max(1, min(n, 64))


class CpuOracle:
    """A fork pool of oracle workers, each evaluating independent row chunks
    (the reference engine is single-threaded numpy; rows are independent,
    so P processes is the best CPU arrangement)."""

    def __init__(self, path, rows_per_task=16):
        import multiprocessing as mp
        self.procs = cpu_pool_size()
        self.rows = rows_per_task
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(self.procs, initializer=_worker_init, initargs=(path,))
        self.pool.map(_worker_run, [(i, 1) for i in range(self.procs)])  # warm plans

    def step(self, tasks_per_proc=1, seed0=0):
        tasks = [(seed0 + i, self.rows) for i in range(self.procs * tasks_per_proc)]
        t0 = time.perf_counter()
        res = self.pool.map(_worker_run, tasks, chunksize=1)
        wall = time.perf_counter() - t0
        return sum(r for r, _ in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # rank 0 alone runs the CPU reference
    from paper_2410_11415_b200.tensorized import load_npz
    tc = load_npz(CIRCUIT)
    cpu = CpuOracle(CIRCUIT)
    for i in range(args.warmup):
        cpu.step(seed0=1000 * i)
    rows = 0
    wall = 0.0
    for i in range(args.steps):
        r, t = cpu.step(seed0=10_000 + 1000 * i)
        rows += r
        wall += t
    cpu.close()
    value = rows / wall
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": nodes,
                   "edges": int(sum(len(l.sources) for l in tc.layers)),
                   "semiring": "log", "pass": "fwd+bwd",
                   "rows_per_step": cpu.procs * cpu.rows},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cpu.procs, "kind": "port",
                         "sample": f"{cpu.procs} processes x {cpu.rows} rows per step, "
                                   "oracle/engine_port.py (numpy restatement of "
                                   "laycirc/engine.py), fp32 log fwd+bwd"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def measure_config(name, semiring, dtype, B, with_backward, dev, iters=20):
    """Device-timed evals/s of another BASELINE config (inputs in HBM)."""
    import torch
    from paper_2410_11415_b200 import _lib, engine
    from paper_2410_11415_b200.tensorized import load_npz

    tc = load_npz(os.path.join(ROOT, "data", "circuits", f"{name}.npz"))
    plan = engine.device_plan(tc, dev)
    code = {"real": _lib.KLAY_REAL, "log": _lib.KLAY_LOG, "bool": _lib.KLAY_BOOL,
            "bool_packed": _lib.KLAY_BOOL}[semiring]
    rng = np.random.Generator(np.random.Philox(key=1))
    if semiring.startswith("bool"):
        w = rng.integers(0, 2, size=(B, tc.num_inputs)).astype(np.float64)
    else:
        w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
        if semiring == "log":
            w = np.log(w)
    wd = torch.from_numpy(w.astype(np.float32 if dtype == "u1" else dtype)).to(dev)
    vals = plan.alloc_values(B, dtype, retain=with_backward)
    fw = plan.forward_workspace(B, dtype)
    work = plan.workspace(B, dtype) if with_backward else None

    def step():
        plan.forward(wd, code, dtype, retain=with_backward, values=vals, workspace=fw)
        if with_backward:
            plan.backward(vals, B, code, dtype, workspace=work)

    for _ in range(3):
        step()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(iters):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / iters
    s = 8 if dtype == np.float64 else (1 / 8 if dtype == "u1" else 4)
    dom = semiring if semiring in ("log", "real") else "log"
    fwd_b, bwd_b = survey_layer_bytes(tc, s, B, dom)
    alg = sum(fwd_b.values()) + (sum(bwd_b.values()) if with_backward else 0)
    fwd_n, bwd_n = layer_bytes(tc, s, B, dom, alias=(semiring == "log" and with_backward))
    nec = sum(fwd_n.values()) + (sum(bwd_n.values()) if with_backward else 0)
    peak, _ = load_peaks()
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    return {"nodes": nodes, "semiring": semiring,
            "dtype": {8: "f64", 4: "f32"}.get(s, "u1 (bit-packed)"), "batch": B,
            "pass": "fwd+bwd" if with_backward else "fwd", "ms_per_batch": ms,
            "evals_per_s": B / (ms / 1e3), "roofline_frac": alg / (ms / 1e3) / 1e9 / peak,
            "frac_necessary": nec / (ms / 1e3) / 1e9 / peak}


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    from paper_2410_11415_b200 import engine, _lib
    from paper_2410_11415_b200.tensorized import load_npz

    tc = load_npz(CIRCUIT)
    B = args.batch
    s = 4  # fp32
    dt = np.float32

    # CPU baseline first (rank 0, N = 1 only), before CUDA is initialised,
    # so the fork pool never inherits a CUDA context.
    cpu_line = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = CpuOracle(CIRCUIT)
        cpu.step(seed0=77)
        rows = wall = 0
        t_end = time.perf_counter() + args.cpu_seconds
        i = 0
        while time.perf_counter() < t_end or i == 0:
            r, t = cpu.step(seed0=100 + 1000 * i)
            rows += r
            wall += t
            i += 1
        cpu.close()
        cpu_line = {"value": rows / wall, "unit": "evals/s", "cores": cpu.procs, "kind": "port",
                    "sample": f"{rows} rows of config C in {wall:.1f} s ({cpu.procs} processes x "
                              f"{cpu.rows}-row chunks), oracle/engine_port.py, fp32 log fwd+bwd"}

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    plan = engine.device_plan(tc, dev)

    rng = np.random.Generator(np.random.Philox(key=0))
    w_all = np.log(rng.uniform(0.05, 0.95, size=(B * world, tc.num_inputs)))
    w_host = w_all[rank * B:(rank + 1) * B]
    w_dev = torch.from_numpy(w_host.astype(np.float32)).to(dev)
    values = plan.alloc_values(B, dt, retain=True)
    outputs = torch.empty((B, tc.num_roots), dtype=torch.float32, device=dev)
    grads = torch.empty((B, tc.num_inputs), dtype=torch.float32, device=dev)
    work = plan.workspace(B, dt)
    gathered = [torch.empty_like(outputs) for _ in range(world)] if world > 1 else None
    launches_per_step = None

    # the timed step replays one CUDA graph holding the whole fwd + bwd
    # (~100 kernels for config C); the instrumented step below launches them
    # one by one on the stream to time each
    cap = plan.capture(B, dt, _lib.KLAY_LOG, backward=True)
    cap.weights.copy_(w_dev)

    def step():
        cap.replay()
        if world > 1:
            dist.all_gather(gathered, cap.outputs)

    stream = torch.cuda.current_stream(dev)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # kernels per step (a graph replay launches the captured kernels; count
    # them on one stream-launched step)
    n_a = lib.klay_launch_count()
    plan.forward(w_dev, _lib.KLAY_LOG, dt, retain=True, values=values, outputs=outputs)
    plan.backward(values, B, _lib.KLAY_LOG, dt, grads=grads, workspace=work)
    launches_per_step = lib.klay_launch_count() - n_a
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    launches = launches_per_step * args.steps
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    ms_per_step = ms / args.steps
    value = world * B / (ms_per_step / 1e3)

    # ---- per-launch timing of one instrumented step (roofline) ----------
    lib.klay_profiler_begin()
    plan.forward(w_dev, _lib.KLAY_LOG, dt, retain=True, values=values, outputs=outputs)
    plan.backward(values, B, _lib.KLAY_LOG, dt, grads=grads, workspace=work)
    import ctypes
    nslots = 4 * len(tc.layers) + 16
    kinds = (ctypes.c_int32 * nslots)()
    layers = (ctypes.c_int32 * nslots)()
    tms = (ctypes.c_float * nslots)()
    nrec = ctypes.c_int32()
    lib.klay_profiler_end(nslots, kinds, layers, tms, ctypes.byref(nrec))
    # the contract's figure and the bytes the implemented
    # dataflow must move (unary-node aliases and routes skip rows)
    fwd_b, bwd_b = survey_layer_bytes(tc, s, B)
    fwd_n, bwd_n = layer_bytes(tc, s, B)
    per_kind = {0: [0.0, 0.0, 0, 0.0], 1: [0.0, 0.0, 0, 0.0]}
    other_ms = 0.0
    for i in range(min(nrec.value, nslots)):
        k, l, t = kinds[i], layers[i], tms[i]
        if k in (0, 1):
            per_kind[k][0] += t
            per_kind[k][1] += (fwd_b if k == 0 else bwd_b)[l]
            per_kind[k][2] += 1
            per_kind[k][3] += (fwd_n if k == 0 else bwd_n)[l]
        else:
            other_ms += t
    peak, peak_kind = load_peaks()
    dom = max(per_kind, key=lambda k: per_kind[k][0])
    dom_name = ["fwd_layer_kernel", "bwd_layer_kernel"][dom]
    traffic = None
    try:  # DRAM bytes of the same launches, from the committed ncu launch list
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh).get(dom_name)
    except Exception:
        pass
    dms, dbytes, dn, dnec = per_kind[dom]
    achieved = dbytes / (dms / 1e3) / 1e9
    achieved_nec = dnec / (dms / 1e3) / 1e9
    bpe = bytes_per_eval(tc, s, B, survey=True)
    bpe_nec = bytes_per_eval(tc, s, B)

    # ---- e2e: public API with host buffers ------------------------------
    e2e = None
    if not args.no_e2e:
        W = engine.WeightAssignment(w_host, "log")
        for _ in range(2):
            engine.gradient(tc, W, log_domain=True, dtype=np.float32)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        n_e2e = max(3, min(args.steps, 20))
        for _ in range(n_e2e):
            out, g = engine.gradient(tc, W, log_domain=True, dtype=np.float32)
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
        engine.clear_cache()
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": world * B * n_e2e / el, "unit": "evals/s",
               "h2d_bytes_per_step": int(w_host.size * 4),
               "d2h_bytes_per_step": int(out.nbytes + g.nbytes),
               "api": "engine.gradient(log_domain=True, dtype=float32): numpy in/out; one "
                      "CUDA graph per call holding the pinned H2D copy, fwd, bwd and D2H copies"}

    extra = None
    if world == 1 and not args.no_extra:
        # the other BASELINE configs, device-timed (parity cases; not the headline)
        extra = {
            "A_real_f64_b1_fwd": measure_config("A", "real", np.float64, 1, False, dev),
            "B_log_f64_b256_fwd_bwd": measure_config("B", "log", np.float64, 256, True, dev),
            "B_real_f64_b256_fwd_bwd": measure_config("B", "real", np.float64, 256, True, dev),
            "D_bool_b4096_fwd": measure_config("D", "bool", np.float32, 4096, False, dev),
            "D_bool_packed_b4096_fwd": measure_config("D", "bool_packed", "u1", 4096, False, dev),
            "D_real_f32_b4096_fwd": measure_config("D", "real", np.float32, 4096, False, dev),
            "E_log_f64_b128_fwd_bwd": measure_config("E", "log", np.float64, 128, True, dev),
            "Cp_log_f32_b1024_fwd_bwd": measure_config("Cp", "log", np.float32, 1024, True, dev, iters=5),
        }

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": nodes,
                   "edges": int(sum(len(l.sources) for l in tc.layers)),
                   "gate_layers": len(tc.layers), "semiring": "log", "pass": "fwd+bwd",
                   "batch_per_gpu": B, "global_batch": B * world,
                   "parallelism": f"dp{world} (batch-sharded, plan replicated)",
                   "l2": f"no flush: per-step working set {nodes * B * s / 1e9:.2f} GB trace "
                         ">> 126 MB L2",
                   "bytes_per_eval": bpe,
                   "bytes_model": "SURVEY §8(d) (reference dataflow: every layer read and "
                                  "written, c_l = 2 for log-sum layers)",
                   "step_roofline_frac": value / world * bpe / (peak * 1e9),
                   "bytes_per_eval_necessary": bpe_nec,
                   "step_frac_necessary": value / world * bpe_nec / (peak * 1e9),
                   "necessary_model": "bytes the implemented dataflow must move: unary-node "
                                      "aliases and adjoint routes skip rows (bench.py "
                                      "layer_bytes / alias_plan)"},
        "roofline": {"bound": "hbm", "kernel": dom_name,
                     "launches_per_step": dn, "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "alg_bytes_per_step": dbytes,
                     "alg_model": "SURVEY §8(d) per-layer bytes x launches",
                     "necessary": {"alg_bytes_per_step": dnec, "achieved": achieved_nec,
                                   "frac": achieved_nec / peak},
                     "traffic": traffic,
                     "traffic_scope": "DRAM read+write bytes per step of the same launches "
                                      "(ncu launch list, profiles/traffic.json)",
                     "kernel_ms_per_step": dms,
                     "fwd_ms": per_kind[0][0], "bwd_ms": per_kind[1][0],
                     "boundary_ms": other_ms},
        "gpu_launches": int(launches),
        "launch_mode": "CUDA graph replay of the captured fwd+bwd "
                       f"({launches_per_step} libklay kernels per step)",
        "clocks": clk,
        "cpu_baseline": cpu_line,
        "e2e": e2e,
        "extra_configs": extra,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1024, help="rows per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other-config measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
