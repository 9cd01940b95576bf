"""Benchmark: circuit evaluations/s, forward+backward, log semiring.

Workload (BASELINE.json configs[2]): the 1,016,536-node
d-DNNF compiled from gen_3cnf(56, 128, seed 1) (data/circuits/C.npz), log
semiring fp32, global batch 1024 sharded over the N GPUs (strong scaling, the
north star's "batch 1024 at 1/2/4/8 B200"; `--scaling weak` gives every GPU
its own 1024 rows), Philox(key=0) weights p ~ U(0.05, 0.95) per literal. One
step = forward (trace retained) + backward (all-ones seed) of this rank's rows
as one CUDA-graph replay, then NCCL all-gathers of the outputs [B, R] and the
input gradients [B, K] (distributed.ShardedPass).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` outside torchrun re-launches itself as N ranks. Rank 0 prints ONE
JSON line. `value` = device-timed evals/s with inputs resident in HBM (CUDA
events, max over ranks); `e2e` = the same metric through the public API
(engine.gradient with host numpy arrays on each rank's rows, gathered);
`roofline` = per launch class (template) the bytes the implemented dataflow
must move over its in-graph time (time_classes), the dominant class on top;
`cpu_baseline` = the CPU oracle (numpy restatement of the reference engine)
on this host's cores, with the single-process figure beside it.
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
# per-template (launch class) byte model and in-graph timing
# ---------------------------------------------------------------------------

# launch classes of libklay (include/klay.h KLAY_CLASS_*)
CLASS_NAMES = ["fwd_prod", "fwd_sum", "bwd_pass", "bwd_logsum", "bwd_realprod",
               "fwd_micro", "bwd_micro", "tail", "boundary"]


def kernel_class(name, domain="log"):
    """Launch class of an ncu kernel name (log semiring: product layers
    reduce with RK_SUM = 0, sum layers with RK_LSE = 4)."""
    n = name.replace("void ", "")
    if n.startswith(("items_kernel", "combine_kernel")):
        args = n[n.index("<") + 1:].split(",")
        if "BwdGather" in n:
            mode = int(n.split("BwdGather<")[1].split(",")[1].split(">")[0])
            return {0: "bwd_pass", 3: "bwd_pass", 1: "bwd_logsum", 4: "bwd_logsum",
                    2: "bwd_realprod"}[mode]
        rk = int(args[1])
        if domain == "log":
            return "fwd_prod" if rk == 0 else "fwd_sum"
        return "fwd_prod" if rk == 1 else "fwd_sum"
    if n.startswith("micro_bwd_kernel"):
        return "bwd_micro"
    if n.startswith("micro_kernel"):
        return "fwd_micro"
    if n.startswith("tail_kernel"):
        return "tail"
    return "boundary"


def schedule(plan, B, s):
    """Which gate layers (0-based) run in which launch class at batch B
    (klay.cu forward_impl / backward_impl; micro tails and heads only when
    their grid fits two waves, klay.cu micro_fits)."""
    import torch
    L = plan.num_layers
    ld = plan.row_stride(B, np.float64 if s == 8 else np.float32)
    V = ld * s // 16
    sms = torch.cuda.get_device_properties(plan.device).multi_processor_count
    ok = (V + 1) // 2 <= 2 * sms
    sc = plan.schedule
    micro = sc["micro"] if ok else L
    microb = sc["micro_bwd"] if ok else L
    head = sc["head"] if ok else 0
    headb = sc["head_bwd"] if ok else 0
    tail = sc["tail"]
    fwd = {}
    for l in range(L):
        fwd[l] = ("fwd_micro" if (l < head or l >= micro) else
                  "tail" if l >= tail else None)
    bwd = {}
    for l in range(L):
        bwd[l] = ("bwd_micro" if (l < headb or l >= microb) else
                  "tail" if l >= tail else None)
    return fwd, bwd, dict(micro=micro, microb=microb, head=head, headb=headb, tail=tail)


def class_bytes(tc, plan, B, s):
    """Per launch class: (necessary bytes per step, SURVEY-model bytes per
    step, layer list). Layer kernels use layer_bytes / survey_layer_bytes;
    the micro tails and heads move their first layer's input rows, every
    stored output row and their CSR (forward), or the top adjoints, the
    weighted (log-sum) layers' value rows, the lowest adjoints and the CSR
    (backward); boundary kernels the [B,K] / [B,R] host-layout tensors."""
    fwd_n, bwd_n = layer_bytes(tc, s, B)
    fwd_s, bwd_s = survey_layer_bytes(tc, s, B)
    fcls, bcls, sc = schedule(plan, B, s)
    row = s * B
    widths = [tc.num_inputs] + [l.width for l in tc.layers]
    nec = {c: 0.0 for c in CLASS_NAMES}
    sur = {c: 0.0 for c in CLASS_NAMES}
    layers = {c: [] for c in CLASS_NAMES}
    micro_f, micro_b = [], []
    for l, layer in enumerate(tc.layers):
        E = len(layer.sources)
        c = fcls[l] or ("fwd_prod" if layer.op == "prod" else "fwd_sum")
        layers[c].append(l)
        sur[c] += fwd_s[l + 1]
        if c == "fwd_micro":
            micro_f.append(l)
            nec[c] += row * widths[l + 1] + 4 * (widths[l + 1] + 1 + E)
        else:
            nec[c] += fwd_n[l + 1]
        c = bcls[l] or ("bwd_pass" if layer.op == "prod" else "bwd_logsum")
        layers[c].append(l)
        sur[c] += bwd_s[l + 1]
        if c == "bwd_micro":
            micro_b.append(l)
            weighted = layer.op != "prod"
            nec[c] += (row * (widths[l + 1] + widths[l]) if weighted else 0) \
                + 4 * (widths[l] + 1 + E)
        else:
            nec[c] += bwd_n[l + 1]
    # input rows of each forward micro launch, output adjoints of each backward one
    for lo in (0, sc["micro"]):
        if lo in micro_f:
            nec["fwd_micro"] += row * widths[lo]
    for top, low in ((sc["headb"] - 1, 0), (len(tc.layers) - 1, sc["microb"])):
        if top in micro_b:
            nec["bwd_micro"] += row * (widths[top + 1] + widths[low])
    K, R = tc.num_inputs, tc.num_roots
    nec["boundary"] = sur["boundary"] = 2 * row * (K + R) + row * widths[-1]
    return nec, sur, layers


def time_classes(lib, run_step, iters=20):
    """In-graph device time per launch class: one CUDA graph per class
    holding only that class's launches of a full step (klay_set_launch_filter),
    replayed `iters` times between CUDA events. Work is data-independent in
    the log semiring, so a class times the same as inside the full graph
    (up to its neighbours' overlap through programmatic dependent launch)."""
    import torch
    out = {}
    for c, name in enumerate(CLASS_NAMES):
        prev = lib.klay_set_launch_filter(1 << c)
        n0 = lib.klay_launch_count()
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):
                run_step()
        finally:
            lib.klay_set_launch_filter(prev)
        n = lib.klay_launch_count() - n0
        if n == 0:
            continue
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"launches": int(n), "ms": e0.elapsed_time(e1) / iters}
        del g
    return out


def ncu_class_traffic(path, domain="log"):
    """Per launch class from a committed ncu launch list (profiles/):
    DRAM read+write bytes and device time per step, launches per step."""
    import csv
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    try:
        hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    except IndexError:
        return None
    h = rows[hi]
    ik, im, iu, iv = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit",
                                           "Metric Value"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
             "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    per = {}
    ids = {}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        c = kernel_class(r[ik], domain)
        d = per.setdefault(c, {"dram_bytes": 0.0, "ms": 0.0})
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
        if r[im].startswith("dram__bytes"):
            d["dram_bytes"] += v
        elif r[im] == "gpu__time_duration.sum":
            d["ms"] += v * 1e3
        ids.setdefault(c, set()).add(r[0])
    steps = 1
    meta = path[:-4] + ".json"
    if os.path.exists(meta):
        with open(meta) as fh:
            steps = json.load(fh).get("steps", 1)
    return {c: {"dram_bytes": d["dram_bytes"] / steps, "ms": d["ms"] / steps,
                "launches": len(ids[c]) // steps} for c, d in per.items()}


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


def cpu_pool_size(per_worker_gb=1.5):
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

    def step(self, rows, seed0=0):
        """`rows` rows split into one task per process (the last ones
        shorter); returns (rows, wall seconds)."""
        per = -(-rows // self.procs)
        tasks = []
        left = rows
        i = 0
        while left > 0:
            tasks.append((seed0 + i, min(per, left)))
            left -= per
            i += 1
        t0 = time.perf_counter()
        res = self.pool.map(_worker_run, tasks, chunksize=1)
        wall = time.perf_counter() - t0
        return sum(r for r, _ in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def single_process_cpu(seconds, rows=64):
    """The reference's own arrangement (bench.py:177-183 of the reference:
    one process, single-threaded numpy): evals/s of the oracle port in this
    process on `rows`-row chunks for about `seconds`."""
    _worker_init(CIRCUIT)
    _worker_run((5, 1))
    done = wall = 0.0
    i = 0
    while wall < seconds or i == 0:
        r, t = _worker_run((500 + i, rows))
        done += r
        wall += t
        i += 1
    return {"value": done / wall, "unit": "evals/s", "cores": 1, "kind": "port",
            "sample": f"{int(done)} rows of config C in {wall:.1f} s, one process, "
                      f"{rows}-row chunks, oracle/engine_port.py, fp32 log fwd+bwd"}


def run_reference_arm(args):
    """The reference's CPU engine (oracle port, same ufunc sequence as
    laycirc/engine.py) on the GPU arm's workload: each step is the same
    1024-row config C fwd+bwd, split over one process per core."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # rank 0 alone runs the CPU reference
    from paper_2410_11415_b200.tensorized import load_npz
    tc = load_npz(CIRCUIT)
    single = single_process_cpu(args.cpu_single_seconds)
    cpu = CpuOracle(CIRCUIT)
    for i in range(args.warmup):
        cpu.step(cpu.procs, seed0=1000 * i)  # untimed warm-up: one row per process
    rows = 0
    wall = 0.0
    for i in range(args.steps):
        r, t = cpu.step(args.batch, seed0=10_000 + 1000 * i)
        rows += r
        wall += t
    cpu.close()
    value = rows / wall
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": nodes,
                   "edges": int(sum(len(l.sources) for l in tc.layers)),
                   "semiring": "log", "pass": "fwd+bwd", "global_batch": args.batch,
                   "rows_per_step": args.batch,
                   "warmup_rows": f"{cpu.procs} (one per process: warms the plans)"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cpu.procs, "kind": "port",
                         "sample": f"{args.steps} steps x {args.batch} rows ({cpu.procs} "
                                   "processes, one chunk each), oracle/engine_port.py (numpy "
                                   "restatement of laycirc/engine.py), fp32 log fwd+bwd",
                         "single_process": single},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _timed_replays(fn, n, dev):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / n


def measure_config(name, semiring, dtype, B, with_backward, dev, iters=20):
    """Device-timed evals/s of another BASELINE config (inputs in HBM; one
    CUDA-graph replay per batch, like the headline)."""
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

    for _ in range(2):
        step()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream(dev).wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    ms = _timed_replays(g.replay, iters, dev)
    s = 8 if dtype == np.float64 else (1 / 8 if dtype == "u1" else 4)
    dom = semiring if semiring in ("log", "real") else "log"
    fwd_b, bwd_b = survey_layer_bytes(tc, s, B, dom)
    alg = sum(fwd_b.values()) + (sum(bwd_b.values()) if with_backward else 0)
    fwd_n, bwd_n = layer_bytes(tc, s, B, dom, alias=(semiring == "log" and with_backward))
    nec = sum(fwd_n.values()) + (sum(bwd_n.values()) if with_backward else 0)
    peak, _ = load_peaks()
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    del g
    return {"nodes": nodes, "semiring": semiring,
            "dtype": {8: "f64", 4: "f32"}.get(s, "u1 (bit-packed)"), "batch": B,
            "pass": "fwd+bwd" if with_backward else "fwd", "ms_per_batch": ms,
            "evals_per_s": B / (ms / 1e3), "contract_frac": alg / (ms / 1e3) / 1e9 / peak,
            "frac_necessary": nec / (ms / 1e3) / 1e9 / peak}


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch this script as N
    ranks (torch.distributed.run, 127.0.0.1); rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)",
              file=sys.stderr)
    from paper_2410_11415_b200 import _lib, engine
    from paper_2410_11415_b200.distributed import ShardedPass, sharded_eval
    from paper_2410_11415_b200.tensorized import load_npz

    tc = load_npz(CIRCUIT)
    s = 4  # fp32
    dt = np.float32
    strong = args.scaling == "strong"
    B_global = args.batch if strong else args.batch * world

    # CPU baselines first (rank 0, N = 1 only), before CUDA is initialised,
    # so the fork pool never inherits a CUDA context.
    cpu_line = None
    if world == 1 and not args.no_cpu_baseline:
        single = single_process_cpu(args.cpu_single_seconds)
        cpu = CpuOracle(CIRCUIT)
        rows = wall = 0
        t_end = time.perf_counter() + args.cpu_seconds
        i = 0
        while time.perf_counter() < t_end or i == 0:
            r, t = cpu.step(cpu.procs * cpu.rows, seed0=100 + 1000 * i)
            rows += r
            wall += t
            i += 1
        cpu.close()
        cpu_line = {"value": rows / wall, "unit": "evals/s", "cores": cpu.procs, "kind": "port",
                    "sample": f"{rows} rows of config C in {wall:.1f} s ({cpu.procs} processes x "
                              f"{cpu.rows}-row chunks), oracle/engine_port.py, fp32 log fwd+bwd",
                    "single_process": single}

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()

    rng = np.random.Generator(np.random.Philox(key=0))
    w_all = np.log(rng.uniform(0.05, 0.95, size=(B_global, tc.num_inputs)))

    # one step: a CUDA-graph replay of this rank's forward + backward
    # (~100 kernels for config C), then NCCL all-gathers of the outputs
    # [B, R] and input gradients [B, K] into every rank's device buffers
    sp = ShardedPass(tc, B_global, dt, _lib.KLAY_LOG, world, rank, device=dev)
    B = sp.local_batch
    w_host = w_all[sp.lo:sp.hi]
    sp.weights.copy_(torch.from_numpy(w_host.astype(np.float32)))
    plan = sp.plan

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        sp.step()
    torch.cuda.synchronize(dev)
    # kernels per step: count one stream-launched step (a replay launches
    # the same captured kernels)
    cap = sp.cap
    n_a = lib.klay_launch_count()
    plan.forward(cap.weights, _lib.KLAY_LOG, dt, retain=True, values=cap.values,
                 outputs=cap.outputs, workspace=cap._fw)
    plan.backward(cap.values, B, _lib.KLAY_LOG, dt, grads=cap.grads, workspace=cap._bw)
    launches_per_step = lib.klay_launch_count() - n_a
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev)
    ev0.record(stream)
    for _ in range(args.steps):
        sp.step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    ms_per_step = ms / args.steps
    value = B_global / (ms_per_step / 1e3)

    # ---- sustained: the same step replayed for >= args.sustain seconds ---
    sustained = None
    if args.sustain > 0:
        n_sus = max(args.steps, int(args.sustain * 1e3 / ms_per_step) + 1)
        cs = ClockSampler(local)
        cs.start()
        if world > 1:
            dist.barrier()
        ms_s = _timed_replays(sp.step, n_sus, dev) * n_sus
        if world > 1:
            t = torch.tensor([ms_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_s = float(t.item())
        sustained = {"steps": n_sus, "seconds": ms_s / 1e3,
                     "value": B_global * n_sus / (ms_s / 1e3), "ms_per_step": ms_s / n_sus,
                     "clocks": cs.stop()}

    # ---- per-template roofline: in-graph time of each launch class -------
    def full_step():
        plan.forward(cap.weights, _lib.KLAY_LOG, dt, retain=True, values=cap.values,
                     outputs=cap.outputs, workspace=cap._fw)
        plan.backward(cap.values, B, _lib.KLAY_LOG, dt, grads=cap.grads, workspace=cap._bw)

    ctimes = time_classes(lib, full_step, iters=max(10, min(args.steps, 50)))
    nec_b, sur_b, cls_layers = class_bytes(tc, plan, B, s)
    peak, peak_kind = load_peaks()
    ncu = ncu_class_traffic(os.path.join(ROOT, "profiles", args.launch_list))
    templates = {}
    for c, t in ctimes.items():
        sec = t["ms"] / 1e3
        row = {"launches": t["launches"], "layers": len(cls_layers[c]), "ms": t["ms"],
               "necessary_bytes": nec_b[c], "contract_bytes": sur_b[c],
               "achieved_gbs": nec_b[c] / sec / 1e9, "frac": nec_b[c] / sec / 1e9 / peak,
               "contract_frac": sur_b[c] / sec / 1e9 / peak}
        if ncu and c in ncu:
            row["ncu_dram_bytes"] = ncu[c]["dram_bytes"]
            row["ncu_ms"] = ncu[c]["ms"]
            row["ncu_frac"] = (nec_b[c] / (ncu[c]["ms"] / 1e3) / 1e9 / peak
                               if ncu[c]["ms"] else None)
        templates[c] = row
    dom = max(templates, key=lambda c: templates[c]["ms"])
    dt_ = templates[dom]
    nl = dt_["launches"]
    bpe = bytes_per_eval(tc, s, B, survey=True)
    bpe_nec = sum(nec_b.values()) / B

    # ---- e2e: public API with host buffers ------------------------------
    e2e = None
    if not args.no_e2e:
        def api(rows):
            return engine.gradient(tc, engine.WeightAssignment(rows, "log"), log_domain=True,
                                   dtype=np.float32)
        for _ in range(2):
            sharded_eval(api, w_all, world, rank)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        n_e2e = max(3, min(args.steps, 20))
        for _ in range(n_e2e):
            out, g = sharded_eval(api, w_all, world, rank)
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
        engine.clear_cache()
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": B_global * n_e2e / el, "unit": "evals/s",
               "h2d_bytes_per_step": int(w_host.size * 4),
               "d2h_bytes_per_step": int(B * (tc.num_roots + tc.num_inputs) * 4),
               "api": "engine.gradient(log_domain=True, dtype=float32) on this rank's rows: "
                      "numpy in/out, one CUDA graph per call holding the pinned H2D copy, fwd, "
                      "bwd and D2H copies" + ("; outputs + grads all-gathered "
                                              "(distributed.sharded_eval)" if world > 1 else "")}

    # ---- weak scaling (N > 1): 1024 rows per rank ------------------------
    weak = None
    if world > 1 and strong and not args.no_weak:
        wp = ShardedPass(tc, args.batch * world, dt, _lib.KLAY_LOG, world, rank, device=dev)
        rng2 = np.random.Generator(np.random.Philox(key=2))
        wp.weights.copy_(torch.from_numpy(np.log(rng2.uniform(
            0.05, 0.95, size=(wp.local_batch, tc.num_inputs))).astype(np.float32)))
        for _ in range(3):
            wp.step()
        dist.barrier()
        ms_w = _timed_replays(wp.step, args.steps, dev)
        t = torch.tensor([ms_w], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_w = float(t.item())
        weak = {"rows_per_gpu": args.batch, "global_batch": args.batch * world,
                "ms_per_step": ms_w, "value": args.batch * world / (ms_w / 1e3)}

    extra = None
    if world == 1 and not args.no_extra:
        # the other BASELINE configs and a 1-GPU batch sweep of config C (the
        # strong-scaling proxy: 1024 / G rows per GPU at G = 2, 4, 8),
        # device-timed; parity cases, not the headline
        extra = {
            "A_real_f64_b1_fwd": measure_config("A", "real", np.float64, 1, False, dev),
            "B_log_f64_b256_fwd_bwd": measure_config("B", "log", np.float64, 256, True, dev),
            "B_real_f64_b256_fwd_bwd": measure_config("B", "real", np.float64, 256, True, dev),
            "D_bool_b4096_fwd": measure_config("D", "bool", np.float32, 4096, False, dev),
            "D_bool_packed_b4096_fwd": measure_config("D", "bool_packed", "u1", 4096, False, dev),
            "D_real_f32_b4096_fwd": measure_config("D", "real", np.float32, 4096, False, dev),
            "E_log_f64_b128_fwd_bwd": measure_config("E", "log", np.float64, 128, True, dev),
            "Cp_log_f32_b1024_fwd_bwd": measure_config("Cp", "log", np.float32, 1024, True, dev,
                                                       iters=5),
        }
        for b in (512, 256, 128):
            r = measure_config("C", "log", np.float32, b, True, dev)
            r["linear_share_ratio"] = r["ms_per_batch"] / (ms_per_step * b / B_global)
            extra[f"C_log_f32_b{b}_fwd_bwd"] = r

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return 0
    nodes = tc.num_inputs + sum(l.width for l in tc.layers)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "nodes": nodes,
                   "edges": int(sum(len(l.sources) for l in tc.layers)),
                   "gate_layers": len(tc.layers), "semiring": "log", "pass": "fwd+bwd",
                   "global_batch": B_global, "batch_per_gpu": B,
                   "parallelism": f"dp{world} (batch-sharded, plan replicated; NCCL all-gather "
                                  "of outputs and grads each step)",
                   "l2": f"no flush: per-step working set {nodes * B * s / 1e9:.2f} GB trace "
                         ">> 126 MB L2",
                   "bytes_per_eval_necessary": bpe_nec,
                   "step_frac_necessary": value / world * bpe_nec / (peak * 1e9),
                   "necessary_model": "bytes the implemented dataflow must move per launch "
                                      "class (bench.py class_bytes: layer_bytes for layer "
                                      "kernels, unary-node aliases and routes skip rows)",
                   "bytes_per_eval_contract": bpe,
                   "step_contract_frac": value / world * bpe / (peak * 1e9),
                   "contract_model": "SURVEY §8(d) (reference dataflow: every layer read and "
                                     "written, c_l = 2 for log-sum layers)"},
        "roofline": {"bound": "hbm", "kernel": dom,
                     "achieved": dt_["achieved_gbs"], "peak": peak, "peak_source": peak_kind,
                     "unit": "GB/s", "frac": dt_["frac"],
                     "contract_frac": dt_["contract_frac"],
                     "traffic": (dt_["ncu_dram_bytes"] / nl) if "ncu_dram_bytes" in dt_ else None,
                     "traffic_scope": f"ncu DRAM read+write bytes per launch of the dominant "
                                      f"class (profiles/{args.launch_list}, same build and "
                                      "workload)",
                     "bytes_per_launch": dt_["necessary_bytes"] / nl,
                     "launches_per_step": nl, "ms_per_step": dt_["ms"],
                     "timing": "in-graph: one CUDA graph of just this class's launches of a "
                               "step, replayed between CUDA events (bench.py time_classes)",
                     "templates": templates,
                     "sum_template_ms": sum(t["ms"] for t in templates.values())},
        "gpu_launches": int(launches_per_step * args.steps),
        "launch_mode": "CUDA graph replay of the captured fwd+bwd "
                       f"({launches_per_step} libklay kernels per step)",
        "clocks": clk,
        "sustained": sustained,
        "cpu_baseline": cpu_line,
        "e2e": e2e,
        "weak_scaling": weak,
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
    ap.add_argument("--batch", type=int, default=1024,
                    help="global batch (strong scaling) or rows per GPU (weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--sustain", type=float, default=2.0, help="seconds of sustained replay")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-single-seconds", type=float, default=4.0)
    ap.add_argument("--launch-list", default="r2_launches.csv",
                    help="committed ncu launch list under profiles/ (per-class DRAM bytes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other-config measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
