"""Batched forward/backward evaluation of tensorized circuits on B200.

Drop-in mirror of the reference engine API
(``/root/reference/pkg/src/laycirc/engine.py``): ``WeightAssignment``,
``weights_from_*``, ``EvalTrace``, ``Semiring`` / ``REAL`` / ``BOOLEAN`` /
``MAX_PRODUCT``, ``forward_real``, ``forward_log``, ``evaluate_semiring``,
``backward``, ``gradient`` — same names, argument meaning, return shapes and
``EvalError`` behaviour. Any object with the reference ``TensorizedCircuit``
attributes is accepted (including a reference instance).

Every layer runs in ``libklay.so`` (hand-written sm_100a kernels, C ABI in
``include/klay.h``); there is no CPU fallback. Host numpy arrays in and out,
as in the reference; ``DevicePlan`` is the device-resident fast path used by
the torch module and the benchmark (inputs already in HBM).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from .tensorized import PRODUCT, Literal

REAL_DOMAIN = "real"
LOG_DOMAIN = "log"


class EvalError(ValueError):
    """Shape or domain mismatch between circuit, weights, and traces (engine.py:30-31)."""


# --------------------------------------------------------------------------
# weights (engine.py:34-118)
# --------------------------------------------------------------------------

@dataclass
class WeightAssignment:
    """Per-input-slot values, one row per batch element."""

    values: np.ndarray  # [batch, num_inputs]
    domain: str = REAL_DOMAIN

    def __post_init__(self) -> None:
        self.values = np.atleast_2d(np.asarray(self.values, dtype=np.float64))
        if self.values.ndim != 2 or self.values.shape[0] < 1:
            raise EvalError("weights must be a [batch, num_inputs] matrix with batch >= 1")
        if self.domain not in (REAL_DOMAIN, LOG_DOMAIN):
            raise EvalError(f"unknown weight domain {self.domain!r}")
        if self.domain == REAL_DOMAIN and not np.all(np.isfinite(self.values)):
            raise EvalError("real-domain weights must be finite")
        if self.domain == LOG_DOMAIN and np.any(self.values == np.inf):
            raise EvalError("log-domain weights must be < +inf")

    @property
    def batch(self) -> int:
        return self.values.shape[0]

    @property
    def num_inputs(self) -> int:
        return self.values.shape[1]

    def to_log(self) -> "WeightAssignment":
        if self.domain == LOG_DOMAIN:
            return self
        with np.errstate(divide="ignore"):
            return WeightAssignment(np.log(self.values), LOG_DOMAIN)


def _code(lit) -> int:
    return int(lit.to_dimacs())


def weights_from_map(input_map: Mapping, per_literal: Mapping, domain: str = REAL_DOMAIN
                     ) -> WeightAssignment:
    """Single-row assignment from an explicit literal -> value map."""
    by_code = {_code(k): float(v) for k, v in per_literal.items()}
    row = np.empty(len(input_map), dtype=np.float64)
    for lit, slot in input_map.items():
        c = _code(lit)
        if c not in by_code:
            raise EvalError(f"missing weight for literal {lit}")
        row[slot] = by_code[c]
    return WeightAssignment(row[np.newaxis, :], domain)


def weights_from_probabilities(input_map: Mapping, prob: Mapping[int, float]) -> WeightAssignment:
    """Real weights from variable probabilities; the negative literal gets 1 - p."""
    per = {}
    for lit in input_map:
        if lit.variable not in prob:
            raise EvalError(f"missing probability for variable {lit.variable}")
        p = float(prob[lit.variable])
        per[Literal(lit.variable, lit.positive)] = p if lit.positive else 1.0 - p
    return weights_from_map(input_map, per)


def weights_from_json(payload, input_map: Mapping) -> WeightAssignment:
    """``{"p": {...}}`` / ``{"w": {...}}`` objects, or a list of them (batched)."""
    rows = payload if isinstance(payload, list) else [payload]
    if not rows:
        raise EvalError("weight file contains no rows")
    out = []
    for row in rows:
        if not isinstance(row, dict) or len(row.keys() & {"p", "w"}) != 1:
            raise EvalError("each weight row must have exactly one of 'p' or 'w'")
        if "p" in row:
            prob = {int(k): float(v) for k, v in row["p"].items()}
            out.append(weights_from_probabilities(input_map, prob).values[0])
        else:
            per = {Literal.from_dimacs(int(k)): float(v) for k, v in row["w"].items()}
            out.append(weights_from_map(input_map, per).values[0])
    return WeightAssignment(np.stack(out), REAL_DOMAIN)


# --------------------------------------------------------------------------
# semirings (engine.py:158-193)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Semiring:
    """Named semiring evaluated by the device kernels (``code`` = KLAY_*)."""

    name: str
    zero: float
    one: float
    code: int


REAL = Semiring("real", 0.0, 1.0, _lib.KLAY_REAL)
BOOLEAN = Semiring("bool", 0.0, 1.0, _lib.KLAY_BOOL)
MAX_PRODUCT = Semiring("maxprod", 0.0, 1.0, _lib.KLAY_MAXPROD)
SEMIRINGS = {s.name: s for s in (REAL, BOOLEAN, MAX_PRODUCT)}


# --------------------------------------------------------------------------
# device plan: the immutable per-circuit device state (engine._plans)
# --------------------------------------------------------------------------

def _torch():
    import torch
    return torch


U1 = "u1"  # bit-packed Boolean rows (KLAY_U1): 32 batch rows per 32-bit word


def _resolve_dtype(dtype):
    if isinstance(dtype, str) and dtype == U1:
        return U1
    if dtype is None:
        return np.float64
    dt = np.dtype(dtype)
    if dt == np.float64:
        return np.float64
    if dt == np.float32:
        return np.float32
    raise EvalError(f"unsupported dtype {dt} (float32 or float64)")


def _klay_dtype(np_dtype) -> int:
    if isinstance(np_dtype, str) and np_dtype == U1:
        return _lib.KLAY_U1
    return _lib.KLAY_F64 if np.dtype(np_dtype) == np.float64 else _lib.KLAY_F32


def _torch_dtype(dtype):
    torch = _torch()
    if isinstance(dtype, str) and dtype == U1:
        return torch.int32
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


class DevicePlan:
    """Device copy of a circuit's index vectors (CSR + transposed CSR).

    Built once per (circuit, device) and cached on the circuit object like
    the reference's ``tc._plans_cache`` (engine.py:138-155). Read-only after
    creation; safe to share across streams.
    """

    def __init__(self, tc, device=None):
        torch = _torch()
        lib = _lib.load()
        if not torch.cuda.is_available():
            raise _lib.KlayLibError("a CUDA device is required (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.num_inputs = int(tc.num_inputs)
        self.num_layers = len(tc.layers)
        self.widths = [int(l.width) for l in tc.layers]
        self.num_roots = int(tc.num_roots)
        widths = np.array(self.widths, dtype=np.int64)
        counts = np.array([len(l.sources) for l in tc.layers], dtype=np.int64)
        for l, layer in enumerate(tc.layers, start=1):
            expected = PRODUCT if l % 2 == 1 else "sum"
            if layer.op != expected:
                from .tensorized import KlayFormatError
                raise KlayFormatError(f"layer {l} op {layer.op!r}, expected {expected!r}")
        if self.num_layers:
            src = np.ascontiguousarray(np.concatenate([np.asarray(l.sources, np.int64) for l in tc.layers]))
            seg = np.ascontiguousarray(np.concatenate([np.asarray(l.segments, np.int64) for l in tc.layers]))
        else:
            src = seg = np.zeros(1, np.int64)
        root_nodes = np.full(self.num_roots, -1, dtype=np.int64)
        const_vals = np.zeros(max(self.num_roots, 1), dtype=np.int8)
        free = [p for p in range(self.num_roots) if p not in tc.constant_roots]
        if len(free) != len(tc.root_indices):
            raise EvalError("root_indices and constant_roots do not add up to num_roots")
        for p, r in zip(free, tc.root_indices):
            root_nodes[p] = int(r)
        for p, b in tc.constant_roots.items():
            const_vals[p] = 1 if b else 0
        root_nodes_buf = np.ascontiguousarray(root_nodes if self.num_roots else np.zeros(1, np.int64))
        handle = ctypes.c_void_p()
        rc = lib.klay_plan_create(
            self.num_inputs, self.num_layers, widths.ctypes.data, counts.ctypes.data,
            src.ctypes.data, seg.ctypes.data, self.num_roots, root_nodes_buf.ctypes.data,
            const_vals.ctypes.data, self.device.index, ctypes.byref(handle))
        _lib.check(rc, "klay_plan_create")
        self._handle = handle
        self._lib = lib
        self.num_nodes = int(lib.klay_plan_num_nodes(handle))
        self.max_width = int(lib.klay_plan_max_width(handle))
        self.layer_offsets = [int(lib.klay_plan_layer_offset(handle, l))
                              for l in range(self.num_layers + 1)]
        sched = (ctypes.c_int64 * 8)()
        _lib.check(lib.klay_plan_schedule(handle, sched), "klay_plan_schedule")
        # {tail, micro, micro_bwd}: first 0-based gate layer of each tail
        # (num_layers = none); aliased rows of a backward-only trace; layers
        # in the forward / backward micro heads; rows of the backward's
        # adjoint buffer (layers with disjoint lifetimes share rows)
        self.schedule = {"tail": sched[0], "micro": sched[1], "micro_bwd": sched[2],
                         "aliased_rows": sched[3], "head": sched[4], "head_bwd": sched[5],
                         "adjoint_rows": sched[6]}

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.klay_plan_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def handle(self):
        return self._handle

    def row_stride(self, batch: int, dtype) -> int:
        return int(self._lib.klay_row_stride(batch, _klay_dtype(dtype)))

    def _stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    # ---- device-resident entry points (torch tensors in / out) ----------
    def alloc_values(self, batch: int, dtype, retain: bool = True):
        torch = _torch()
        ld = self.row_stride(batch, dtype)
        rows = self.num_nodes if retain else 2 * self.max_width
        return torch.empty((rows, ld), dtype=_torch_dtype(dtype), device=self.device)

    def forward_workspace(self, batch: int, dtype):
        """Scratch for split (heavy) segments, or None when not needed."""
        torch = _torch()
        ld = self.row_stride(batch, dtype)
        nbytes = int(self._lib.klay_forward_workspace(self._handle, _klay_dtype(dtype), ld))
        if nbytes == 0:
            return None
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    # ---- caller-buffer validation (the C ABI sees raw pointers only) -------
    def _check_buf(self, t, name, dtype, shape=None, min_rows=None, min_bytes=None):
        """Raise EvalError unless `t` is a contiguous tensor of `dtype` on this
        plan's device with the given exact `shape`, at least `min_rows` rows
        or at least `min_bytes` bytes."""
        if t.device != self.device:
            raise EvalError(f"{name} is on {t.device}, the circuit plan on {self.device}")
        if dtype is not None and t.dtype != dtype:
            raise EvalError(f"{name} has dtype {t.dtype}, expected {dtype}")
        if not t.is_contiguous():
            raise EvalError(f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise EvalError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        if min_rows is not None and (t.dim() != 2 or t.shape[0] < min_rows):
            raise EvalError(f"{name} has {t.shape[0] if t.dim() else 0} rows, needs >= {min_rows}")
        if min_bytes is not None and t.numel() * t.element_size() < min_bytes:
            raise EvalError(f"{name} has {t.numel() * t.element_size()} bytes, needs >= {min_bytes}")

    def _check_values(self, values, batch, dtype, retain):
        ld = self.row_stride(batch, dtype)
        rows = self.num_nodes if retain else 2 * self.max_width
        self._check_buf(values, "values", _torch_dtype(dtype), min_rows=rows)
        if values.shape[1] < ld:
            raise EvalError(f"values rows hold {values.shape[1]} elements, batch {batch} needs {ld}")

    def forward(self, weights, semiring: int, dtype, retain=True, epsilon=0.0,
                values=None, outputs=None, workspace=None):
        """weights: cuda tensor [B, K] (float32/float64, semiring domain).
        retain: False (no trace), True (the trace backward() needs: rows of
        unary nodes may be left out and are filled by fill_trace() /
        on first host access) or "full".
        Returns (outputs [B, R] tensor, values buffer [rows, ld])."""
        torch = _torch()
        if weights.dim() != 2 or weights.shape[1] != self.num_inputs:
            raise EvalError(f"weights have {weights.shape[-1]} columns, circuit expects {self.num_inputs}")
        B = int(weights.shape[0])
        if B < 1:
            raise EvalError("batch must be >= 1")
        if weights.dtype not in (torch.float32, torch.float64):
            raise EvalError("weights must be float32 or float64")
        if weights.device != self.device:
            raise EvalError(f"weights are on {weights.device}, the circuit plan on {self.device}")
        if not weights.is_contiguous():
            weights = weights.contiguous()
        wdt = _lib.KLAY_F64 if weights.dtype == torch.float64 else _lib.KLAY_F32
        if values is None:
            values = self.alloc_values(B, dtype, retain)
        else:
            self._check_values(values, B, dtype, retain)
        ld = values.shape[1]
        # bit-packed Boolean rows return 0/1 outputs in the weights' dtype
        tdt = weights.dtype if _klay_dtype(dtype) == _lib.KLAY_U1 else _torch_dtype(dtype)
        if outputs is None:
            outputs = torch.empty((B, self.num_roots), dtype=tdt, device=self.device)
        else:
            self._check_buf(outputs, "outputs", tdt, shape=(B, self.num_roots))
        need = int(self._lib.klay_forward_workspace(self._handle, _klay_dtype(dtype), ld))
        if workspace is None:
            workspace = torch.empty(need, dtype=torch.uint8, device=self.device) if need else None
        elif need:
            self._check_buf(workspace, "workspace", None, min_bytes=need)
        mode = 0 if not retain else (1 if retain == "full" else _lib.KLAY_RETAIN_BACKWARD)
        rc = self._lib.klay_forward(
            self._handle, semiring, _klay_dtype(dtype), weights.data_ptr(), wdt,
            values.data_ptr(), ld, mode,
            outputs.data_ptr() if self.num_roots else None, B, float(epsilon),
            workspace.data_ptr() if workspace is not None else None, self._stream())
        _lib.check(rc, "klay_forward")
        # the trace's epsilon, for backward()'s unary-parent shortcut
        values.klay_epsilon = float(epsilon) if semiring == _lib.KLAY_LOG else -1.0
        # a backward-only trace: complete it before reading rows on the host
        values.klay_partial = (mode == _lib.KLAY_RETAIN_BACKWARD, B, semiring, float(epsilon))
        return outputs, values

    def fill_trace(self, values, batch: int):
        """Write the rows a backward-only trace left out (klay_fill_trace);
        no-op for complete traces."""
        partial = getattr(values, "klay_partial", None)
        if not partial or not partial[0]:
            return values
        _, B, semiring, epsilon = partial
        if values.dtype in (_torch().float32, _torch().float64):
            dt = _lib.KLAY_F64 if values.dtype == _torch().float64 else _lib.KLAY_F32
            rc = self._lib.klay_fill_trace(self._handle, semiring, dt, values.data_ptr(),
                                           values.shape[1], B, epsilon, self._stream())
            _lib.check(rc, "klay_fill_trace")
        values.klay_partial = None
        return values

    def capture(self, batch: int, dtype, semiring: int, epsilon: float = 0.0,
                backward: bool = True, seeded: bool = False,
                host_io: bool = False) -> "CapturedPass":
        """A CUDA-graph-captured forward (+ backward) over fixed buffers."""
        return CapturedPass(self, batch, dtype, semiring, epsilon, backward, seeded, host_io)

    def workspace(self, batch: int, dtype):
        torch = _torch()
        ld = self.row_stride(batch, dtype)
        nbytes = int(self._lib.klay_backward_workspace(self._handle, _klay_dtype(dtype), ld))
        return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.device)

    def backward(self, values, batch: int, domain: int, dtype, seed=None, grads=None,
                 workspace=None, epsilon=None):
        """values: retained trace buffer from forward(). seed: cuda [B, R] or
        None (ones). epsilon: the trace's epsilon (default: the one forward()
        recorded on `values`; unknown disables the unary-parent shortcut).
        Returns grads [B, K] tensor."""
        torch = _torch()
        if isinstance(dtype, str) and dtype == U1:
            raise EvalError("no backward for bit-packed Boolean rows")
        tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
        if batch < 1:
            raise EvalError("batch must be >= 1")
        self._check_values(values, batch, dtype, True)
        ld = values.shape[1]
        if grads is None:
            grads = torch.empty((batch, self.num_inputs), dtype=tdt, device=self.device)
        else:
            self._check_buf(grads, "grads", tdt, shape=(batch, self.num_inputs))
        need = int(self._lib.klay_backward_workspace(self._handle, _klay_dtype(dtype), ld))
        if workspace is None:
            workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=self.device)
        else:
            self._check_buf(workspace, "workspace", None, min_bytes=need)
        if seed is not None:
            if tuple(seed.shape) != (batch, self.num_roots):
                raise EvalError(f"seed must have shape {(batch, self.num_roots)}")
            seed = seed.to(device=self.device, dtype=tdt).contiguous()
        if epsilon is None:
            epsilon = getattr(values, "klay_epsilon", -1.0)
        if domain != _lib.KLAY_LOG or epsilon != 0.0:
            # this backward reads every row: complete a backward-only trace
            self.fill_trace(values, batch)
        partial = getattr(values, "klay_partial", None)
        retain = _lib.KLAY_RETAIN_BACKWARD if partial and partial[0] else 1
        rc = self._lib.klay_backward(
            self._handle, domain, _klay_dtype(dtype), values.data_ptr(), values.shape[1],
            seed.data_ptr() if seed is not None else None,
            grads.data_ptr() if self.num_inputs else None, workspace.data_ptr(), batch,
            float(epsilon), retain, self._stream())
        _lib.check(rc, "klay_backward")
        return grads


class CapturedPass:
    """One forward (+ backward) pass of a plan over fixed device buffers,
    captured once in a CUDA graph and replayed (no per-layer host launches).

    Write inputs into ``weights`` ([B, K]) and ``seed`` ([B, R], backward
    only), call ``replay()``; results land in ``outputs`` ([B, R]) and
    ``grads`` ([B, K]) on the plan's device, stream-ordered on the current
    stream. The buffers are reused by every replay.
    """

    def __init__(self, plan: DevicePlan, batch: int, dtype, semiring: int, epsilon: float = 0.0,
                 backward: bool = True, seeded: bool = False, host_io: bool = False):
        torch = _torch()
        dt = _resolve_dtype(dtype)
        tdt = torch.float64 if dt == np.float64 else torch.float32
        if backward and semiring not in (_lib.KLAY_REAL, _lib.KLAY_LOG):
            raise EvalError("backward is defined for the real and log semirings only")
        self.plan, self.batch, self.dtype = plan, batch, dt
        dev = plan.device
        self.weights = torch.zeros((batch, plan.num_inputs), dtype=tdt, device=dev)
        self.outputs = torch.empty((batch, plan.num_roots), dtype=tdt, device=dev)
        self.grads = torch.empty((batch, plan.num_inputs), dtype=tdt, device=dev) if backward else None
        self.seed = torch.ones((batch, plan.num_roots), dtype=tdt, device=dev) if seeded else None
        self.values = plan.alloc_values(batch, dt, retain=backward)
        self._fw = plan.forward_workspace(batch, dt)
        self._bw = plan.workspace(batch, dt) if backward else None
        # host_io: pinned host buffers h_weights / h_seed / h_out / h_grad, the
        # copies captured in the graph too (one launch per call)
        self.host_io = host_io
        if host_io:
            pin = dict(dtype=tdt, pin_memory=True)
            self.h_weights = torch.empty(self.weights.shape, **pin)
            self.h_out = torch.empty(self.outputs.shape, **pin)
            self.h_grad = torch.empty(self.grads.shape, **pin) if backward else None
            self.h_seed = torch.empty(self.seed.shape, **pin) if seeded else None

        def run():
            if host_io:
                self.weights.copy_(self.h_weights, non_blocking=True)
                if seeded:
                    self.seed.copy_(self.h_seed, non_blocking=True)
            plan.forward(self.weights, semiring, dt, retain=backward, epsilon=epsilon,
                         values=self.values, outputs=self.outputs, workspace=self._fw)
            if backward:
                plan.backward(self.values, batch, semiring, dt, seed=self.seed, grads=self.grads,
                              workspace=self._bw)
            if host_io:
                self.h_out.copy_(self.outputs, non_blocking=True)
                if backward:
                    self.h_grad.copy_(self.grads, non_blocking=True)

        # warm up outside capture (kernel attributes, lazy module loading)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            run()
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            run()

    def replay(self):
        self.graph.replay()


def device_plan(tc, device=None) -> DevicePlan:
    """Cached DevicePlan of ``tc`` on ``device`` (default: current CUDA device)."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.KlayLibError("a CUDA device is required (no CPU fallback)")
    idx = torch.cuda.current_device() if device is None else (torch.device(device).index or 0)
    cache = getattr(tc, "_klay_device_plans", None)
    if cache is None:
        cache = {}
        try:
            tc._klay_device_plans = cache
        except AttributeError:
            pass
    plan = cache.get(idx)
    if plan is None:
        plan = DevicePlan(tc, torch.device("cuda", idx))
        cache[idx] = plan
    return plan


# --------------------------------------------------------------------------
# traces (engine.py:121-128)
# --------------------------------------------------------------------------

class _NodeValues(Sequence):
    """Lazy host view of a device trace: item l is the [batch, width_l]
    numpy matrix of layer l (0 = inputs), copied on first access."""

    def __init__(self, plan: DevicePlan, values, batch: int):
        self._plan, self._values, self._batch = plan, values, batch
        self._cache = {}

    def __len__(self):
        return self._plan.num_layers + 1

    def __getitem__(self, l):
        if isinstance(l, slice):
            return [self[i] for i in range(*l.indices(len(self)))]
        if l < 0:
            l += len(self)
        if not 0 <= l < len(self):
            raise IndexError(l)
        if l not in self._cache:
            self._plan.fill_trace(self._values, self._batch)
            start = self._plan.layer_offsets[l]
            w = self._plan.num_inputs if l == 0 else self._plan.widths[l - 1]
            block = self._values[start:start + w, :self._batch]
            self._cache[l] = block.t().contiguous().cpu().numpy()
        return self._cache[l]


@dataclass
class EvalTrace:
    """Forward-pass record: per-layer node values (when retained) and root outputs."""

    domain: str
    outputs: np.ndarray  # [batch, num_roots]
    node_values: Sequence | None  # [batch, width_l] per layer 0..L
    epsilon: float = 0.0
    _device_values: object = field(default=None, repr=False)
    _plan: object = field(default=None, repr=False)
    _dtype: object = field(default=None, repr=False)


# --------------------------------------------------------------------------
# reference-facing API (engine.py:196-384)
# --------------------------------------------------------------------------

def _check_shapes(tc, weights: WeightAssignment) -> None:
    if weights.num_inputs != tc.num_inputs:
        raise EvalError(
            f"weights have {weights.num_inputs} columns, circuit expects {tc.num_inputs}")


def _run(tc, values: np.ndarray, code: int, dtype, retain: bool, epsilon: float = 0.0):
    torch = _torch()
    plan = device_plan(tc)
    w = torch.from_numpy(np.ascontiguousarray(values)).to(plan.device, non_blocking=True)
    out, buf = plan.forward(w, code, dtype, retain=retain, epsilon=epsilon)
    return plan, out.cpu().numpy(), buf


def forward_real(tc, weights: WeightAssignment, retain_trace: bool = True, dtype=None) -> EvalTrace:
    """Evaluate in the real semiring; returns the trace with root outputs."""
    if weights.domain != REAL_DOMAIN:
        raise EvalError("forward_real requires real-domain weights")
    _check_shapes(tc, weights)
    dt = _resolve_dtype(dtype)
    plan, out, buf = _run(tc, weights.values, _lib.KLAY_REAL, dt, retain_trace)
    nv = _NodeValues(plan, buf, weights.batch) if retain_trace else None
    return EvalTrace(REAL_DOMAIN, out, nv, 0.0, buf if retain_trace else None, plan, dt)


def forward_log(tc, weights: WeightAssignment, epsilon: float = 0.0, retain_trace: bool = True,
                dtype=None) -> EvalTrace:
    """Log semiring: products are sums, sums a max-trick logsumexp; all -inf
    segments give -inf, never NaN; ``epsilon`` is added inside the log."""
    if weights.domain != LOG_DOMAIN:
        raise EvalError("forward_log requires log-domain weights")
    if epsilon < 0:
        raise EvalError("epsilon must be >= 0")
    _check_shapes(tc, weights)
    dt = _resolve_dtype(dtype)
    plan, out, buf = _run(tc, weights.values, _lib.KLAY_LOG, dt, retain_trace, epsilon)
    nv = _NodeValues(plan, buf, weights.batch) if retain_trace else None
    return EvalTrace(LOG_DOMAIN, out, nv, epsilon, buf if retain_trace else None, plan, dt)


def _device_semiring(semiring) -> Semiring:
    """The device semiring for ``semiring``: one of this module's instances,
    or any object with the reference ``Semiring`` fields (engine.py:158-191)
    whose name and identities are those of a built-in one -- e.g. the
    reference's own REAL / BOOLEAN / MAX_PRODUCT. Semirings with other
    reductions have no device kernels and raise (there is no CPU path)."""
    if isinstance(semiring, Semiring) and SEMIRINGS.get(semiring.name) is semiring:
        return semiring
    name = getattr(semiring, "name", None)
    ours = SEMIRINGS.get(name) if isinstance(name, str) else None
    if ours is None:
        raise EvalError(f"unsupported semiring {name if name is not None else semiring!r}: only "
                        f"{sorted(SEMIRINGS)} and 'log' have device kernels")
    if (float(getattr(semiring, "zero", ours.zero)) != ours.zero
            or float(getattr(semiring, "one", ours.one)) != ours.one):
        raise EvalError(f"semiring {name!r} has identities ({semiring.zero}, {semiring.one}); "
                        f"the device {name!r} semiring uses ({ours.zero}, {ours.one})")
    return ours


def evaluate_semiring(tc, weights: WeightAssignment, semiring) -> np.ndarray:
    """Forward evaluation under a named semiring; returns [batch, roots]."""
    if isinstance(semiring, str):
        if semiring == "log":
            return forward_log(tc, weights.to_log(), retain_trace=False).outputs
        if semiring not in SEMIRINGS:
            raise EvalError(f"unknown semiring {semiring!r}")
        semiring = SEMIRINGS[semiring]
    semiring = _device_semiring(semiring)
    _check_shapes(tc, weights)
    dt = np.float64
    if semiring is BOOLEAN and np.all((weights.values == 0.0) | (weights.values == 1.0)):
        # exact 0/1 inputs: bit-packed rows (AND / OR on 32 rows per word);
        # identical to the float max/min evaluation on 0/1 values
        dt = U1
    _, out, _ = _run(tc, weights.values, semiring.code, dt, False)
    return out


def _upload_trace(tc, trace, plan):
    """Device trace from a host trace (e.g. a reference EvalTrace)."""
    torch = _torch()
    nv = trace.node_values
    dt = np.float64 if nv[0].dtype == np.float64 else np.float32
    batch = nv[0].shape[0]
    buf = plan.alloc_values(batch, dt, retain=True)
    for l, m in enumerate(nv):
        start = plan.layer_offsets[l]
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=dt).T)).to(plan.device)
        buf[start:start + t.shape[0], :batch].copy_(t)
    return buf, dt


def backward(tc, trace: EvalTrace, seed: np.ndarray | None = None) -> np.ndarray:
    """Gradient of ``sum_r seed[:, r] * root_r`` w.r.t. the input slots
    (engine.py:307-355); zero-safe product adjoints in the real domain."""
    torch = _torch()
    if trace.node_values is None:
        raise EvalError("backward requires a trace with retain_trace=True")
    if len(trace.node_values) != len(tc.layers) + 1:
        raise EvalError("trace does not match circuit layer count")
    plan = device_plan(tc)
    buf = getattr(trace, "_device_values", None)
    if buf is None or getattr(trace, "_plan", None) is not plan:
        # a host trace may hold any values: read every parent (epsilon unknown)
        buf, dt = _upload_trace(tc, trace, plan)
        batch = trace.node_values[0].shape[0]
        eps = -1.0
    else:
        dt = trace._dtype
        batch = trace.outputs.shape[0]
        eps = trace.epsilon
    if seed is not None:
        seed = np.asarray(seed, dtype=dt)
        if seed.shape != (batch, tc.num_roots):
            raise EvalError(f"seed must have shape {(batch, tc.num_roots)}")
        seed = torch.from_numpy(np.ascontiguousarray(seed)).to(plan.device, non_blocking=True)
    domain = _lib.KLAY_LOG if trace.domain == LOG_DOMAIN else _lib.KLAY_REAL
    grads = plan.backward(buf, batch, domain, dt, seed=seed, epsilon=eps)
    return grads.cpu().numpy()


# gradient()'s captured passes: at most ONE per device plan, stored on the
# plan itself (so it dies with the circuit) and replaced when the batch,
# dtype, domain, epsilon or seeding changes. A per-plan lock makes the
# write-inputs / replay / read-outputs sequence atomic: concurrent callers on
# one circuit serialize instead of sharing the pinned buffers.
_PLANS_WITH_PASS: "weakref.WeakSet" = None  # filled lazily (clear_cache)
_PASS_LOCK = threading.Lock()               # guards creation of per-plan locks


def _plan_pass_lock(plan) -> threading.Lock:
    lock = getattr(plan, "_grad_lock", None)
    if lock is None:
        with _PASS_LOCK:
            lock = getattr(plan, "_grad_lock", None)
            if lock is None:
                lock = plan._grad_lock = threading.Lock()
    return lock


def clear_cache() -> None:
    """Drop the cached captured passes of ``gradient`` (frees their buffers)."""
    global _PLANS_WITH_PASS
    if _PLANS_WITH_PASS is None:
        return
    for plan in list(_PLANS_WITH_PASS):
        with _plan_pass_lock(plan):
            plan._grad_pass = None
    _PLANS_WITH_PASS.clear()


def cached_passes() -> int:
    """Number of captured ``gradient`` passes currently resident."""
    if _PLANS_WITH_PASS is None:
        return 0
    return sum(1 for p in list(_PLANS_WITH_PASS) if getattr(p, "_grad_pass", None) is not None)


def gradient(tc, weights: WeightAssignment, log_domain: bool = False, epsilon: float = 0.0,
             seed: np.ndarray | None = None, dtype=None) -> tuple[np.ndarray, np.ndarray]:
    """Forward + backward; returns (outputs, input grads) (engine.py:372-384).

    No trace escapes this call, so it runs a CUDA-graph-captured pass: one
    H2D copy of the weights (and seed), one graph replay, one D2H copy of
    outputs and grads. One pass is cached per circuit (replaced when the
    batch, dtype, domain, epsilon or seeding changes); calls on one circuit
    from several threads serialize on a per-circuit lock. ``dtype`` (float64
    default, or float32) is an extension of the reference signature;
    ``clear_cache()`` frees the cached buffers."""
    global _PLANS_WITH_PASS
    torch = _torch()
    w = weights.to_log() if log_domain else weights
    if log_domain and epsilon < 0:
        raise EvalError("epsilon must be >= 0")
    if not log_domain and w.domain != REAL_DOMAIN:
        raise EvalError("forward_real requires real-domain weights")
    _check_shapes(tc, w)
    dt = _resolve_dtype(dtype)
    if dt == U1:
        raise EvalError("gradient needs a float dtype")
    plan = device_plan(tc)
    B = w.batch
    code = _lib.KLAY_LOG if log_domain else _lib.KLAY_REAL
    if seed is not None:
        sd = np.asarray(seed, dtype=np.dtype(dt))
        if sd.shape != (B, tc.num_roots):
            raise EvalError(f"seed must have shape {(B, tc.num_roots)}")
    key = (B, np.dtype(dt).str, code, float(epsilon), seed is not None)
    with _plan_pass_lock(plan):
        entry = getattr(plan, "_grad_pass", None)
        if entry is None or entry[0] != key:
            plan._grad_pass = None  # free the old buffers before allocating new ones
            cap = plan.capture(B, dt, code, epsilon=epsilon, backward=True,
                               seeded=seed is not None, host_io=True)
            plan._grad_pass = (key, cap)
            with _PASS_LOCK:
                if _PLANS_WITH_PASS is None:
                    _PLANS_WITH_PASS = weakref.WeakSet()
                _PLANS_WITH_PASS.add(plan)
        cap = plan._grad_pass[1]
        # (pinned buffers idle: the previous call synchronized; torch's copy_
        # converts on several host threads)
        cap.h_weights.copy_(torch.from_numpy(np.ascontiguousarray(w.values)))
        if seed is not None:
            cap.h_seed.copy_(torch.from_numpy(np.ascontiguousarray(sd)))
        cap.replay()  # H2D, forward, backward, D2H: one graph launch
        torch.cuda.current_stream(plan.device).synchronize()
        return cap.h_out.clone().numpy(), cap.h_grad.clone().numpy()
