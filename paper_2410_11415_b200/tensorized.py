"""Tensorized-circuit data contract: the input layout of the evaluation path.

Mirrors the reference's ``TensorLayer`` / ``TensorizedCircuit`` /
``validate`` (``/root/reference/pkg/src/laycirc/tensorize.py:43-132``) and
its ``.klay`` text format (``tensorize.py:197-313``), plus a compressed
binary ``.npz`` sidecar used for the large benchmark circuits (SURVEY §8(f)
row 2). The engine only duck-types these attributes, so a reference
``laycirc.TensorizedCircuit`` can be passed to ``engine.*`` unchanged.

Per gate layer ``l`` (1-based): ``op`` alternates ``prod`` (odd) / ``sum``
(even); ``sources[e]`` indexes the previous layer (gather), ``segments[e]``
is the nondecreasing parent id covering ``0..width-1``; every node of the
previous layer is read at least once.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping

import numpy as np

PRODUCT = "prod"
SUM = "sum"
KLAY_VERSION = 1


class KlayFormatError(ValueError):
    """Malformed or invariant-violating circuit content (tensorize.py:39-40)."""


@dataclass(frozen=True)
class Literal:
    """A propositional variable (1-based) or its negation (circuit.py:29-53)."""

    variable: int
    positive: bool = True

    def __post_init__(self) -> None:
        if self.variable < 1:
            raise ValueError(f"variable index must be >= 1, got {self.variable}")

    def __neg__(self) -> "Literal":
        return Literal(self.variable, not self.positive)

    @classmethod
    def from_dimacs(cls, code: int) -> "Literal":
        if code == 0:
            raise ValueError("0 is not a DIMACS literal")
        return cls(abs(code), code > 0)

    def to_dimacs(self) -> int:
        return self.variable if self.positive else -self.variable

    def __str__(self) -> str:
        return str(self.to_dimacs())


def _dimacs(lit) -> int:
    """DIMACS code of any literal-like object (ours or the reference's)."""
    return int(lit.to_dimacs())


@dataclass
class TensorLayer:
    op: str
    width: int
    sources: np.ndarray
    segments: np.ndarray

    @property
    def num_edges(self) -> int:
        return len(self.sources)

    def __eq__(self, other: object) -> bool:
        if not hasattr(other, "sources"):
            return NotImplemented
        return (
            self.op == other.op
            and self.width == other.width
            and np.array_equal(self.sources, other.sources)
            and np.array_equal(self.segments, other.segments)
        )


@dataclass
class TensorizedCircuit:
    num_inputs: int
    num_vars: int
    layers: list
    input_map: dict
    root_indices: list
    constant_roots: dict = field(default_factory=dict)

    @property
    def num_roots(self) -> int:
        return len(self.root_indices) + len(self.constant_roots)

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    def __eq__(self, other: object) -> bool:
        if not hasattr(other, "layers"):
            return NotImplemented
        return (
            self.num_inputs == other.num_inputs
            and self.num_vars == other.num_vars
            and len(self.layers) == len(other.layers)
            and all(a == b for a, b in zip(self.layers, other.layers))
            and {_dimacs(k): v for k, v in self.input_map.items()}
            == {_dimacs(k): v for k, v in other.input_map.items()}
            and list(self.root_indices) == list(other.root_indices)
            and dict(self.constant_roots) == dict(other.constant_roots)
        )

    def validate(self) -> None:
        validate(self)


def validate(tc) -> None:
    """Structural invariants of ``tensorize.py:94-132``; raises KlayFormatError."""
    if tc.num_inputs < 0 or tc.num_vars < 0:
        raise KlayFormatError("negative input or variable count")
    if sorted(tc.input_map.values()) != list(range(tc.num_inputs)):
        raise KlayFormatError("input map does not cover slots 0..K-1 exactly once")
    for lit in tc.input_map:
        if lit.variable > tc.num_vars:
            raise KlayFormatError(f"input literal {lit} exceeds declared vars")
    prev_width = tc.num_inputs
    for l, layer in enumerate(tc.layers, start=1):
        expected = PRODUCT if l % 2 == 1 else SUM
        if layer.op != expected:
            raise KlayFormatError(f"layer {l} op {layer.op!r}, expected {expected!r}")
        if layer.width <= 0:
            raise KlayFormatError(f"layer {l} has nonpositive width")
        src = np.asarray(layer.sources)
        seg = np.asarray(layer.segments)
        if len(src) != len(seg):
            raise KlayFormatError(f"layer {l}: edge vectors differ in length")
        if len(src) == 0:
            raise KlayFormatError(f"layer {l} has no edges")
        if np.any(np.diff(seg) < 0):
            raise KlayFormatError(f"layer {l}: aggregation indices not nondecreasing")
        if seg[0] != 0 or seg[-1] != layer.width - 1 or len(np.unique(seg)) != layer.width:
            raise KlayFormatError(f"layer {l}: aggregation indices must cover 0..width-1")
        if src.min() < 0 or src.max() >= prev_width:
            raise KlayFormatError(f"layer {l}: edge index out of range")
        if len(np.unique(src)) != prev_width:
            raise KlayFormatError(f"layer {l}: some previous-layer node is never read")
        prev_width = layer.width
    last_width = tc.layers[-1].width if tc.layers else tc.num_inputs
    for r in tc.root_indices:
        if not 0 <= r < last_width:
            raise KlayFormatError(f"root index {r} outside final layer")
    positions = set(tc.constant_roots)
    if positions and (min(positions) < 0 or max(positions) >= tc.num_roots):
        raise KlayFormatError("constant root position out of range")


# --------------------------------------------------------------------------
# .klay text format (tensorize.py:197-313)
# --------------------------------------------------------------------------

def write_klay(tc, sink) -> None:
    """Serialize to the line-oriented ``.klay`` text format."""
    validate(tc)
    out = [f"klay {KLAY_VERSION}", f"inputs {tc.num_inputs}", f"vars {tc.num_vars}"]
    out.append("roots " + " ".join(str(int(r)) for r in tc.root_indices))
    if tc.constant_roots:
        out.append("constants " + " ".join(
            f"{p}:{int(b)}" for p, b in sorted(tc.constant_roots.items())))
    slots = sorted(tc.input_map.items(), key=lambda kv: kv[1])
    out.append("inputmap " + " ".join(f"{_dimacs(k)}:{v}" for k, v in slots))
    for l, layer in enumerate(tc.layers, start=1):
        out.append(f"layer {l} {layer.op} {layer.width} {len(layer.sources)}")
        out.append("S " + " ".join(map(str, np.asarray(layer.sources).tolist())))
        out.append("R " + " ".join(map(str, np.asarray(layer.segments).tolist())))
    text = "\n".join(out) + "\n"
    try:
        sink.write(text)
    except TypeError:
        sink.write(text.encode("ascii"))


def read_klay(source) -> TensorizedCircuit:
    """Parse and validate ``.klay`` text; rejects (never repairs) bad content.

    Parsed by libklay's C++ reader (``klay_read_klay``, about 10x faster on
    large circuits) when the library is built, else by the Python reader
    below; both accept and reject the same inputs (tests/test_boundary.py)."""
    text = source.read() if hasattr(source, "read") else source
    try:
        from . import _lib
        lib = _lib.load()
    except Exception:
        lib = None
    if lib is not None:
        return _read_klay_native(lib, text)
    return read_klay_py(text)


def _read_klay_native(lib, text) -> TensorizedCircuit:
    import ctypes
    data = text if isinstance(text, bytes) else text.encode("ascii", errors="strict")
    h = ctypes.c_void_p()
    rc = lib.klay_read_klay(data, len(data), ctypes.byref(h))
    if rc != 0:
        msg = (lib.klay_read_klay_error() or b"").decode(errors="replace")
        raise KlayFormatError(msg or f"klay_read_klay failed ({rc})")
    try:
        sz = np.zeros(7, np.int64)
        lib.klay_file_info(h, sz.ctypes.data)
        K, V, L, E, R, C, M = (int(x) for x in sz)
        widths, counts = np.empty(L, np.int64), np.empty(L, np.int64)
        src, seg = np.empty(E, np.int64), np.empty(E, np.int64)
        roots = np.empty(R, np.int64)
        cpos, cval = np.empty(C, np.int64), np.empty(C, np.int64)
        codes, slots = np.empty(M, np.int64), np.empty(M, np.int64)
        lib.klay_file_export(h, widths.ctypes.data, counts.ctypes.data, src.ctypes.data,
                             seg.ctypes.data, roots.ctypes.data, cpos.ctypes.data,
                             cval.ctypes.data, codes.ctypes.data, slots.ctypes.data)
    finally:
        lib.klay_file_destroy(h)
    layers, e0 = [], 0
    for l in range(L):
        n = int(counts[l])
        layers.append(TensorLayer(PRODUCT if l % 2 == 0 else SUM, int(widths[l]),
                                  src[e0:e0 + n].copy(), seg[e0:e0 + n].copy()))
        e0 += n
    input_map = {Literal.from_dimacs(int(c)): int(s) for c, s in zip(codes, slots)}
    return TensorizedCircuit(K, V, layers, input_map, [int(r) for r in roots],
                             {int(p): bool(v) for p, v in zip(cpos, cval)})


def read_klay_py(text) -> TensorizedCircuit:
    """The Python `.klay` reader (reference behaviour, tensorize.py:197-313)."""
    if isinstance(text, bytes):
        text = text.decode("ascii")
    rows = [ln.split() for ln in text.splitlines() if ln.split()]
    if not rows:
        raise KlayFormatError("empty file")
    pos = 0

    def nxt(want=None):
        nonlocal pos
        if pos >= len(rows):
            if want is None:
                return None
            raise KlayFormatError(f"unexpected end of file, wanted {want!r}")
        toks = rows[pos]
        pos += 1
        if want is not None and toks[0] != want:
            raise KlayFormatError(f"expected {want!r} line, got {toks[0]!r}")
        return toks

    try:
        head = nxt("klay")
        if len(head) != 2 or not head[1].isdigit():
            raise KlayFormatError("malformed version header")
        if int(head[1]) != KLAY_VERSION:
            raise KlayFormatError(f"unsupported format version {head[1]}")
        t = nxt("inputs")
        if len(t) != 2:
            raise KlayFormatError("malformed inputs line")
        num_inputs = int(t[1])
        t = nxt("vars")
        if len(t) != 2:
            raise KlayFormatError("malformed vars line")
        num_vars = int(t[1])
        roots = [int(x) for x in nxt("roots")[1:]]
        t = nxt()
        constants: dict[int, bool] = {}
        if t is not None and t[0] == "constants":
            for entry in t[1:]:
                p, _, b = entry.partition(":")
                if b not in ("0", "1"):
                    raise KlayFormatError(f"malformed constants entry {entry!r}")
                if int(p) in constants:
                    raise KlayFormatError(f"duplicate constant root position {p}")
                constants[int(p)] = b == "1"
            t = nxt()
        if t is None or t[0] != "inputmap":
            raise KlayFormatError("missing inputmap line")
        input_map: dict[Literal, int] = {}
        for entry in t[1:]:
            code, _, slot = entry.partition(":")
            try:
                lit = Literal.from_dimacs(int(code))
            except ValueError as exc:
                raise KlayFormatError(f"malformed inputmap entry {entry!r}") from exc
            if lit in input_map:
                raise KlayFormatError(f"duplicate literal in inputmap: {entry!r}")
            input_map[lit] = int(slot)
        layers = []
        t = nxt()
        while t is not None:
            if t[0] != "layer" or len(t) != 5:
                raise KlayFormatError(f"expected layer header, got {t!r}")
            idx, op, width, ne = int(t[1]), t[2], int(t[3]), int(t[4])
            if idx != len(layers) + 1:
                raise KlayFormatError(f"layer {idx} out of sequence")
            if op not in (PRODUCT, SUM):
                raise KlayFormatError(f"unknown layer op {op!r}")
            s, r = nxt("S"), nxt("R")
            if len(s) - 1 != ne or len(r) - 1 != ne:
                raise KlayFormatError(f"layer {idx}: edge count mismatch with header")
            layers.append(TensorLayer(op, width,
                                      np.array(s[1:], dtype=np.int64),
                                      np.array(r[1:], dtype=np.int64)))
            t = nxt()
        tc = TensorizedCircuit(num_inputs, num_vars, layers, input_map, roots, constants)
        validate(tc)
    except KlayFormatError:
        raise
    except Exception as exc:  # malformed ints surface as format errors
        raise KlayFormatError(str(exc)) from exc
    return tc


# --------------------------------------------------------------------------
# Binary .npz sidecar (compressed; used for the benchmark circuits)
# --------------------------------------------------------------------------

def save_npz(tc, path) -> None:
    widths = np.array([l.width for l in tc.layers], dtype=np.int64)
    counts = np.array([len(l.sources) for l in tc.layers], dtype=np.int64)
    src = (np.concatenate([np.asarray(l.sources) for l in tc.layers])
           if tc.layers else np.zeros(0))
    seg = (np.concatenate([np.asarray(l.segments) for l in tc.layers])
           if tc.layers else np.zeros(0))
    lits = sorted(tc.input_map.items(), key=lambda kv: kv[1])
    np.savez_compressed(
        path,
        header=np.array([tc.num_inputs, tc.num_vars], dtype=np.int64),
        widths=widths,
        counts=counts,
        sources=src.astype(np.int32),
        # segments are nondecreasing: store the per-parent fan-in instead
        fanin=np.concatenate([np.bincount(np.asarray(l.segments), minlength=l.width)
                              for l in tc.layers]).astype(np.int32)
        if tc.layers else np.zeros(0, np.int32),
        roots=np.asarray(tc.root_indices, dtype=np.int64),
        const_pos=np.array(sorted(tc.constant_roots), dtype=np.int64),
        const_val=np.array([int(tc.constant_roots[p]) for p in sorted(tc.constant_roots)],
                           dtype=np.int64),
        input_lits=np.array([_dimacs(k) for k, _ in lits], dtype=np.int64),
    )


def load_npz(path) -> TensorizedCircuit:
    z = np.load(path)
    num_inputs, num_vars = (int(x) for x in z["header"])
    widths, counts = z["widths"], z["counts"]
    src, fanin = z["sources"].astype(np.int64), z["fanin"]
    layers = []
    e0 = w0 = 0
    for l, (w, c) in enumerate(zip(widths.tolist(), counts.tolist()), start=1):
        seg = np.repeat(np.arange(w, dtype=np.int64), fanin[w0:w0 + w])
        layers.append(TensorLayer(PRODUCT if l % 2 == 1 else SUM, w, src[e0:e0 + c], seg))
        e0 += c
        w0 += w
    input_map = {Literal.from_dimacs(int(c)): i for i, c in enumerate(z["input_lits"])}
    constants = {int(p): bool(v) for p, v in zip(z["const_pos"], z["const_val"])}
    return TensorizedCircuit(num_inputs, num_vars, layers, input_map,
                             [int(r) for r in z["roots"]], constants)


def stats(tc) -> dict:
    """Node/edge counts (layerize.py:274-313, TensorizedCircuit branch)."""
    widths = [tc.num_inputs] + [l.width for l in tc.layers]
    edges = [len(l.sources) for l in tc.layers]
    dense = [widths[i] * widths[i + 1] for i in range(len(widths) - 1)]
    return {
        "nodes_total": int(sum(widths)),
        "nodes_per_layer": widths,
        "edges_total": int(sum(edges)),
        "edges_per_layer": edges,
        "sparsity": (sum(edges) / sum(dense)) if sum(dense) else None,
        "sparsity_per_layer": [e / d for e, d in zip(edges, dense)],
    }
