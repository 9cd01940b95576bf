"""Fast host-side layerize + tensorize.

``layerize_tensorize(circuits)`` returns the same TensorizedCircuit as the
reference's ``tensorize(layerize(circuits))`` (laycirc/layerize.py:158-271,
tensorize.py:135-194) -- identical widths, sources, segments, input map and
roots -- computed by the C++ restatement in ``libklay.so``
(csrc/layerize.cpp). Circuits are duck-typed like the reference's
``Circuit``: ``.nodes`` (kind, literal, children), ``.roots``, ``.num_vars``;
they must be constant-folded (``fold_constants``) as for the reference.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .tensorized import PRODUCT, SUM, Literal, TensorizedCircuit, TensorLayer, validate

_KINDS = {"leaf": 0, "and": 1, "or": 2, "true": 3, "false": 4}


class CircuitError(ValueError):
    """Malformed circuit for layerization (circuit.py:25-26)."""


def _flatten(circuits):
    kinds, lits, coff, kids, roots = [], [], [0], [], []
    node_off, root_off, nvars = [0], [0], []
    for c in circuits:
        for node in c.nodes:
            kind, literal, children = node[0], node[1], node[2]
            kinds.append(_KINDS[kind])
            lits.append(int(literal.to_dimacs()) if literal is not None else 0)
            kids.extend(children)
            coff.append(len(kids))
        node_off.append(len(kinds))
        roots.extend(c.roots)
        root_off.append(len(roots))
        nvars.append(int(c.num_vars))
    as_ = np.ascontiguousarray
    return (as_(np.array(node_off, np.int64)), as_(np.array(kinds, np.int8)),
            as_(np.array(lits, np.int32)), as_(np.array(coff, np.int64)),
            as_(np.array(kids if kids else [0], np.int32)), as_(np.array(root_off, np.int64)),
            as_(np.array(roots if roots else [0], np.int32)), as_(np.array(nvars, np.int32)))


def layerize_tensorize(circuits) -> TensorizedCircuit:
    """tensorize(layerize(circuits)) of the reference, in C++."""
    circuits = list(circuits)
    lib = _lib.load()
    if not circuits:
        raise CircuitError("layerize requires at least one circuit")
    node_off, kinds, lits, coff, kids, root_off, roots, nvars = _flatten(circuits)
    h = ctypes.c_void_p()
    rc = lib.klay_layerize(len(circuits), node_off.ctypes.data, kinds.ctypes.data, lits.ctypes.data,
                           coff.ctypes.data, kids.ctypes.data, root_off.ctypes.data,
                           roots.ctypes.data, nvars.ctypes.data, ctypes.byref(h))
    if rc != _lib.KLAY_OK:
        raise CircuitError(lib.klay_layerize_error().decode())
    try:
        info = [int(lib.klay_layered_info(h, i)) for i in range(6)]
        K, V, L, E, R, C = info
        widths = np.empty(max(L, 1), np.int64)
        counts = np.empty(max(L, 1), np.int64)
        src = np.empty(max(E, 1), np.int64)
        seg = np.empty(max(E, 1), np.int64)
        ilits = np.empty(max(K, 1), np.int32)
        rix = np.empty(max(R, 1), np.int64)
        cpos = np.empty(max(C, 1), np.int64)
        cval = np.empty(max(C, 1), np.int8)
        lib.klay_layered_export(h, widths.ctypes.data, counts.ctypes.data, src.ctypes.data,
                                seg.ctypes.data, ilits.ctypes.data, rix.ctypes.data,
                                cpos.ctypes.data, cval.ctypes.data)
    finally:
        lib.klay_layered_destroy(h)
    layers = []
    e0 = 0
    for l in range(L):
        n = int(counts[l])
        layers.append(TensorLayer(PRODUCT if l % 2 == 0 else SUM, int(widths[l]),
                                  src[e0:e0 + n].copy(), seg[e0:e0 + n].copy()))
        e0 += n
    tc = TensorizedCircuit(
        num_inputs=K, num_vars=V, layers=layers,
        input_map={Literal.from_dimacs(int(code)): i for i, code in enumerate(ilits[:K])},
        root_indices=[int(r) for r in rix[:R]],
        constant_roots={int(p): bool(v) for p, v in zip(cpos[:C], cval[:C])})
    validate(tc)
    return tc
