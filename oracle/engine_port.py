"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference evaluation engine
(``/root/reference/pkg/src/laycirc/engine.py``), used as the parity checker
for the CUDA path and as the reference arm / ``cpu_baseline`` of
``bench.py``. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``
may import it.

Parity is PINNED: ``tests/test_oracle.py`` checks this module against the
reference's committed golden dumps (``pkg/consumer/tests/fixtures/*.json``,
reproduced bit-exactly by the reference engine) and against the golden
vectors that ``tools/gen_golden.py`` produced by running the reference
engine itself in the build container.

Arithmetic lives in numpy's ufuncs exactly as in the reference, so results
are bit-identical to it (numpy 2.3.x; ``add.reduceat`` sums a segment as
``x0 + pairwise(x[1:])``, ``multiply.reduceat`` is sequential — SURVEY P1).
"""

from __future__ import annotations

import numpy as np

PRODUCT = "prod"


class OracleError(ValueError):
    pass


def _layer_plan(layer):
    """CSR starts of the parent segments and the transposed (child-major)
    edge order — ``engine.py:138-155``. The stable argsort keeps ascending
    edge order inside every child's group."""
    seg = np.asarray(layer.segments)
    src = np.asarray(layer.sources)
    fan = np.bincount(seg, minlength=layer.width)
    starts = np.concatenate(([0], np.cumsum(fan)[:-1])).astype(np.int64)
    order = np.argsort(src, kind="stable")
    nprev = int(src[order[-1]]) + 1 if len(src) else 0
    gfan = np.bincount(src[order], minlength=nprev)
    gstarts = np.concatenate(([0], np.cumsum(gfan)[:-1])).astype(np.int64)
    return starts, order, gstarts


def plans(tc):
    cache = getattr(tc, "_oracle_plans", None)
    if cache is None:
        cache = [_layer_plan(l) for l in tc.layers]
        try:
            tc._oracle_plans = cache
        except AttributeError:
            pass
    return cache


# ---- segment reductions per semiring (engine.py:169-193, 264-282) --------

def _lse(edge_vals, starts, seg, eps):
    """Max-trick segment logsumexp; all -inf segments stay -inf
    (engine.py:274-282)."""
    peak = np.maximum.reduceat(edge_vals, starts, axis=-1)
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        z = np.exp(edge_vals - peak[:, seg])
        z[np.isnan(z)] = 0.0
        res = np.log(np.add.reduceat(z, starts, axis=-1) + eps) + peak
    res[peak == -np.inf] = -np.inf
    return res


def _reducer(semiring, op, eps):
    prod = op == PRODUCT
    if semiring == "real":
        return (lambda e, s, g: np.multiply.reduceat(e, s, axis=-1)) if prod else \
               (lambda e, s, g: np.add.reduceat(e, s, axis=-1))
    if semiring == "log":
        return (lambda e, s, g: np.add.reduceat(e, s, axis=-1)) if prod else \
               (lambda e, s, g: _lse(e, s, g, eps))
    if semiring == "bool":
        return (lambda e, s, g: np.minimum.reduceat(e, s, axis=-1)) if prod else \
               (lambda e, s, g: np.maximum.reduceat(e, s, axis=-1))
    if semiring == "maxprod":
        return (lambda e, s, g: np.multiply.reduceat(e, s, axis=-1)) if prod else \
               (lambda e, s, g: np.maximum.reduceat(e, s, axis=-1))
    raise OracleError(f"unknown semiring {semiring!r}")


_IDENT = {"real": (0.0, 1.0), "log": (-np.inf, 0.0), "bool": (0.0, 1.0), "maxprod": (0.0, 1.0)}


def forward(tc, values, semiring="real", epsilon=0.0, retain=True):
    """Layer loop (engine.py:215-223) + root assembly (engine.py:203-212).

    ``values``: [B, K] array in the semiring's domain (log values for
    "log"); its dtype is the compute dtype. Returns (outputs [B, R],
    node_values list or None)."""
    if semiring == "log" and epsilon < 0:
        raise OracleError("epsilon must be >= 0")
    cur = np.asarray(values)
    trace = [cur] if retain else None
    for layer, (starts, _, _) in zip(tc.layers, plans(tc)):
        seg = np.asarray(layer.segments)
        edge_vals = cur[:, np.asarray(layer.sources)]
        cur = _reducer(semiring, layer.op, epsilon)(edge_vals, starts, seg)
        if retain:
            trace.append(cur)
    zero, one = _IDENT[semiring]
    out = np.empty((cur.shape[0], tc.num_roots), dtype=cur.dtype)
    free = [p for p in range(tc.num_roots) if p not in tc.constant_roots]
    for p, r in zip(free, tc.root_indices):
        out[:, p] = cur[:, r]
    for p, b in tc.constant_roots.items():
        out[:, p] = one if b else zero
    return out, trace


def _zero_safe_product_grad(edge_vals, g_parent, starts, seg):
    """engine.py:358-369: divide form when no zero edge exists anywhere;
    otherwise a single zero edge receives the nonzero sibling product and
    segments with two or more zeros propagate nothing."""
    is_zero = edge_vals == 0.0
    if not is_zero.any():
        p = np.multiply.reduceat(edge_vals, starts, axis=-1)
        return (g_parent * p)[:, seg] / edge_vals
    safe = np.where(is_zero, 1.0, edge_vals)
    pnz = np.multiply.reduceat(safe, starts, axis=-1)[:, seg]
    nz = np.add.reduceat(is_zero.astype(edge_vals.dtype), starts, axis=-1)[:, seg]
    g = g_parent[:, seg]
    one_zero = np.where((nz == 1) & is_zero, g * pnz, 0.0)
    return np.where(nz == 0, g * pnz / safe, one_zero)


def backward(tc, trace, domain, seed=None):
    """Reverse sweep of engine.py:307-355 over a retained trace."""
    if trace is None:
        raise OracleError("backward requires a retained trace")
    if len(trace) != len(tc.layers) + 1:
        raise OracleError("trace does not match circuit layer count")
    B = trace[0].shape[0]
    dt = trace[0].dtype
    seed = np.ones((B, tc.num_roots), dt) if seed is None else np.asarray(seed, dt)
    if seed.shape != (B, tc.num_roots):
        raise OracleError(f"seed must have shape {(B, tc.num_roots)}")
    top = tc.layers[-1].width if tc.layers else tc.num_inputs
    g = np.zeros((B, top), dt)
    free = [p for p in range(tc.num_roots) if p not in tc.constant_roots]
    for p, r in zip(free, tc.root_indices):
        g[:, r] += seed[:, p]
    pl = plans(tc)
    for l in range(len(tc.layers) - 1, -1, -1):
        layer = tc.layers[l]
        starts, order, gstarts = pl[l]
        seg = np.asarray(layer.segments)
        src = np.asarray(layer.sources)
        if domain == "real" and layer.op == PRODUCT:
            ge = _zero_safe_product_grad(trace[l][:, src], g, starts, seg)
        elif domain == "log" and layer.op != PRODUCT:
            with np.errstate(invalid="ignore"):
                w = np.exp(trace[l][:, src] - trace[l + 1][:, seg])
            w[~np.isfinite(w)] = 0.0
            ge = g[:, seg] * w
        else:  # log products and real sums pass the parent adjoint through
            ge = g[:, seg]
        g = np.add.reduceat(ge[:, order], gstarts, axis=-1)
    return g
