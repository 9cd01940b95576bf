"""Random layered circuits (tensorized directly, every invariant of
tensorize.py:94-132 respected) against the CPU oracle: many unary nodes and
single-parent children (aliases, multi-layer adjoint routes), shared
children, heavy fan-ins (> 129 edges: split leaves), zero weights (-inf log
values). Real fp64: bit-exact; log fp64: rel 1e-12."""

import numpy as np
import pytest

from conftest import fp32_close, rel_close

pytestmark = pytest.mark.gpu


def random_circuit(seed, K=24, L=9, wmax=60, grow=1):
    from paper_2410_11415_b200.tensorized import Literal, TensorizedCircuit, TensorLayer, validate
    rng = np.random.default_rng(seed)
    layers = []
    prev = K
    for l in range(L):
        op = "prod" if l % 2 == 0 else "sum"
        W = int(rng.integers(max(1, prev // 3), max(2, min(wmax, grow * prev + 8))))
        W = max(1, min(W, prev)) if l == L - 1 else W
        # every previous node feeds some parent; extra edges give fan-in > 1
        owner = rng.integers(0, W, size=prev)
        segs = [[] for _ in range(W)]
        for c, p in enumerate(owner):
            segs[p].append(c)
        for p in range(W):
            r = rng.random()
            extra = 0 if r < 0.45 else (int(rng.integers(1, 4)) if r < 0.97 else int(rng.integers(130, 300)))
            if extra:
                segs[p].extend(rng.integers(0, prev, size=extra).tolist())
            if not segs[p]:
                segs[p].append(int(rng.integers(0, prev)))
        src = np.array([c for p in range(W) for c in segs[p]], np.int64)
        seg = np.array([p for p in range(W) for _ in segs[p]], np.int64)
        layers.append(TensorLayer(op, W, src, seg))
        prev = W
    input_map = {Literal(v, pos): 2 * (v - 1) + (0 if pos else 1)
                 for v in range(1, K // 2 + 1) for pos in (True, False)}
    roots = sorted(set(rng.integers(0, prev, size=min(prev, 4)).tolist()))
    tc = TensorizedCircuit(K, K // 2, layers, input_map, roots, {})
    validate(tc)
    return tc


@pytest.mark.parametrize("seed", range(24))
def test_random_circuits_match_oracle(cuda, seed):
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    tc = random_circuit(seed)
    plan = device_plan(tc)
    rng = np.random.default_rng(100 + seed)
    B = (37, 1, 64, 5)[seed % 4]
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    w[rng.uniform(size=w.shape) < 0.04] = 0.0
    # real fp64: bit-exact values and gradients (odd seeds: signed weights)
    wr = w * rng.choice([-2.0, 1.5], size=w.shape) if seed % 2 else w
    x = torch.tensor(wr, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_REAL, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_REAL, np.float64)
    ref, tr = oracle.forward(tc, wr, "real")
    assert np.array_equal(out.cpu().numpy(), ref, equal_nan=True)
    np.testing.assert_array_equal(g.cpu().numpy(), oracle.backward(tc, tr, "real"))
    # log fp64 (aliases and routes on: epsilon 0, backward-only trace)
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    with np.errstate(all="ignore"):
        ref, tr = oracle.forward(tc, lw, "log")
        gref = oracle.backward(tc, tr, "log")
    rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
    rel_close(g.cpu().numpy(), gref, 1e-12, 1e-12)
    from paper_2410_11415_b200.engine import _NodeValues
    nv = _NodeValues(plan, vals, B)
    for l in range(len(tr)):
        rel_close(nv[l], tr[l], 1e-12, 1e-12)


def sweep_case(seed):
    """tools/fuzz_sweep.py's case for a seed: a random shape, then (circuit,
    batch, weights in (0.05, 0.95) with 4 % zeros), or None when the shape
    is too narrow to draw."""
    rng = np.random.default_rng(seed)
    K = int(rng.integers(4, 120)) * 2
    L = int(rng.integers(2, 16))
    try:
        tc = random_circuit(seed, K=K, L=L, wmax=int(rng.integers(8, 3000)), grow=int(rng.integers(1, 4)))
    except ValueError:
        return None
    B = int(rng.integers(1, 300))
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    w[rng.uniform(size=w.shape) < 0.04] = 0.0
    return tc, B, w


@pytest.mark.parametrize("seed", [52093, 52235, 52249, 52294])
def test_route_masks_odd_row_widths(cuda, seed):
    """Adjoint routes read the finiteness masks the forward leaves per
    512-byte column chunk. Row widths that are not a multiple of two chunks
    (these sweep seeds: fp64 B = 172, 141, 274, 293) once broke the streaming
    kernel's mask layout (stream_kernels.cuh stream_threads); test_stream_gpu
    runs this under KLAY_STREAM=1 too. Log fp64, backward-only trace."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    tc, B, w = sweep_case(seed)
    plan = device_plan(tc)
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    with np.errstate(all="ignore"):
        ref, tr = oracle.forward(tc, lw, "log")
        gref = oracle.backward(tc, tr, "log")
    assert plan.schedule["aliased_rows"] > 0 and (B * 8 // 16) % 64
    rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
    rel_close(g.cpu().numpy(), gref, 1e-12, 1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_random_wide_circuits_all_semirings(cuda, seed):
    """Wider random circuits (regular layer kernels, aliases and routes at the
    default tail): fp32 real bit-exact vs the reference's own fp32 run, fp32 log
    elementwise within max(1e-5 rel, 2x the reference's own fp32 error) of fp64, Boolean (bit-packed) and max-product bit-exact,
    seeded backward."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan, engine
    tc = random_circuit(1000 + seed, K=40, L=11, wmax=700, grow=3)
    plan = device_plan(tc)
    rng = np.random.default_rng(7 + seed)
    B = (1, 45, 130, 33)[seed % 4]
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    w[rng.uniform(size=w.shape) < 0.03] = 0.0
    # fp32 real, seeded backward: bit-exact vs the oracle in fp32
    w32 = w.astype(np.float32)
    seed_m = rng.uniform(-1, 1, size=(B, tc.num_roots)).astype(np.float32)
    x = torch.tensor(w32, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_REAL, np.float32)
    g = plan.backward(vals, B, _lib.KLAY_REAL, np.float32, seed=torch.tensor(seed_m, device=cuda))
    ref, tr = oracle.forward(tc, w32, "real")
    assert np.array_equal(out.cpu().numpy(), ref, equal_nan=True)
    np.testing.assert_array_equal(g.cpu().numpy(), oracle.backward(tc, tr, "real", seed_m))
    # fp32 log vs the fp64 oracle
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw.astype(np.float32), device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float32)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float32)
    with np.errstate(all="ignore"):
        ref, tr = oracle.forward(tc, lw, "log")
        gref = oracle.backward(tc, tr, "log")
        ref32, tr32 = oracle.forward(tc, lw.astype(np.float32), "log")  # the reference's own fp32 run
        gref32 = oracle.backward(tc, tr32, "log")
    fp32_close(out.cpu().numpy(), ref, ref32)
    fp32_close(g.cpu().numpy(), gref, gref32)
    # Boolean on 0/1 inputs (bit-packed path) and max-product: bit-exact
    wb = (rng.uniform(size=w.shape) < 0.6).astype(np.float64)
    ref, _ = oracle.forward(tc, wb, "bool", retain=False)
    got = engine.evaluate_semiring(tc, engine.WeightAssignment(wb), "bool")
    assert np.array_equal(got, ref)
    ref, _ = oracle.forward(tc, w, "maxprod", retain=False)
    got = engine.evaluate_semiring(tc, engine.WeightAssignment(w), "maxprod")
    assert np.array_equal(got, ref)


def fanin_circuit(seed, K=64, L=8, W=48, fmax=110):
    """Every sum node draws its fan-in from 1..fmax, every product node from
    1..3 (children with repetition allowed, each previous node read at least
    once; values stay finite): numpy's 8-accumulator pairwise order inside
    the micro tails (fan-in and fan-out 9..129)."""
    from paper_2410_11415_b200.tensorized import Literal, TensorizedCircuit, TensorLayer, validate
    rng = np.random.default_rng(seed)
    layers, prev = [], K
    for l in range(L):
        w = W if l < L - 1 else 2
        f = 3 if l % 2 == 0 else fmax
        segs = [rng.integers(0, prev, size=int(rng.integers(1, f + 1))).tolist() for _ in range(w)]
        for c in range(prev):  # every child read
            segs[int(rng.integers(0, w))].append(c)
        src = np.array([c for s in segs for c in s], np.int64)
        seg = np.array([p for p, s in enumerate(segs) for _ in s], np.int64)
        layers.append(TensorLayer("prod" if l % 2 == 0 else "sum", w, src, seg))
        prev = w
    input_map = {Literal(v, pos): 2 * (v - 1) + (0 if pos else 1)
                 for v in range(1, K // 2 + 1) for pos in (True, False)}
    tc = TensorizedCircuit(K, K // 2, layers, input_map, [0, 1], {})
    validate(tc)
    return tc


@pytest.mark.parametrize("seed", range(6))
def test_micro_tail_pairwise_fanin(cuda, seed):
    """Fan-ins and fan-outs up to 129 inside the micro tails: real fp64
    values and gradients bit-exact (x0 + numpy pairwise of the rest), log
    fp64 within 1e-12."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    tc = fanin_circuit(300 + seed)
    assert max(np.bincount(l.segments).max() for l in tc.layers) > 64
    assert max(np.bincount(l.sources).max() for l in tc.layers) > 32
    plan = device_plan(tc)
    assert plan.schedule["micro"] == 0 and plan.schedule["micro_bwd"] == 0
    rng = np.random.default_rng(seed)
    B = (1, 7, 64)[seed % 3]
    w = rng.uniform(0.05, 0.15, size=(B, tc.num_inputs)) * rng.choice([-1.0, 1.0], size=(B, tc.num_inputs))
    x = torch.tensor(w, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_REAL, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_REAL, np.float64)
    ref, tr = oracle.forward(tc, w, "real")
    assert np.array_equal(out.cpu().numpy(), ref, equal_nan=True)
    np.testing.assert_array_equal(g.cpu().numpy(), oracle.backward(tc, tr, "real"))
    lw = np.log(np.abs(w))
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    ref, tr = oracle.forward(tc, lw, "log")
    rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
    rel_close(g.cpu().numpy(), oracle.backward(tc, tr, "log"), 1e-12, 1e-12)


def head_circuit(seed, K=48, W=40):
    """Thin bottom layers (micro heads); layers 4 and 9 with a 300-edge
    segment and a 140-parent child (layer kernels, heavy leaves) around
    aliased layers; thin layers above (persistent / micro tails)."""
    from paper_2410_11415_b200.tensorized import Literal, TensorizedCircuit, TensorLayer, validate
    rng = np.random.default_rng(seed)
    layers, prev = [], K
    for l in range(13):
        w = 2 if l == 12 else W
        segs = [rng.integers(0, prev, size=int(rng.integers(1, 4))).tolist() for _ in range(w)]
        if l in (4, 9):  # a 300-edge segment and a child read 140 times
            segs[0].extend(rng.integers(0, prev, size=300).tolist())
            segs[1].extend([0] * 140)
        for c in range(prev):
            segs[int(rng.integers(0, w))].append(c)
        src = np.array([c for s in segs for c in s], np.int64)
        seg = np.array([p for p, s in enumerate(segs) for _ in s], np.int64)
        layers.append(TensorLayer("prod" if l % 2 == 0 else "sum", w, src, seg))
        prev = w
    input_map = {Literal(v, pos): 2 * (v - 1) + (0 if pos else 1)
                 for v in range(1, K // 2 + 1) for pos in (True, False)}
    tc = TensorizedCircuit(K, K // 2, layers, input_map, [0, 1], {})
    validate(tc)
    return tc


@pytest.mark.parametrize("seed", range(4))
def test_micro_heads(cuda, seed):
    """Micro heads below layer kernels below a micro tail: real fp64
    bit-exact, log fp64 within 1e-12 (values, gradients, every trace layer of
    a backward-only trace, so aliases start above the heads)."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    from paper_2410_11415_b200.engine import _NodeValues
    tc = head_circuit(500 + seed)
    plan = device_plan(tc)
    assert plan.schedule["head"] >= 2 and plan.schedule["head_bwd"] >= 2
    # no trace (ping-pong rows): every semiring through heads and tails
    from paper_2410_11415_b200 import engine
    rs = np.random.default_rng(50 + seed)
    wr = rs.uniform(0.05, 0.95, size=(9, tc.num_inputs))
    wb = (rs.uniform(size=wr.shape) < 0.6).astype(np.float64)
    for sr, ww in (("real", wr), ("maxprod", wr), ("bool", wb)):
        ref, _ = oracle.forward(tc, ww, sr, retain=False)
        assert np.array_equal(engine.evaluate_semiring(tc, engine.WeightAssignment(ww), sr), ref), sr
    rng = np.random.default_rng(seed)
    B = (1, 33, 128, 5)[seed]
    w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
    w[rng.uniform(size=w.shape) < 0.05] = 0.0
    x = torch.tensor(w, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_REAL, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_REAL, np.float64)
    ref, tr = oracle.forward(tc, w, "real")
    assert np.array_equal(out.cpu().numpy(), ref, equal_nan=True)
    np.testing.assert_array_equal(g.cpu().numpy(), oracle.backward(tc, tr, "real"))
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    with np.errstate(all="ignore"):
        ref, tr = oracle.forward(tc, lw, "log")
        gref = oracle.backward(tc, tr, "log")
    rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
    rel_close(g.cpu().numpy(), gref, 1e-12, 1e-12)
    nv = _NodeValues(plan, vals, B)
    for l in range(len(tr)):
        rel_close(nv[l], tr[l], 1e-12, 1e-12)
