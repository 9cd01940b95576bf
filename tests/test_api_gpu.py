"""Drop-in API behaviour around the device path: gradient()'s pass cache
(bounded, thread-safe), caller-buffer validation of DevicePlan, and
evaluate_semiring with semiring objects (the reference's own included)."""

import threading

import numpy as np
import pytest

from conftest import load_case, load_config, rel_close

pytestmark = pytest.mark.gpu


def test_gradient_cache_keeps_one_pass_per_circuit(cuda):
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import engine
    tc, _ = load_case("corpus_5")
    engine.clear_cache()
    rng = np.random.default_rng(3)
    for B in (3, 8, 5):
        w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
        out, g = engine.gradient(tc, engine.WeightAssignment(w), log_domain=True)
        ref_out, tr = oracle.forward(tc, np.log(w), "log")
        rel_close(out, ref_out, 1e-12)
        rel_close(g, oracle.backward(tc, tr, "log"), 1e-12, 1e-12)
        assert engine.cached_passes() == 1
    tc2, _ = load_case("fig_main")
    engine.gradient(tc2, engine.WeightAssignment(rng.uniform(0.1, 0.9, (2, tc2.num_inputs))))
    assert engine.cached_passes() == 2  # one per circuit
    engine.clear_cache()
    assert engine.cached_passes() == 0


def test_gradient_is_thread_safe(cuda):
    """Threads calling gradient() on one circuit and batch size get their own
    results (the captured pass's pinned buffers are shared: per-plan lock)."""
    import torch

    from paper_2410_11415_b200 import engine
    tc, _ = load_case("corpus_5")
    rng = np.random.default_rng(4)
    ws = [rng.uniform(0.05, 0.95, size=(6, tc.num_inputs)) for _ in range(8)]
    expect = [engine.gradient(tc, engine.WeightAssignment(w)) for w in ws]
    got = [None] * len(ws)
    errors = []

    def worker(i):
        try:
            torch.cuda.set_device(cuda)
            for _ in range(10):
                got[i] = engine.gradient(tc, engine.WeightAssignment(ws[i]))
                assert np.array_equal(got[i][0], expect[i][0])
                assert np.array_equal(got[i][1], expect[i][1])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(ws))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    engine.clear_cache()


def test_device_plan_rejects_bad_buffers(cuda):
    import torch

    from paper_2410_11415_b200 import _lib, engine
    tc, _ = load_case("corpus_5")
    plan = engine.device_plan(tc, cuda)
    B = 4
    w = torch.zeros((B, tc.num_inputs), dtype=torch.float32, device=cuda)
    small = plan.alloc_values(B, np.float32, retain=False)
    if small.shape[0] < plan.num_nodes:
        with pytest.raises(engine.EvalError, match="rows"):
            plan.forward(w, _lib.KLAY_LOG, np.float32, retain=True, values=small)
    with pytest.raises(engine.EvalError, match="dtype"):
        plan.forward(w, _lib.KLAY_LOG, np.float32, values=plan.alloc_values(B, np.float64))
    with pytest.raises(engine.EvalError, match="cpu"):
        plan.forward(w.cpu(), _lib.KLAY_LOG, np.float32)
    with pytest.raises(engine.EvalError, match="shape"):
        plan.forward(w, _lib.KLAY_LOG, np.float32,
                     outputs=torch.empty((B + 1, tc.num_roots), device=cuda))
    out, vals = plan.forward(w, _lib.KLAY_LOG, np.float32)
    with pytest.raises(engine.EvalError, match="bytes"):
        plan.backward(vals, B, _lib.KLAY_LOG, np.float32,
                      workspace=torch.empty(16, dtype=torch.uint8, device=cuda))
    with pytest.raises(engine.EvalError, match="shape"):
        plan.backward(vals, B, _lib.KLAY_LOG, np.float32,
                      grads=torch.empty((B, tc.num_inputs + 1), device=cuda))
    if small.shape[0] < plan.num_nodes:
        with pytest.raises(engine.EvalError, match="rows"):
            plan.backward(small, B, _lib.KLAY_LOG, np.float32)
    # a correctly sized caller buffer set still works
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float32,
                      workspace=plan.workspace(B, np.float32))
    assert g.shape == (B, tc.num_inputs)


def test_evaluate_semiring_accepts_semiring_objects(cuda):
    from dataclasses import dataclass

    from paper_2410_11415_b200 import engine
    tc, gold = load_case("fig_pair_merge")

    @dataclass(frozen=True)
    class ForeignSemiring:  # shaped like the reference's laycirc.engine.Semiring
        name: str
        zero: float
        one: float
        reduce_sum: object = None
        reduce_prod: object = None

    w = engine.WeightAssignment(gold["w_real"])
    for name in ("real", "bool", "maxprod"):
        ref = engine.evaluate_semiring(tc, w, name)
        got = engine.evaluate_semiring(tc, w, ForeignSemiring(name, 0.0, 1.0))
        assert np.array_equal(got, ref)
        assert np.array_equal(engine.evaluate_semiring(tc, w, engine.SEMIRINGS[name]), ref)
    with pytest.raises(engine.EvalError, match="unsupported semiring"):
        engine.evaluate_semiring(tc, w, ForeignSemiring("tropical", float("inf"), 0.0))
    with pytest.raises(engine.EvalError, match="identities"):
        engine.evaluate_semiring(tc, w, ForeignSemiring("real", 1.0, 0.0))


def test_backward_workspace_shares_rows_between_layers(cuda):
    """Adjoint rows of node layers with disjoint lifetimes share memory
    (klay.cu assign_adjoint_blocks). Config C' (no unary chains: every
    adjoint block lives two steps) needs 5 % of the trace's rows; config C's
    adjoint routes keep layers live for up to ~10 steps, which bounds any
    layer-granular layout at 0.786 of the trace: the plan
    gets within 5 % of that bound."""
    from paper_2410_11415_b200 import engine
    for name, bound in (("Cp", 0.06), ("C", 0.786 * 1.05)):
        tc, _ = load_config(name)
        plan = engine.device_plan(tc, cuda)
        rows = plan.schedule["adjoint_rows"]
        assert rows <= bound * plan.num_nodes, (name, rows / plan.num_nodes)
        ld = plan.row_stride(1024, np.float32)
        work = int(plan._lib.klay_backward_workspace(plan.handle, 0, ld))
        assert work < plan.num_nodes * ld * 4
