"""Parity of the CUDA path (through libklay.so) with the reference.

Tolerances (north star): Boolean / max-product outputs and real-semiring
fp64 results are compared bit-exactly (the kernels reproduce numpy's
summation order); log-semiring fp64 values and gradients within
rel 1e-12; fp32 log values and gradients elementwise within
max(1e-5 * |ref64|, 2 * |ref32 - ref64|) of the fp64 reference, ref32 being
the reference's own fp32 run (conftest.fp32_close): every entry, however
small, is held to the north star's rel 1e-5 or to the reference's own fp32
error at that entry.
"""

import math
import os

import numpy as np
import pytest

from conftest import (CONFIGS, CONSUMER_DUMPS, SMALL_CASES, consumer_case, fp32_close, load_case,
                      load_config, rel_close)

pytestmark = pytest.mark.gpu


def _engine():
    import paper_2410_11415_b200 as k
    return k


# ---------------------------------------------------------------------------
# the reference's committed golden dumps (criterion 9 of the consumer suite)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dump", sorted(CONSUMER_DUMPS))
def test_consumer_dumps(cuda, dump):
    k = _engine()
    tc, w, roots, grad, log, eps = consumer_case(dump)
    if log:
        tr = k.forward_log(tc, w.to_log(), epsilon=eps)
        rel_close(tr.outputs, roots, 1e-12)
    else:
        tr = k.forward_real(tc, w)
        assert np.array_equal(tr.outputs, roots)
        if grad is None:
            assert np.array_equal(k.evaluate_semiring(tc, w, "real"), roots)
    if grad is not None:
        g = k.backward(tc, tr)
        if log:
            rel_close(g, grad, 1e-12)
        else:
            assert np.array_equal(g, grad)


# ---------------------------------------------------------------------------
# golden suites: small circuits (all edge cases) and configs A-D (8 rows)
# ---------------------------------------------------------------------------

def _suite(tc, gold):
    k = _engine()
    W = k.WeightAssignment(gold["w_real"])
    L = W.to_log()
    # real fp64: bit-exact
    tr = k.forward_real(tc, W)
    assert np.array_equal(tr.outputs, gold["real_out"], equal_nan=True)
    np.testing.assert_array_equal(k.backward(tc, tr), gold["real_grad"])
    np.testing.assert_array_equal(k.backward(tc, tr, gold["seed"]), gold["real_grad_seed"])
    # real fp32: bit-exact vs the reference's own fp32 run
    tr32 = k.forward_real(tc, W, dtype=np.float32)
    assert tr32.outputs.dtype == np.float32
    np.testing.assert_array_equal(tr32.outputs, gold["real32_out"])
    np.testing.assert_array_equal(k.backward(tc, tr32), gold["real32_grad"])
    # log fp64: rel 1e-12
    tr = k.forward_log(tc, L)
    rel_close(tr.outputs, gold["log_out"], 1e-12)
    rel_close(k.backward(tc, tr), gold["log_grad"], 1e-12, 1e-12)
    rel_close(k.backward(tc, tr, gold["seed"]), gold["log_grad_seed"], 1e-12, 1e-12)
    tr = k.forward_log(tc, L, epsilon=1e-3)
    rel_close(tr.outputs, gold["logeps_out"], 1e-12)
    rel_close(k.backward(tc, tr), gold["logeps_grad"], 1e-12, 1e-12)
    # log fp32 vs the fp64 reference, elementwise (fp32_close)
    tr32 = k.forward_log(tc, L, dtype=np.float32)
    fp32_close(tr32.outputs, gold["log_out"], gold["log32_out"])
    fp32_close(k.backward(tc, tr32), gold["log_grad"], gold["log32_grad"])
    # Boolean / max-product: bit-exact
    bo = k.evaluate_semiring(tc, k.WeightAssignment(gold["w_bool"]), "bool")
    np.testing.assert_array_equal(bo, gold["bool_out"])
    np.testing.assert_array_equal(k.evaluate_semiring(tc, W, "maxprod"), gold["maxprod_out"])
    np.testing.assert_array_equal(k.evaluate_semiring(tc, W, k.MAX_PRODUCT), gold["maxprod_out"])
    # forward-only log matches the retained path
    rel_close(k.evaluate_semiring(tc, W, "log"), gold["log_out"], 1e-12)


@pytest.mark.parametrize("name", SMALL_CASES)
def test_golden_small(cuda, name):
    tc, gold = load_case(name)
    with np.errstate(all="ignore"):
        _suite(tc, gold)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_golden_configs(cuda, cfg):
    tc, gold = load_config(cfg)
    with np.errstate(all="ignore"):
        _suite(tc, gold)


# ---------------------------------------------------------------------------
# full-size properties (config C, B = 1024 fp32 as benchmarked)
# ---------------------------------------------------------------------------

def test_config_c_full_batch_rows_match_golden(cuda):
    """The golden rows embedded in a full 1024-row batch at fp32: row
    independence + parity at the benchmarked size; repeat bit-identical."""
    import torch
    k = _engine()
    tc, gold = load_config("C")
    rng = np.random.Generator(np.random.Philox(key=0))
    w = rng.uniform(0.05, 0.95, size=(1024, tc.num_inputs))
    w[100:108] = gold["w_real"]
    L = k.WeightAssignment(w).to_log()
    tr = k.forward_log(tc, L, dtype=np.float32)
    g = k.backward(tc, tr)
    fp32_close(tr.outputs[100:108], gold["log_out"], gold["log32_out"])
    fp32_close(g[100:108], gold["log_grad"], gold["log32_grad"])
    tr2 = k.forward_log(tc, L, dtype=np.float32)
    assert np.array_equal(tr.outputs, tr2.outputs)
    assert np.array_equal(g, k.backward(tc, tr2))
    # permutation equivariance
    perm = rng.permutation(1024)
    trp = k.forward_log(tc, k.WeightAssignment(L.values[perm], "log"), dtype=np.float32)
    assert np.array_equal(trp.outputs, tr.outputs[perm])
    assert np.array_equal(k.backward(tc, trp), g[perm])
    # exp(log) ~= real (criterion 4): same circuit, same rows, fp64
    real = k.forward_real(tc, k.WeightAssignment(w[:64]), retain_trace=False).outputs
    logv = k.forward_log(tc, k.WeightAssignment(w[:64]).to_log(), retain_trace=False).outputs
    rel_close(np.exp(logv), real, 1e-9)
    torch.cuda.synchronize()


def test_config_d_bool_bit_exact_at_4096(cuda):
    """Config D (256 roots), B = 4096 Boolean rows: bit-exact vs the oracle
    on a row subset, and all 0/1."""
    from oracle import engine_port as oracle
    k = _engine()
    tc, _ = load_config("D")
    rng = np.random.Generator(np.random.Philox(key=3))
    wb = rng.integers(0, 2, size=(4096, tc.num_inputs)).astype(np.float64)
    out = k.evaluate_semiring(tc, k.WeightAssignment(wb), "bool")
    assert out.shape == (4096, tc.num_roots)
    assert set(np.unique(out)) <= {0.0, 1.0}
    sub = slice(1000, 1064)
    ref, _ = oracle.forward(tc, wb[sub], "bool", retain=False)
    assert np.array_equal(out[sub], ref)
    real = k.evaluate_semiring(tc, k.WeightAssignment(wb[sub] * 0.5 + 0.25), "real")
    ref, _ = oracle.forward(tc, wb[sub] * 0.5 + 0.25, "real", retain=False)
    assert np.array_equal(real, ref)


# ---------------------------------------------------------------------------
# mirrors of the reference's engine tests (test_engine.py)
# ---------------------------------------------------------------------------

def _fig():
    return load_case("fig_main")[0]


def _half(tc):
    k = _engine()
    return k.WeightAssignment(np.full((1, tc.num_inputs), 0.5))


def test_figure_at_uniform_half(cuda):
    k = _engine()
    tc = _fig()
    out = k.forward_real(tc, _half(tc), retain_trace=False).outputs
    assert out[0, 0] == pytest.approx(0.8125, abs=1e-15)
    out = k.forward_log(tc, _half(tc).to_log()).outputs
    assert out[0, 0] == pytest.approx(math.log(0.8125), rel=1e-12)
    assert k.evaluate_semiring(tc, _half(tc), "maxprod")[0, 0] == pytest.approx(0.25)


def test_trace_has_one_matrix_per_layer(cuda):
    k = _engine()
    tc = _fig()
    trace = k.forward_real(tc, _half(tc))
    assert len(trace.node_values) == tc.num_layers + 1
    assert [m.shape[1] for m in trace.node_values] == [tc.num_inputs] + [l.width for l in tc.layers]
    from oracle import engine_port as oracle
    _, ref = oracle.forward(tc, _half(tc).values, "real")
    for a, b in zip(trace.node_values, ref):
        assert np.array_equal(a, b)


def test_errors_map_to_eval_error(cuda):
    k = _engine()
    tc = _fig()
    with pytest.raises(k.EvalError):
        k.forward_real(tc, k.WeightAssignment(np.ones((1, 3))))
    with pytest.raises(k.EvalError):
        k.forward_real(tc, _half(tc).to_log())
    with pytest.raises(k.EvalError):
        k.forward_log(tc, _half(tc))
    with pytest.raises(k.EvalError):
        k.forward_log(tc, _half(tc).to_log(), epsilon=-1.0)
    with pytest.raises(k.EvalError):
        k.evaluate_semiring(tc, _half(tc), "tropical")
    trace = k.forward_real(tc, _half(tc), retain_trace=False)
    assert trace.node_values is None
    with pytest.raises(k.EvalError):
        k.backward(tc, trace)
    trace = k.forward_real(tc, _half(tc))
    with pytest.raises(k.EvalError):
        k.backward(tc, trace, seed=np.ones((1, 5)))
    with pytest.raises(k.EvalError):
        k.WeightAssignment(np.array([[np.inf]]))


def test_all_minus_inf_segment_yields_minus_inf(cuda):
    k = _engine()
    tc, _ = load_case("dup_child")
    w = k.WeightAssignment(np.zeros((1, tc.num_inputs))).to_log()
    for eps in (0.0, 1e-8):
        for dt in (np.float64, np.float32):
            tr = k.forward_log(tc, w, epsilon=eps, dtype=dt)
            assert tr.outputs[0, 0] == -math.inf
            g = k.backward(tc, tr)
            assert not np.isnan(g).any()


def test_backward_accepts_host_trace(cuda):
    """A host-side trace (e.g. a reference EvalTrace) is uploaded and used."""
    from oracle import engine_port as oracle
    k = _engine()
    tc, gold = load_case("corpus_3")
    out, nv = oracle.forward(tc, np.log(gold["w_real"][:1]), "log")
    host = k.EvalTrace("log", out, nv)
    rel_close(k.backward(tc, host), gold["log_grad"][:1], 1e-12, 1e-12)


def test_batch_one_and_odd_batches(cuda):
    from oracle import engine_port as oracle
    k = _engine()
    tc, gold = load_case("corpus_5")
    rng = np.random.default_rng(5)
    for B in (1, 3, 5, 129, 257):
        w = rng.uniform(0.05, 0.95, size=(B, tc.num_inputs))
        tr = k.forward_real(tc, k.WeightAssignment(w))
        ref, rtr = oracle.forward(tc, w, "real")
        assert np.array_equal(tr.outputs, ref)
        assert np.array_equal(k.backward(tc, tr), oracle.backward(tc, rtr, "real"))


def test_captured_graph_pass_matches_stream_path(cuda):
    """DevicePlan.capture: the CUDA-graph replay of fwd+bwd gives the same
    bits as the stream-launched path, replay after replay (incl. the tail)."""
    import torch
    from paper_2410_11415_b200 import _lib, device_plan
    for name, loader in (("corpus_5", load_case), ("B", load_config)):
        tc, gold = loader(name)
        plan = device_plan(tc)
        lw = torch.tensor(np.log(gold["w_real"]), dtype=torch.float64, device=cuda)
        B = lw.shape[0]
        cap = plan.capture(B, np.float64, _lib.KLAY_LOG, backward=True, seeded=True)
        seed = torch.tensor(gold["seed"], dtype=torch.float64, device=cuda)
        out_ref, vals = plan.forward(lw, _lib.KLAY_LOG, np.float64)
        g_ref = plan.backward(vals, B, _lib.KLAY_LOG, np.float64, seed=seed)
        for _ in range(2):
            cap.weights.copy_(lw)
            cap.seed.copy_(seed)
            cap.replay()
            torch.cuda.synchronize()
            assert torch.equal(cap.outputs, out_ref)
            assert torch.equal(cap.grads, g_ref)
        rel_close(cap.grads.cpu().numpy(), gold["log_grad_seed"], 1e-12, 1e-12)


def test_bool_bit_packed_matches_float_path(cuda):
    """0/1 inputs take the bit-packed path (32 rows per word, AND/OR);
    outputs are bit-identical to the float max/min path and the oracle,
    including constant roots, odd batch sizes and the persistent tail."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan, engine
    rng = np.random.default_rng(9)
    cases = [load_case(n) for n in ("constants", "fig_pair_merge", "rnnf_wide")] + [load_config("D")]
    for tc, _ in cases:
        plan = device_plan(tc)
        for B in (1, 33, 1000):
            wb = rng.integers(0, 2, size=(B, tc.num_inputs)).astype(np.float64)
            ref, _ = oracle.forward(tc, wb, "bool", retain=False)
            out = engine.evaluate_semiring(tc, engine.WeightAssignment(wb), "bool")
            assert out.dtype == np.float64
            assert np.array_equal(out, ref)
            # explicit device call in float32 outputs
            o32, _ = plan.forward(torch.tensor(wb, dtype=torch.float32, device=cuda), _lib.KLAY_BOOL,
                                  engine.U1, retain=False)
            assert np.array_equal(o32.cpu().numpy(), ref.astype(np.float32))
    # non-0/1 inputs keep the float path (max/min on arbitrary values)
    tc, gold = load_case("fig_main")
    w = gold["w_real"]
    ref, _ = oracle.forward(tc, w, "bool", retain=False)
    assert np.array_equal(engine.evaluate_semiring(tc, engine.WeightAssignment(w), "bool"), ref)


def test_gradient_captured_pass_matches_trace_path(cuda):
    """engine.gradient (cached CUDA-graph pass) == forward + backward, and
    repeated calls with new weights / seeds do not leak state."""
    k = _engine()
    for name in ("constants", "corpus_5"):
        tc, gold = load_case(name)
        W = k.WeightAssignment(gold["w_real"])
        for log_domain in (True, False):
            for seed in (None, gold["seed"]):
                for dt in (np.float64, np.float32):
                    out, g = k.gradient(tc, W, log_domain=log_domain, seed=seed, dtype=dt)
                    tr = (k.forward_log(tc, W.to_log(), dtype=dt) if log_domain
                          else k.forward_real(tc, W, dtype=dt))
                    assert np.array_equal(out, tr.outputs)
                    assert np.array_equal(g, k.backward(tc, tr, seed))
        W2 = k.WeightAssignment(gold["w_real"][::-1].copy())
        out2, g2 = k.gradient(tc, W2, log_domain=True)
        tr = k.forward_log(tc, W2.to_log())
        assert np.array_equal(out2, tr.outputs) and np.array_equal(g2, k.backward(tc, tr))
    k.clear_cache()


def test_config_c_large_batch_4096(cuda):
    """B = 4096 fp32 (16.6 GB trace): 64-bit row addressing, 32 column
    chunks; golden rows embedded at both ends of the batch."""
    import torch
    from paper_2410_11415_b200 import _lib, device_plan
    tc, gold = load_config("C")
    plan = device_plan(tc)
    B = 4096
    rng = np.random.Generator(np.random.Philox(key=4))
    w = np.log(rng.uniform(0.05, 0.95, size=(B, tc.num_inputs)))
    lw = np.log(gold["w_real"])
    w[:8] = lw
    w[-8:] = lw
    wd = torch.from_numpy(w.astype(np.float32)).to(cuda)
    out, vals = plan.forward(wd, _lib.KLAY_LOG, np.float32)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float32)
    out, g = out.cpu().numpy(), g.cpu().numpy()
    for sl in (slice(0, 8), slice(B - 8, B)):
        fp32_close(out[sl], gold["log_out"], gold["log32_out"])
        fp32_close(g[sl], gold["log_grad"], gold["log32_grad"])
    del vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["fig_main", "corpus_5", "rnnf_small", "B", "Cp"])
def test_unary_parent_shortcut_is_bit_exact(cuda, name):
    """With epsilon 0 the log-sum backward skips the values of unary parents
    (klay.cu: bit 31 of the transposed CSR). Gradients must be bit-identical
    to the path that reads every parent (epsilon unknown = -1), including
    rows with -inf children (zero weights)."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    tc, gold = (load_config if name in CONFIGS else load_case)(name)
    plan = device_plan(tc)
    w = np.array(gold["w_real"], dtype=np.float64)[:64]
    w[::3, ::2] = 0.0  # -inf log-weights
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    for dt in (np.float64, np.float32):
        x = torch.tensor(lw, dtype=torch.float64 if dt == np.float64 else torch.float32,
                         device=cuda)
        _, vals = plan.forward(x, _lib.KLAY_LOG, dt)
        assert vals.klay_epsilon == 0.0
        g_short = plan.backward(vals, x.shape[0], _lib.KLAY_LOG, dt)
        g_full = plan.backward(vals, x.shape[0], _lib.KLAY_LOG, dt, epsilon=-1.0)
        assert torch.equal(torch.isnan(g_short), torch.isnan(g_full))
        assert torch.equal(torch.nan_to_num(g_short), torch.nan_to_num(g_full))
    # with epsilon > 0 every parent is read (the reference's exp(x - P))
    _, tr = oracle.forward(tc, lw, "log", epsilon=1e-3)
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    _, vals = plan.forward(x, _lib.KLAY_LOG, np.float64, epsilon=1e-3)
    g = plan.backward(vals, x.shape[0], _lib.KLAY_LOG, np.float64)
    rel_close(g.cpu().numpy(), oracle.backward(tc, tr, "log"), 1e-12, 1e-12)


@pytest.mark.parametrize("name", ["fig_main", "corpus_5", "rnnf_small", "rnnf_wide", "B"])
@pytest.mark.parametrize("eps", [0.0, 1e-3])
def test_log_domain_nonfinite_inputs_match_oracle(cuda, name, eps):
    """+inf / -inf / NaN log-weights follow the reference's masked
    logsumexp (engine.py:274-282: a +inf peak gives NaN, or +inf with
    epsilon > 0) and its masked backward weights (engine.py:346-352)."""
    import torch
    from oracle import engine_port as oracle
    from paper_2410_11415_b200 import _lib, device_plan
    tc, gold = (load_config if name in CONFIGS else load_case)(name)
    rng = np.random.default_rng(11)
    B = 48
    lw = np.log(rng.uniform(0.05, 0.95, size=(B, tc.num_inputs)))
    kinds = rng.integers(0, 8, size=lw.shape)
    lw[kinds == 0] = np.inf
    lw[kinds == 1] = -np.inf
    lw[(kinds == 2) & (rng.uniform(size=lw.shape) < 0.2)] = np.nan
    lw[: B // 4] = np.log(rng.uniform(0.05, 0.95, size=(B // 4, tc.num_inputs)))  # finite rows
    plan = device_plan(tc)
    with np.errstate(all="ignore"):
        ref, tr = oracle.forward(tc, lw, "log", epsilon=eps)
        gref = oracle.backward(tc, tr, "log")
    x = torch.tensor(lw, dtype=torch.float64, device=cuda)
    out, vals = plan.forward(x, _lib.KLAY_LOG, np.float64, epsilon=eps)
    g = plan.backward(vals, B, _lib.KLAY_LOG, np.float64)
    rel_close(out.cpu().numpy(), ref, 1e-12, 1e-12)
    rel_close(g.cpu().numpy(), gref, 1e-10, 1e-12)
    from paper_2410_11415_b200.engine import _NodeValues
    nv = _NodeValues(plan, vals, B)
    for l in range(len(tr)):
        rel_close(nv[l], tr[l], 1e-12, 1e-12)


@pytest.mark.parametrize("name", ["fig_main", "rnnf_wide", "A", "B", "C", "E", "Cp"])
def test_backward_only_trace_matches_full_trace(cuda, name):
    """retain=2 (unary nodes aliased: never written, adjoints routed down
    chains; klay.cu build_aliases) against retain=1 (every row written, plain
    backward): after klay_fill_trace the traces are bitwise equal, and the
    gradients of the two backward paths are bitwise equal, also with
    non-finite inputs."""
    import torch
    from paper_2410_11415_b200 import _lib, device_plan
    tc, gold = (load_config if name in CONFIGS else load_case)(name)
    plan = device_plan(tc)
    rng = np.random.default_rng(3)
    B = 40
    lw = np.log(rng.uniform(0.05, 0.95, size=(B, tc.num_inputs)))
    lw[rng.uniform(size=lw.shape) < 0.05] = -np.inf
    lw[rng.uniform(size=lw.shape) < 0.01] = np.inf
    lw[rng.uniform(size=lw.shape) < 0.01] = np.nan
    lw[: B // 2] = np.log(rng.uniform(0.05, 0.95, size=(B // 2, tc.num_inputs)))
    for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32)):
        x = torch.tensor(lw, dtype=tdt, device=cuda)
        out_p, vals_p = plan.forward(x, _lib.KLAY_LOG, dt)                  # backward-only
        out_f, vals_f = plan.forward(x, _lib.KLAY_LOG, dt, retain="full")   # every row
        assert torch.equal(out_p.nan_to_num(), out_f.nan_to_num())
        g_p = plan.backward(vals_p, B, _lib.KLAY_LOG, dt)   # aliases + routes
        g_f = plan.backward(vals_f, B, _lib.KLAY_LOG, dt)   # plain
        assert torch.equal(torch.isnan(g_p), torch.isnan(g_f))
        assert torch.equal(g_p.nan_to_num(), g_f.nan_to_num())
        plan.fill_trace(vals_p, B)
        a, b = vals_p[:, :B], vals_f[:, :B]
        assert torch.equal(torch.isnan(a), torch.isnan(b))
        assert torch.equal(a.nan_to_num(), b.nan_to_num())


@pytest.mark.parametrize("tail_edges,no_micro", [("0", "0"), ("100000", "0"), ("256", "1")])
def test_alias_and_tail_extremes(cuda, tail_edges, no_micro):
    """The persistent tail (and its shared-memory micro tail) normally takes
    every small circuit whole (no aliases there). Re-run the golden,
    non-finite and trace-equality suites with no tail (every unary node below
    the last layer aliased, routes everywhere), with an all-tail schedule, and
    with the micro tail off (the thinnest layers in the cluster tail);
    KLAY_TAIL_EDGES / KLAY_NO_MICRO are read when libklay loads, hence the
    subprocess."""
    import subprocess
    import sys
    env = dict(os.environ, KLAY_TAIL_EDGES=tail_edges, KLAY_NO_MICRO=no_micro)
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(os.path.dirname(__file__), "test_engine_gpu.py"),
         os.path.join(os.path.dirname(__file__), "test_fuzz_gpu.py"),
         "-k", "golden_small or nonfinite or backward_only or consumer or random_circuits"],
        env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("cfg", ["A", "B", "C", "D", "E"])
def test_plan_schedule_matches_byte_model(cuda, cfg):
    """bench.py's byte model restates the plan builder's schedule (tail and
    micro-tail boundaries) and its unary-node aliases; both must agree with
    the library's own plan (klay_plan_schedule)."""
    import bench
    from paper_2410_11415_b200 import device_plan
    tc, _ = load_config(cfg)
    plan = device_plan(tc)
    s = plan.schedule
    assert s["tail"] == bench._tail_from(tc)
    assert s["micro"] == bench._micro_from(tc, True)
    assert s["micro_bwd"] == bench._micro_from(tc, False)
    assert s["head"] == bench._micro_head(tc, True)
    assert s["head_bwd"] == bench._micro_head(tc, False)
    ap = bench.alias_plan(tc)
    n_alias = sum(int(np.asarray(a).sum()) for a in ap["ali"]) if ap is not None else 0
    assert s["aliased_rows"] == n_alias
