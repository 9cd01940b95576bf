"""Pin the CPU oracle (oracle/engine_port.py) to the reference's own golden
vectors before trusting it as the checker of the CUDA path. CPU only."""

import numpy as np
import pytest

from conftest import (CONFIGS, CONSUMER_DUMPS, SMALL_CASES, consumer_case, load_case,
                      load_config)
from oracle import engine_port as oracle


@pytest.mark.parametrize("dump", sorted(CONSUMER_DUMPS))
def test_oracle_reproduces_reference_consumer_dumps(dump):
    """The 10 committed dumps of the reference CLI, bit-exactly."""
    tc, w, roots, grad, log, eps = consumer_case(dump)
    if log:
        with np.errstate(divide="ignore"):
            vals = np.log(w.values)
        out, trace = oracle.forward(tc, vals, "log", epsilon=eps)
    else:
        out, trace = oracle.forward(tc, w.values, "real")
    assert np.array_equal(out, roots)
    if grad is not None:
        g = oracle.backward(tc, trace, "log" if log else "real")
        assert np.array_equal(g, grad)


def _check_suite(tc, gold):
    w = gold["w_real"]
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    out, tr = oracle.forward(tc, w, "real")
    assert np.array_equal(out, gold["real_out"])
    assert np.array_equal(oracle.backward(tc, tr, "real"), gold["real_grad"], equal_nan=True)
    assert np.array_equal(oracle.backward(tc, tr, "real", gold["seed"]), gold["real_grad_seed"],
                          equal_nan=True)
    out, tr = oracle.forward(tc, lw, "log")
    assert np.array_equal(out, gold["log_out"])
    assert np.array_equal(oracle.backward(tc, tr, "log"), gold["log_grad"])
    assert np.array_equal(oracle.backward(tc, tr, "log", gold["seed"]), gold["log_grad_seed"])
    out, tr = oracle.forward(tc, lw, "log", epsilon=1e-3)
    assert np.array_equal(out, gold["logeps_out"])
    assert np.array_equal(oracle.backward(tc, tr, "log"), gold["logeps_grad"])
    out, tr = oracle.forward(tc, w.astype(np.float32), "real")
    assert np.array_equal(out, gold["real32_out"])
    assert np.array_equal(oracle.backward(tc, tr, "real"), gold["real32_grad"], equal_nan=True)
    out, tr = oracle.forward(tc, lw.astype(np.float32), "log")
    assert np.array_equal(out, gold["log32_out"])
    assert np.array_equal(oracle.backward(tc, tr, "log"), gold["log32_grad"])
    out, _ = oracle.forward(tc, gold["w_bool"], "bool", retain=False)
    assert np.array_equal(out, gold["bool_out"])
    out, _ = oracle.forward(tc, w, "maxprod", retain=False)
    assert np.array_equal(out, gold["maxprod_out"])


@pytest.mark.parametrize("name", SMALL_CASES)
def test_oracle_matches_reference_goldens_small(name):
    tc, gold = load_case(name)
    with np.errstate(all="ignore"):
        _check_suite(tc, gold)


@pytest.mark.parametrize("cfg", ["A", "B", "D", "E"])
def test_oracle_matches_reference_goldens_configs(cfg):
    tc, gold = load_config(cfg)
    with np.errstate(all="ignore"):
        _check_suite(tc, gold)


@pytest.mark.parametrize("cfg", ["C", "Cp"])
def test_oracle_matches_reference_goldens_config_c_log(cfg):
    tc, gold = load_config(cfg)
    w = gold["w_real"]
    with np.errstate(divide="ignore"):
        lw = np.log(w)
    out, tr = oracle.forward(tc, lw, "log")
    assert np.array_equal(out, gold["log_out"])
    assert np.array_equal(oracle.backward(tc, tr, "log"), gold["log_grad"])


def test_pairwise_emulation_matches_numpy_reduceat():
    """The summation order the CUDA kernels implement (x0 + numpy pairwise
    of the rest) reproduces np.add.reduceat bit-for-bit."""
    from tests_support_pairwise import np_segment_sum_emulated
    rng = np.random.default_rng(7)
    for dt in (np.float32, np.float64):
        for n in list(range(1, 140)) + [255, 256, 257, 1000, 1391, 4100]:
            x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, n)).astype(dt)
            ref = np.add.reduceat(x[None, :], [0], axis=-1)[0, 0]
            assert np_segment_sum_emulated(x) == ref, (dt, n)


def test_oracle_rejects_bad_inputs():
    tc, gold = load_case("fig_main")
    with pytest.raises(oracle.OracleError):
        oracle.forward(tc, gold["w_real"], "tropical")
    with pytest.raises(oracle.OracleError):
        oracle.forward(tc, gold["w_real"], "log", epsilon=-1.0)
    _, tr = oracle.forward(tc, gold["w_real"], "real")
    with pytest.raises(oracle.OracleError):
        oracle.backward(tc, tr, "real", seed=np.ones((1, 5)))
    with pytest.raises(oracle.OracleError):
        oracle.backward(tc, None, "real")
