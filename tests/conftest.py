"""Shared helpers: golden fixtures (frozen reference outputs) and markers."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
CONSUMER = os.path.join(GOLDEN, "consumer")
CIRCUITS = os.path.join(ROOT, "data", "circuits")

SMALL_CASES = sorted(
    f[:-4] for f in os.listdir(os.path.join(GOLDEN, "circuits")) if f.endswith(".npz"))
CONFIGS = ["A", "B", "C", "D", "E", "Cp"]

# The reference CLI commands that produced each committed consumer dump
# (/root/reference/pkg/scripts/make_consumer_fixtures.py:54-70):
# (circuit, weights, mode, log, epsilon)
CONSUMER_DUMPS = {
    "fig_half_eval.json": ("fig_main.klay", "w_half.json", "eval", False, 0.0),
    "fig_mixed_eval.json": ("fig_main.klay", "w_mixed.json", "eval", False, 0.0),
    "fig_mixed_eval_log.json": ("fig_main.klay", "w_mixed.json", "eval", True, 0.0),
    "fig_mixed_eval_log_eps.json": ("fig_main.klay", "w_mixed.json", "eval", True, 1e-3),
    "fig_batch_eval.json": ("fig_main.klay", "w_batch.json", "eval", False, 0.0),
    "fig_mixed_grad.json": ("fig_main.klay", "w_mixed.json", "grad", False, 0.0),
    "fig_mixed_grad_log.json": ("fig_main.klay", "w_mixed.json", "grad", True, 0.0),
    "fig_batch_grad.json": ("fig_main.klay", "w_batch.json", "grad", False, 0.0),
    "pair_eval.json": ("pair.klay", "w_pair.json", "eval", False, 0.0),
    "pair_grad.json": ("pair.klay", "w_pair.json", "grad", False, 0.0),
}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libklay.so)")


def load_case(name):
    from paper_2410_11415_b200.tensorized import load_npz
    tc = load_npz(os.path.join(GOLDEN, "circuits", f"{name}.npz"))
    return tc, dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def load_config(name):
    from paper_2410_11415_b200.tensorized import load_npz
    tc = load_npz(os.path.join(CIRCUITS, f"{name}.npz"))
    return tc, dict(np.load(os.path.join(GOLDEN, f"cfg{name}.npz")))


def consumer_case(dump):
    """(tc, real weights [B,K], expected roots [B,R], expected grad or None, log, eps)."""
    from paper_2410_11415_b200.engine import weights_from_json
    from paper_2410_11415_b200.tensorized import read_klay
    circ, wfile, mode, log, eps = CONSUMER_DUMPS[dump]
    with open(os.path.join(CONSUMER, circ)) as fh:
        tc = read_klay(fh.read())
    with open(os.path.join(CONSUMER, wfile)) as fh:
        w = weights_from_json(json.load(fh), tc.input_map)
    with open(os.path.join(CONSUMER, dump)) as fh:
        exp = json.load(fh)
    roots = np.atleast_2d(np.asarray(exp["roots"], dtype=np.float64))
    grad = np.asarray(exp["grad"], dtype=np.float64) if mode == "grad" else None
    return tc, w, roots, grad, log, eps


def rel_close(got, exp, rtol, atol_frac=0.0):
    """|got-exp| <= rtol*|exp| + atol_frac*max|exp| elementwise, with
    identical -inf/+inf/NaN positions."""
    got = np.asarray(got, dtype=np.float64)
    exp = np.asarray(exp, dtype=np.float64)
    assert got.shape == exp.shape, (got.shape, exp.shape)
    fin = np.isfinite(exp)
    assert np.array_equal(np.isnan(got), np.isnan(exp)), "NaN positions differ"
    assert np.array_equal(got[~fin & ~np.isnan(exp)], exp[~fin & ~np.isnan(exp)]), "inf mismatch"
    if fin.any():
        scale = np.abs(exp[fin]).max()
        err = np.abs(got[fin] - exp[fin])
        tol = rtol * np.abs(exp[fin]) + atol_frac * scale
        bad = err > tol
        assert not bad.any(), (
            f"{bad.sum()} of {bad.size} beyond tol; worst rel "
            f"{(err / np.maximum(np.abs(exp[fin]), 1e-300)).max():.3e}")


def fp32_close(got, ref64, ref32, rtol=1e-5):
    """Elementwise fp32 gate against the reference's own fp32 error: with
    ref64 the reference in fp64 and ref32 the reference run in fp32,
    |got - ref64| <= max(rtol * |ref64|, 2 * |ref32 - ref64|) at every finite
    ref64 entry (no scale-relative slack), identical -inf/+inf/NaN positions
    elsewhere. So an fp32 result may be off by the north star's rel 1e-5 or
    by twice what the reference's own fp32 evaluation is off, whichever is
    larger -- small gradients are checked at their own size."""
    got = np.asarray(got, dtype=np.float64)
    ref64 = np.asarray(ref64, dtype=np.float64)
    ref32 = np.asarray(ref32, dtype=np.float64)
    assert got.shape == ref64.shape == ref32.shape, (got.shape, ref64.shape, ref32.shape)
    fin = np.isfinite(ref64)
    assert np.array_equal(np.isnan(got[~fin]), np.isnan(ref64[~fin])), "NaN positions differ"
    nonnan = ~fin & ~np.isnan(ref64)
    assert np.array_equal(got[nonnan], ref64[nonnan]), "inf mismatch"
    if fin.any():
        with np.errstate(invalid="ignore"):
            tol = np.maximum(rtol * np.abs(ref64[fin]), 2.0 * np.abs(ref32[fin] - ref64[fin]))
        tol = np.where(np.isnan(tol), np.inf, tol)
        err = np.abs(got[fin] - ref64[fin])
        bad = ~(err <= tol)
        assert not bad.any(), (
            f"{bad.sum()} of {bad.size} beyond the fp32 gate; worst err/tol "
            f"{np.max(err[bad] / np.maximum(tol[bad], 1e-300)):.3e} at ref {ref64[fin][bad][:3]}, "
            f"got {got[fin][bad][:3]}, ref32 {ref32[fin][bad][:3]}")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    from paper_2410_11415_b200 import _lib
    _lib.load()  # fail loudly when the library is missing
    return torch.device("cuda", 0)
