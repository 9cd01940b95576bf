"""The online logsumexp recurrence of the CUDA kernels (csrc/common.cuh:
LseOp::push (branch-free form) / result and lse_merge for split segments),
restated in Python,
equals the reference's masked max-trick logsumexp (engine.py:274-282) on
every combination of finite, +-inf and NaN elements, whole or split into
leaves. CPU only: a design check of the recurrence the GPU tests exercise."""

import itertools

import numpy as np
import pytest

INF = np.inf
VALS = [-1.0, 0.5, 2.0, -INF, INF, np.nan]


def _push_all(xs):
    m, t = -INF, 0.0
    for k, x in enumerate(xs):
        if k == 0:
            m, t = x, (0.0 if x == -INF else 1.0)
            continue
        d = x - m
        e = np.exp(-abs(d))
        if d != d:
            e = d if (x != x or m != m) else 0.0
        if d > 0:
            t, m = t * e + 1.0, x
        else:
            t = t + e
    return m, t


def _merge(m, t, m2, t2):
    if m2 > m:
        return m2, t * np.exp(m - m2) + t2
    if m2 == -INF or m2 == INF:
        return m, (t2 if np.isnan(t2) else t)
    return m, t + t2 * np.exp(m2 - m)


def _result(m, t, eps):
    res = m if (t == 1.0 and eps == 0.0) else np.log(t + eps) + m
    if m == INF and not np.isnan(t):
        res = INF if eps > 0 else np.nan
    return -INF if (m == -INF and not np.isnan(t)) else res


def _reference(xs, eps):
    xs = np.asarray(xs, dtype=np.float64)
    peak = np.maximum.reduce(xs)
    z = np.exp(xs - peak)
    z[np.isnan(z)] = 0.0
    r = np.log(z.sum() + eps) + peak
    return -INF if peak == -INF else r


def _same(a, b):
    return (np.isnan(a) and np.isnan(b)) or a == b or abs(a - b) <= 1e-12 * max(1.0, abs(b))


@pytest.mark.parametrize("eps", [0.0, 1e-3])
def test_online_logsumexp_matches_reference(eps):
    with np.errstate(all="ignore"):
        for n in range(1, 5):
            for xs in itertools.product(VALS, repeat=n):
                assert _same(_result(*_push_all(xs), eps), _reference(xs, eps)), xs


def test_split_logsumexp_matches_reference():
    with np.errstate(all="ignore"):
        for n in range(2, 6):
            for xs in itertools.product(VALS, repeat=n):
                for cuts in itertools.combinations(range(1, n), 2 if n > 2 else 1):
                    bounds = (0,) + cuts + (n,)
                    m, t = _push_all(xs[:bounds[1]])
                    for a, b in zip(bounds[1:-1], bounds[2:]):
                        m, t = _merge(m, t, *_push_all(xs[a:b]))
                    assert _same(_result(m, t, 0.0), _reference(xs, 0.0)), (xs, cuts)
