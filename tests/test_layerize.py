"""The C++ layerizer (csrc/layerize.cpp) reproduces the reference's
tensorize(layerize(circuits)) bit for bit. CPU only.

Circuits come from the reference itself when /root/reference is importable
(build container); tests/golden/sources/*.npz holds a few flattened source
circuits so the comparison also runs without it."""

import os
import sys
import time

import numpy as np
import pytest

from conftest import GOLDEN, load_case

REF = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF)


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import laycirc
    return laycirc


def _refconf():
    """The reference's tests/conftest.py (fixture builders), by path: our own
    tests/conftest.py shadows the module name."""
    import importlib.util
    _ref()
    spec = importlib.util.spec_from_file_location("laycirc_ref_conftest",
                                                  "/root/reference/pkg/tests/conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Node(tuple):
    pass


class FlatCircuit:
    """Minimal Circuit duck type rebuilt from a flattened source fixture."""

    def __init__(self, kinds, lits, coff, kids, roots, num_vars):
        from paper_2410_11415_b200.tensorized import Literal
        names = ["leaf", "and", "or", "true", "false"]
        self.nodes = [(names[k], Literal.from_dimacs(int(l)) if k == 0 else None,
                       tuple(int(c) for c in kids[coff[i]:coff[i + 1]]))
                      for i, (k, l) in enumerate(zip(kinds, lits))]
        self.roots = [int(r) for r in roots]
        self.num_vars = int(num_vars)


def _sources(name):
    z = np.load(os.path.join(GOLDEN, "sources", f"{name}.npz"))
    out = []
    for i in range(int(z["n"])):
        out.append(FlatCircuit(z[f"kinds{i}"], z[f"lits{i}"], z[f"coff{i}"], z[f"kids{i}"],
                               z[f"roots{i}"], z[f"nvars{i}"]))
    return out


@pytest.mark.parametrize("name", ["fig_main", "fig_pair_merge", "constants", "corpus_5",
                                  "rnnf_small"])
def test_layerize_matches_frozen_reference_output(name):
    """Stored source circuits -> the tensorized circuits the reference made."""
    from paper_2410_11415_b200.layerize import layerize_tensorize
    tc_ref, _ = load_case(name)
    assert layerize_tensorize(_sources(name)) == tc_ref


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable")
def test_layerize_matches_reference_on_fixture_and_random_circuits():
    from paper_2410_11415_b200.layerize import layerize_tensorize
    laycirc = _ref()
    refconf = _refconf()
    from laycirc.bench import gen_3cnf, gen_random_nnf, rng_for
    cases = [[c] for _, c in refconf.all_fixtures()]
    cases.append([refconf.build_fig_main(), refconf.build_fig_second(), refconf.build_fig_main()])
    unsat = laycirc.Circuit(num_vars=1)
    unsat.set_roots([unsat.add_false()])
    cases.append([refconf.build_fig_main(), unsat, refconf.build_single_leaf()])
    rng = rng_for(77)
    for i in range(40):
        nv = int(rng.integers(4, 14))
        cnf = gen_3cnf(nv, int(rng.integers(nv, 4 * nv)), i)
        cases.append([laycirc.fold_constants(laycirc.compile_cnf(cnf))])
    cases.append([gen_random_nnf(10, 200, 5, 3, 3)])
    cases.append([laycirc.fold_constants(laycirc.compile_cnf(gen_3cnf(12, 30, s))) for s in range(20)])
    for circuits in cases:
        ref = laycirc.tensorize(laycirc.layerize(circuits))
        got = layerize_tensorize(circuits)
        assert got == ref


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable")
def test_layerize_errors_match_reference_cases():
    from paper_2410_11415_b200.layerize import CircuitError, layerize_tensorize
    laycirc = _ref()
    c = laycirc.Circuit(num_vars=1)
    x = c.add_leaf(laycirc.Literal(1))
    t = c.add_true()
    c.set_roots([c.add_and([x, t])])
    with pytest.raises(CircuitError):
        layerize_tensorize([c])  # internal constant: fold_constants first
    with pytest.raises(CircuitError):
        layerize_tensorize([])
    empty = laycirc.Circuit(num_vars=1)
    empty.add_leaf(laycirc.Literal(1))
    with pytest.raises(CircuitError):
        layerize_tensorize([empty])  # no roots


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable")
def test_layerize_config_b_speed_and_parity():
    """Config B (107,747 nodes): bit-exact, and much faster than Python."""
    from paper_2410_11415_b200.layerize import layerize_tensorize
    from paper_2410_11415_b200.tensorized import load_npz
    laycirc = _ref()
    from laycirc.bench import gen_3cnf
    circuit = laycirc.fold_constants(laycirc.compile_cnf(gen_3cnf(45, 100, 1)))
    t0 = time.perf_counter()
    got = layerize_tensorize([circuit])
    t_fast = time.perf_counter() - t0
    assert got == load_npz(os.path.join(os.path.dirname(GOLDEN), "..", "data", "circuits", "B.npz"))
    t0 = time.perf_counter()
    laycirc.tensorize(laycirc.layerize([circuit]))
    t_ref = time.perf_counter() - t0
    assert t_fast < t_ref
