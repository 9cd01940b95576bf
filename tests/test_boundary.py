"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/klay.h declares; the circuit container and
.klay reader behave like the reference's (tensorize.py:94-313)."""

import io
import os
import re

import numpy as np
import pytest

from conftest import CONSUMER, ROOT, SMALL_CASES, load_case


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "klay.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(klay_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2410_11415_b200 import _lib
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table and header disagree"
    assert b"sm_100a" in lib.klay_version()


def test_library_is_sm100a_code():
    import subprocess
    so = os.path.join(ROOT, "paper_2410_11415_b200", "libklay.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_row_stride_and_plan_errors_without_gpu():
    from paper_2410_11415_b200 import _lib
    lib = _lib.load()
    assert lib.klay_row_stride(1, _lib.KLAY_F32) == 4
    assert lib.klay_row_stride(5, _lib.KLAY_F32) == 8
    assert lib.klay_row_stride(5, _lib.KLAY_F64) == 6
    assert lib.klay_row_stride(1024, _lib.KLAY_F32) == 1024
    # the host-side format validation runs before any device work
    import ctypes
    h = ctypes.c_void_p()
    widths = np.array([2], np.int64)
    counts = np.array([2], np.int64)
    src = np.array([0, 5], np.int64)  # out of range
    seg = np.array([0, 1], np.int64)
    roots = np.array([0], np.int64)
    cv = np.zeros(1, np.int8)
    rc = lib.klay_plan_create(2, 1, widths.ctypes.data, counts.ctypes.data, src.ctypes.data,
                              seg.ctypes.data, 1, roots.ctypes.data, cv.ctypes.data, 0,
                              ctypes.byref(h))
    assert rc == _lib.KLAY_EFORMAT
    assert "out of range" in _lib.last_error()
    assert lib.klay_forward(None, 0, 0, None, 0, None, 4, 1, None, 1, 0.0, None, None) == _lib.KLAY_EINVAL


@pytest.mark.parametrize("name", SMALL_CASES)
def test_klay_and_npz_roundtrip(name):
    from paper_2410_11415_b200.tensorized import load_npz, read_klay, save_npz, write_klay
    tc, _ = load_case(name)
    buf = io.StringIO()
    write_klay(tc, buf)
    assert read_klay(buf.getvalue()) == tc
    b = io.BytesIO()
    save_npz(tc, b)
    b.seek(0)
    assert load_npz(b) == tc


def test_read_reference_klay_fixture():
    from paper_2410_11415_b200.tensorized import read_klay
    with open(os.path.join(CONSUMER, "fig_main.klay")) as fh:
        tc = read_klay(fh.read())
    assert tc.num_inputs == 8 and [l.width for l in tc.layers] == [7, 6, 3, 1]
    assert tc.layers[0].sources.tolist() == [5, 4, 6, 2, 7, 1, 3, 1, 0]


BAD = {
    "empty": "",
    "version": "klay 2\ninputs 1\nvars 1\nroots 0\ninputmap 1:0\n",
    "no_inputmap": "klay 1\ninputs 1\nvars 1\nroots 0\n",
    "dup_literal": "klay 1\ninputs 2\nvars 1\nroots 0\ninputmap 1:0 1:1\n",
    "wrong_op": "klay 1\ninputs 2\nvars 2\nroots 0\ninputmap 1:0 2:1\nlayer 1 sum 1 2\nS 0 1\nR 0 0\n",
    "unread": "klay 1\ninputs 2\nvars 2\nroots 0\ninputmap 1:0 2:1\nlayer 1 prod 1 1\nS 0\nR 0\n",
    "decreasing": "klay 1\ninputs 2\nvars 2\nroots 0\ninputmap 1:0 2:1\nlayer 1 prod 2 2\nS 0 1\nR 1 0\n",
    "count": "klay 1\ninputs 2\nvars 2\nroots 0\ninputmap 1:0 2:1\nlayer 1 prod 1 3\nS 0 1\nR 0 0\n",
    "root_range": "klay 1\ninputs 2\nvars 2\nroots 4\ninputmap 1:0 2:1\nlayer 1 prod 1 2\nS 0 1\nR 0 0\n",
    "garbage": "klay 1\ninputs x\nvars 2\n",
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_read_klay_rejects(case):
    from paper_2410_11415_b200.tensorized import KlayFormatError, read_klay, read_klay_py
    with pytest.raises(KlayFormatError):
        read_klay(BAD[case])     # libklay's C++ reader
    with pytest.raises(KlayFormatError):
        read_klay_py(BAD[case])  # the Python reader


def _accepts(reader, text):
    from paper_2410_11415_b200.tensorized import KlayFormatError
    try:
        return reader(text)
    except KlayFormatError:
        return None


@pytest.mark.parametrize("name", ["fig_main", "corpus_3", "rnnf_small", "constants", "dup_child"])
def test_native_and_python_klay_readers_agree(name):
    """Round trips are equal, and randomly corrupted files are accepted or
    rejected alike (and parse to the same circuit when accepted)."""
    from paper_2410_11415_b200.tensorized import read_klay, read_klay_py, write_klay
    tc, _ = load_case(name)
    buf = io.StringIO()
    write_klay(tc, buf)
    text = buf.getvalue()
    assert read_klay(text) == read_klay_py(text) == tc
    rng = np.random.default_rng(5)
    toks = text.split(" ")
    for _ in range(150):
        t = list(toks)
        k = int(rng.integers(len(t)))
        t[k] = str(rng.choice(["0", "1", "-1", "7", "x", "", "2:1", "1:0", "99999"]))
        bad = " ".join(t)
        a, b = _accepts(read_klay, bad), _accepts(read_klay_py, bad)
        assert (a is None) == (b is None), (k, t[k])
        if a is not None:
            assert a == b


def test_weight_constructors_match_reference_semantics():
    from paper_2410_11415_b200 import EvalError, Literal, weights_from_json
    from paper_2410_11415_b200.tensorized import read_klay
    with open(os.path.join(CONSUMER, "fig_main.klay")) as fh:
        tc = read_klay(fh.read())
    w = weights_from_json({"p": {"1": 0.3, "2": 0.5, "3": 0.5, "4": 0.5}}, tc.input_map)
    assert w.values[0, tc.input_map[Literal(1)]] == pytest.approx(0.3)
    assert w.values[0, tc.input_map[Literal(1, False)]] == pytest.approx(0.7)
    row = {str(lit.to_dimacs()): 1.0 for lit in tc.input_map}
    assert weights_from_json([{"w": row}, {"w": row}], tc.input_map).batch == 2
    with pytest.raises(EvalError):
        weights_from_json({"w": {"1": 0.5}}, tc.input_map)
    with pytest.raises(EvalError):
        weights_from_json({"p": {"1": 0.5}}, tc.input_map)
    with pytest.raises(EvalError):
        weights_from_json([], tc.input_map)
