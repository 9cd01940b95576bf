"""Run-time bounds checking (compute-sanitizer is closed on the GPU pool, so
this is the memcheck stand-in): libklay_checks.so is libklay built with
-DKLAY_CHECKS, where every global row access of the layer, tail, micro and
streaming kernels is verified against the call's buffers (common.cuh chk;
the small boundary kernels -- inputs, roots, seeds, grads -- are not)
and a violation fails the call instead of faulting. The parity suites must
pass on it with zero violations, and accesses beyond a deliberately
shrunken valid range (KLAY_CHECKS_SHRINK) must be reported."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKS = os.path.join(ROOT, "paper_2410_11415_b200", "libklay_checks.so")

PROBE = r"""
import ctypes, os, numpy as np, torch, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import load_config
from paper_2410_11415_b200 import _lib, engine
lib = _lib.load()
assert b"bounds-checked" in lib.klay_version(), lib.klay_version()
tc, gold = load_config("B")
plan = engine.device_plan(tc, torch.device("cuda", 0))
B = 64
w = torch.zeros((B, tc.num_inputs), dtype=torch.float32, device="cuda")
# KLAY_CHECKS_SHRINK (set by the test) declares only the first rows of the
# trace valid: the forward's legal writes past them must be reported
try:
    plan.forward(w, _lib.KLAY_LOG, np.float32, retain="full")
    raise SystemExit("no violation reported")
except RuntimeError as e:
    msg = str(e)
assert "bounds check failed" in msg, msg
print("probe ok:", msg)
"""


def _env():
    if not os.path.exists(CHECKS):
        pytest.fail("libklay_checks.so missing: run __graft_entry__.build()")
    return dict(os.environ, KLAY_LIB=CHECKS)


def test_checked_build_reports_out_of_range_access(cuda):
    """Negative control: with the values buffer declared 1 MB long, the
    forward's accesses beyond it are reported (and redirected, not made)."""
    env = dict(_env(), KLAY_CHECKS_SHRINK=str(1 << 20))
    r = subprocess.run([sys.executable, "-c", PROBE, ROOT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "probe ok" in r.stdout


def test_parity_suites_clean_under_bounds_checks(cuda):
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(ROOT, "tests", "test_engine_gpu.py"), os.path.join(ROOT, "tests", "test_fuzz_gpu.py"),
           os.path.join(ROOT, "tests", "test_api_gpu.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    env = dict(_env(), KLAY_STREAM="1")  # the streaming kernel too
    cmd[-3:] = [os.path.join(ROOT, "tests", "test_engine_gpu.py")]
    cmd += ["-k", "golden or consumer or full_batch"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
