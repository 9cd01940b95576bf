"""The opt-in streaming kernel (KLAY_STREAM=1: cp.async.bulk row streams,
stream_kernels.cuh) under the same golden parity suites as the default
items_kernel path. libklay reads the switch once at load, so the suites run
in a child process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _child(*args):
    env = dict(os.environ, KLAY_STREAM="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_stream_kernel_golden_parity(cuda):
    _child(os.path.join(ROOT, "tests", "test_engine_gpu.py"),
           "-k", "consumer or golden_small or golden_configs or full_batch or backward_only")


def test_stream_kernel_random_circuits(cuda):
    """Random circuits with aliases and adjoint routes, incl. row widths that
    are not a multiple of the 512-byte mask chunk."""
    _child(os.path.join(ROOT, "tests", "test_fuzz_gpu.py"),
           "-k", "random_circuits_match_oracle or route_masks_odd_row_widths")
