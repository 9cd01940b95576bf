"""bench.py's measurement model on the CPU: launch-class mapping of ncu kernel
names, per-class traffic from the committed launch list, the byte models,
and the multi-GPU self-spawn command."""

import json
import os
import sys

import pytest

from conftest import ROOT, load_config

sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("name,cls", [
    ("void items_kernel<float, 0, FwdGather<float, 1>>(LayerArgs<T1>)", "fwd_prod"),
    ("void items_kernel<float, 0, FwdGather<float, 0>>(LayerArgs<T1>)", "fwd_prod"),
    ("void items_kernel<float, 4, FwdGather<float, 0>>(LayerArgs<T1>)", "fwd_sum"),
    ("void combine_kernel<double, 4, FwdGather<double, 0>>(LayerArgs<T1>)", "fwd_sum"),
    ("void items_kernel<float, 0, BwdGather<float, 3>>(LayerArgs<T1>)", "bwd_pass"),
    ("void items_kernel<float, 0, BwdGather<float, 0>>(LayerArgs<T1>)", "bwd_pass"),
    ("void items_kernel<float, 0, BwdGather<float, 1>>(LayerArgs<T1>)", "bwd_logsum"),
    ("void items_kernel<double, 0, BwdGather<double, 4>>(LayerArgs<T1>)", "bwd_logsum"),
    ("void items_kernel<double, 0, BwdGather<double, 2>>(LayerArgs<T1>)", "bwd_realprod"),
    ("void micro_kernel<float, 0, 4, 2>(MicroArgs<T1>)", "fwd_micro"),
    ("void micro_bwd_kernel<float, 1, 2>(MicroBwdArgs<T1>)", "bwd_micro"),
    ("void tail_kernel<float, 0, 4, FwdGather<float, 0>, FwdGather<float, 0>>(TailArgs<T1>)", "tail"),
    ("void seed_kernel<float>(const T1 *, const int *, const int *, T1 *, int, int, long long, long long)",
     "boundary"),
])
def test_kernel_class_of_ncu_names(name, cls):
    assert bench.kernel_class(name) == cls


def test_committed_launch_list_per_class():
    """profiles/r2_launches.csv (one fwd+bwd step of config C): every launch
    lands in one class; the layer-kernel classes hold 24 launches each and
    together almost all of the step's DRAM bytes."""
    path = os.path.join(ROOT, "profiles", "r2_launches.csv")
    t = bench.ncu_class_traffic(path)
    assert t is not None
    assert {c: v["launches"] for c, v in t.items()} == {
        "fwd_prod": 24, "fwd_sum": 24, "bwd_pass": 24, "bwd_logsum": 24,
        "fwd_micro": 1, "bwd_micro": 1, "boundary": 4}
    total = sum(v["dram_bytes"] for v in t.values())
    big = sum(t[c]["dram_bytes"] for c in ("fwd_prod", "fwd_sum", "bwd_pass", "bwd_logsum"))
    assert big > 0.97 * total
    with open(os.path.join(ROOT, "profiles", "r2_launches.json")) as fh:
        assert json.load(fh)["steps"] == 1


@pytest.mark.parametrize("cfg", ["B", "C"])
def test_byte_models(cfg):
    """The implemented dataflow never needs more bytes than the plain
    (reference-order) dataflow, which in turn is at most SURVEY §8(d)'s
    contract model (the contract charges log-sum layers both layers twice)."""
    tc, _ = load_config(cfg)
    for s, B in ((4, 1024), (8, 256)):
        nec = bench.bytes_per_eval(tc, s, B)
        plain = bench.bytes_per_eval(tc, s, B, alias=False)
        contract = bench.bytes_per_eval(tc, s, B, survey=True)
        assert 0 < nec <= plain <= contract


def test_spawn_ranks_command(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-runs itself as N ranks on
    127.0.0.1 with the same arguments."""
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])

    class A:
        gpus = 4

    bench.spawn_ranks(A)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    assert os.path.basename(cmd[-5]) == "bench.py"
