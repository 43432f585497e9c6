"""bench.py's launcher contract on CPU: `python bench.py --gpus N` outside
torchrun re-runs itself under torch.distributed.run with N ranks (one process
per GPU, rendezvous on 127.0.0.1); under torchrun (WORLD_SIZE set) it runs."""

import importlib.util
import os
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_plain_gpus_n_spawns_n_ranks(monkeypatch):
    bench = _bench()
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3"])
    with pytest.raises(SystemExit) as e:
        bench.maybe_spawn(types.SimpleNamespace(gpus=2))
    assert e.value.code == 0 and len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "2", "--steps", "3", "--warmup", "3"]


def test_under_torchrun_or_one_gpu_runs_in_process(monkeypatch):
    bench = _bench()
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: pytest.fail("must not re-spawn"))
    monkeypatch.setenv("WORLD_SIZE", "2")
    bench.maybe_spawn(types.SimpleNamespace(gpus=2))  # already a rank of a torchrun job
    monkeypatch.delenv("WORLD_SIZE")
    bench.maybe_spawn(types.SimpleNamespace(gpus=1))  # one GPU: this process
