"""bench.py host logic (no GPU): --gpus N handling (re-launch under torchrun, or fail on a WORLD_SIZE
mismatch) and the oracle sample used by cpu_baseline / --impl reference."""
import subprocess
import sys
import types

import pytest

import bench


def _args(**kw):
    d = dict(gpus=1)
    d.update(kw)
    return types.SimpleNamespace(**d)


def test_gpus_one_runs_in_process(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.maybe_relaunch(_args(gpus=1)) is False


def test_world_size_mismatch_fails(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.maybe_relaunch(_args(gpus=4))
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.maybe_relaunch(_args(gpus=4)) is False


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0
    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "3"])
    assert bench.maybe_relaunch(_args(gpus=8)) is True
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=8" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "8", "--steps", "3"]


def test_oracle_sample_counts_evals():
    import fsmt_gen
    smp = bench.OracleSample(fsmt_gen.config("cfg4s"), 200, restarts=2)
    wall, evals = smp.run(cores=1)
    assert evals == smp.n * 2 and wall > 0
