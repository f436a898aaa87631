"""bench.py's launch contract on CPU: --gpus N is never
ignored -- without WORLD_SIZE it re-launches itself under torch.distributed.run
with N ranks, and a WORLD_SIZE that disagrees with --gpus is an error."""

import sys

import pytest

import bench


def test_gpus_n_respawns_under_torchrun(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env=None: calls.append((cmd, env)) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    (cmd, env), = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]
    assert env["NCCL_DEBUG"] == "INFO"


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "WORLD_SIZE=2" in str(e.value.code)


def test_single_gpu_runs_in_process(monkeypatch):
    ran = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench, "run_b200", lambda a: ran.append(a.gpus))
    monkeypatch.setattr(bench, "respawn", lambda a: pytest.fail("N=1 must not respawn"))
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    bench.main()
    assert ran == [1]
