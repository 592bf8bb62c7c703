"""bench.py host logic (no GPU): the workload per N, the Sigma-gate FP64
count of SURVEY §8(d), the self-spawn of N ranks, and the reference arm's
bounded sample (rank 0 only)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from workloads import circuits as C  # noqa: E402


def test_workload_per_world_size():
    name, n, init, gates = bench.workload_for(1, "auto")
    assert (name, n, init, len(gates)) == ("config2_random_brickwork", 24, 0, 1420)
    name, n, _, gates = bench.workload_for(8, "auto")
    assert name == "config5_random36" and n == 36  # N = 8 is config 5 itself
    assert bench.workload_for(2, "auto")[1] == 34 and bench.workload_for(4, "config2")[1] == 26


def test_sigma_gate_flops_config2():
    # 960 Haar U2 x 14 flop per amplitude; the 460 CNOTs are exact swaps (0)
    assert bench.sigma_gate_flop_per_amp(C.config2_random().gates) == 960 * 14


def test_spawn_uses_torchrun_on_localhost(monkeypatch):
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    args = type("A", (), {"gpus": 4})()
    assert bench.spawn(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]


def test_reference_arm_other_ranks_exit(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    args = type("A", (), {"gpus": 2, "steps": 3, "warmup": 3})()
    assert bench.run_reference(args) == 0
    assert capsys.readouterr().out == ""


@pytest.mark.slow
def test_reference_arm_line(monkeypatch, capsys):
    """Rank 0 prints one JSON line with impl=reference, a cpu_baseline and an
    e2e object with zero copies (a small bounded sample: 1 step)."""
    monkeypatch.setenv("RANK", "0")
    args = type("A", (), {"gpus": 1, "steps": 1, "warmup": 0})()
    assert bench.run_reference(args) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
