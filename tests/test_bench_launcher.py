"""bench.py's N-rank launcher (CPU, gloo): ``--gpus N`` without a torchrun
environment re-launches the script under torch.distributed.run with N ranks,
each rank maps to cuda:LOCAL_RANK, and only rank 0 prints the JSON line;
asking for more GPUs than are visible fails loudly instead of reporting a
smaller run."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def test_relaunch_two_ranks_one_json_line():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["NCCL_DEBUG"] = "WARN"
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--impl",
                          "selftest"], capture_output=True, text=True, timeout=300, env=env,
                         cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["rank"] == 0 and res["device"] == "cuda:0"
    assert res["sum"] == 3.0  # ranks 1 + 2 all-reduced


def test_too_few_gpus_fails_loudly():
    import bench
    with pytest.raises(SystemExit) as e:
        bench.check_gpus(2, 1)
    assert "only 1 CUDA device" in str(e.value)
    bench.check_gpus(2, 8)  # enough: no exit


def test_launch_command_uses_loopback_and_n_ranks():
    import bench
    cmd = bench.launch_command(4, ["--gpus", "4", "--steps", "3"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_reference_arm_falls_back_to_the_oracle_port(monkeypatch, tmp_path):
    """Without the staged reference (oracle/_ref), --impl reference still
    times the same sampled config-4 pieces, through the oracle port, and
    says so (cpu_baseline.kind == "port")."""
    import bench
    from oracle import reference
    monkeypatch.setattr(reference, "REF_DIR", tmp_path / "absent")

    class Args:
        steps, warmup = 1, 0
    res = bench.run_reference(Args)
    assert res["impl"] == "reference" and res["cpu_baseline"]["kind"] == "port"
    assert res["value"] > 0 and res["e2e"]["value"] == res["value"]
    assert res["higher_is_better"] is True and res["unit"] == bench.UNIT
