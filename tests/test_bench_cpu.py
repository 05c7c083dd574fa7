"""bench.py host logic on CPU: the clock sampler keeps only samples taken
inside the timed region and parses clocks / throttle reasons (a fake
nvidia-smi on PATH stands in for the driver tool)."""

import os
import stat
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _fake_smi(tmp_path, clock_mhz, power_cap):
    script = tmp_path / "nvidia-smi"
    cap = "Active" if power_cap else "Not Active"
    script.write_text("#!/bin/bash\n"
                      "while true; do\n"
                      f"  echo '0, {clock_mhz}, 1965, 900.0, 0x4, Not Active, Not Active, Not Active, {cap}'\n"
                      "  sleep 0.02\n"
                      "done\n")
    script.chmod(script.stat().st_mode | stat.S_IEXEC)
    return str(tmp_path)


def test_clock_sampler_region_samples_and_reasons(tmp_path, monkeypatch):
    import bench
    monkeypatch.setenv("PATH", _fake_smi(tmp_path, 1840, True) + os.pathsep + os.environ["PATH"])
    s = bench.ClockSampler(0, period_ms=20)
    with s:
        time.sleep(0.2)
    out = s.summary()
    assert out["samples"] >= 3
    assert out["sm_mhz"] == 1840.0 and out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]


def test_clock_sampler_short_region_gets_a_sample(tmp_path, monkeypatch):
    import bench
    monkeypatch.setenv("PATH", _fake_smi(tmp_path, 1965, False) + os.pathsep + os.environ["PATH"])
    s = bench.ClockSampler(0, period_ms=20)
    with s:
        pass
    out = s.summary()
    assert out["samples"] >= 1 and out["sm_mhz"] == 1965.0 and out["reasons"] == []


def test_clock_sampler_without_nvidia_smi(monkeypatch, tmp_path):
    import bench
    monkeypatch.setenv("PATH", str(tmp_path))
    s = bench.ClockSampler(0)
    with s:
        pass
    assert s.summary()["reasons"] == ["nvidia-smi unavailable"]


def _run_bench(*args, env_extra=None, timeout=240):
    import subprocess
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def test_gpus_flag_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-executes itself as 2 ranks
    (torch.distributed.run on 127.0.0.1) that join one process group."""
    import json
    r = _run_bench("--gpus", "2", "--launch-check")
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["world"] == 2 and sorted(out["ranks"]) == [0, 1]


def test_gpus_flag_fails_loudly_without_enough_gpus():
    import torch
    if torch.cuda.device_count() >= 4:
        return
    r = _run_bench("--gpus", "4", "--steps", "1")
    assert r.returncode != 0 and "CUDA device" in (r.stderr + r.stdout)


def test_world_size_must_match_gpus():
    r = _run_bench("--gpus", "3", "--steps", "1", env_extra={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)
