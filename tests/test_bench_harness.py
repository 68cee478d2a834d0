"""bench.py's multi-rank plumbing on CPU (no GPU): rank mapping, process-group
init for both backends, and the harness-check flag in the JSON config."""
import importlib.util
import os
import socket
import sys
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _load_bench(monkeypatch, shared):
    if shared:
        monkeypatch.setenv("FGBD_BENCH_SHARED_GPU", "1")
    else:
        monkeypatch.delenv("FGBD_BENCH_SHARED_GPU", raising=False)
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _args():
    return SimpleNamespace(n=1000, kind="ramp", sigma=10.0)


def test_dist_env_maps_ranks_to_devices(monkeypatch):
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("LOCAL_RANK", "3")
    b = _load_bench(monkeypatch, shared=False)
    assert b.dist_env() == (3, 4, 3)
    assert "harness_check" not in b.config_block(_args(), 4)
    assert b.config_block(_args(), 4)["parallelism"] == "frame-parallel x4"
    b = _load_bench(monkeypatch, shared=True)
    assert b.dist_env() == (3, 4, 0)
    assert "harness_check" in b.config_block(_args(), 4)


def test_init_dist_gloo_single_rank(monkeypatch):
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    for k, v in {"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": "0",
                 "WORLD_SIZE": "1"}.items():
        monkeypatch.setenv(k, v)
    b = _load_bench(monkeypatch, shared=True)
    b.init_dist(0)
    try:
        assert dist.get_backend() == "gloo" and dist.get_world_size() == 1
    finally:
        dist.destroy_process_group()


def test_init_dist_nccl_path_resolves_names(monkeypatch):
    # the NCCL branch must not depend on a module-level torch import
    b = _load_bench(monkeypatch, shared=False)
    calls = []
    import torch.distributed as dist

    monkeypatch.setattr(dist, "init_process_group", lambda *a, **k: calls.append((a, k)))
    b.init_dist(1)
    (a, k), = calls
    assert a == ("nccl",) and str(k["device_id"]) == "cuda:1"


def test_launch_plan_relaunches_without_torchrun(monkeypatch):
    b = _load_bench(monkeypatch, shared=False)
    what, cmd = b.launch_plan(4, {}, ["--gpus", "4", "--steps", "2"])
    assert what == "relaunch"
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    assert b.launch_plan(None, {}, []) == ("run", 1)
    assert b.launch_plan(1, {}, []) == ("run", 1)


def test_launch_plan_checks_world_size(monkeypatch):
    b = _load_bench(monkeypatch, shared=False)
    assert b.launch_plan(2, {"WORLD_SIZE": "2"}, []) == ("run", 2)
    assert b.launch_plan(None, {"WORLD_SIZE": "8"}, []) == ("run", 8)
    with pytest.raises(SystemExit):
        b.launch_plan(4, {"WORLD_SIZE": "2"}, [])
    with pytest.raises(SystemExit):
        b.launch_plan(0, {}, [])


def test_config_block_identical_across_arms(monkeypatch):
    b = _load_bench(monkeypatch, shared=False)
    a = SimpleNamespace(n=1000, kind="ramp", sigma=10.0, warmup=1)
    assert b.config_block(a, 1) == b.config_block(a, 1)
    assert b.warmup_steps(a) == 3
    src = (ROOT / "bench.py").read_text()
    # both arms build their config block from config_block(args, world) alone
    assert "config_block(args, world, " not in src


def test_relaunch_runs_ranks_end_to_end(tmp_path):
    """`python bench.py --gpus 2 --impl reference` without torchrun: the
    script starts 2 ranks itself; rank 0 prints the one line, with n_gpus 2."""
    import json
    import subprocess

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["FGBD_BENCH_SHARED_GPU"] = "1"
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "1", "--warmup", "0", "--n", "2000"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=tmp_path)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
