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
