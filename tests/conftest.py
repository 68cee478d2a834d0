"""Shared fixtures: golden vectors frozen from the reference, input regeneration."""

from __future__ import annotations

import hashlib
import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA library")
    config.addinivalue_line("markers", "slow: full-size (1M point) cases")


def digest(a) -> str:
    """SHA-256 with the same canonicalisation as tests/golden/make_golden.py."""
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype("<i8")
    elif a.dtype.kind == "f":
        a = a.astype("<f8")
    elif a.dtype.kind == "b":
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


@lru_cache(maxsize=1)
def golden_index() -> dict:
    return json.loads((GOLDEN / "index.json").read_text())["cases"]


def golden_case(name: str):
    rec = golden_index()[name]
    path = GOLDEN / f"{name}.npz"
    arrays = dict(np.load(path)) if path.exists() else {}
    return rec, arrays


def golden_names(prefix: str = "", require=None):
    out = []
    for name, rec in sorted(golden_index().items()):
        if not name.startswith(prefix):
            continue
        if require and not all(k in rec for k in require):
            continue
        out.append(name)
    return out


def regen_input(rec):
    """Rebuild (clean, noisy) for a synthetic golden case and check its digests."""
    from paper_2401_09721_b200 import add_gaussian_noise, generate_cloud

    clean, _ = generate_cloud(rec["kind"], rec["n"], bits=rec["bits"], seed=rec["seed"])
    noisy = add_gaussian_noise(clean, rec["sigma"], seed=rec["noise_seed"]) \
        if rec["sigma"] > 0 else clean
    assert digest(noisy.coords) == rec["sha_coords"], "generator drifted (coords)"
    assert digest(clean.colors) == rec["sha_clean_colors"], "generator drifted (colors)"
    assert digest(noisy.colors) == rec["sha_noisy_colors"], "noise generator drifted"
    return clean, noisy


def custom_input(arrays, rec):
    from paper_2401_09721_b200 import PointCloud

    return PointCloud(arrays["coords"], arrays["colors"], rec["bit_depth"])


def cfg_kwargs(rec):
    c = dict(rec.get("cfg") or {})
    return c


@pytest.fixture(scope="session")
def gpu_ready():
    """Skip-free guard: GPU tests must fail loudly if the library is absent."""
    from paper_2401_09721_b200 import _native

    _native.load_library()
    return _native.context()
