"""quantize_coordinates and psnr on the device against
outputs of the unmodified reference (tests/golden/make_cloud_golden.py):
both are bit-identical -- the quantised grid exactly, the PSNR to the last
bit (numpy's pairwise summation is reproduced)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
_Z = np.load(GOLD / "cloud.npz")
Z = {k: _Z[k] for k in _Z.files}
QUANT = sorted({k.split("/")[0] for k in Z if k.endswith("/in")})
PSNR = sorted({k.split("/")[0] for k in Z if k.endswith("/psnr")}, key=lambda s: int(s[5:]))


def psnr_inputs(n: int):
    rng = np.random.default_rng(n)
    a = rng.uniform(0, 255, size=(n, 3))
    return a, np.clip(a + rng.normal(0, 9, size=(n, 3)), 0, 255)


def cloud(coords, colors=None):
    colors = np.zeros((coords.shape[0], 3)) if colors is None else colors
    return fb.PointCloud(coords, colors, None)


@pytest.mark.parametrize("bits", [0, 22, -3])
def test_quantize_bad_bits(bits):
    with pytest.raises(fb.CloudError, match=r"bits must be in \[1, 21\]"):
        fb.quantize_coordinates(cloud(np.zeros((2, 3))), bits)


def test_psnr_size_mismatch():
    with pytest.raises(fb.CloudError, match="size mismatch: 2 vs 3 points"):
        fb.psnr(cloud(np.zeros((2, 3))), cloud(np.zeros((3, 3))))


@pytest.mark.gpu
@pytest.mark.parametrize("name", QUANT)
def test_quantize_matches_reference(gpu_ready, name):
    pc = cloud(Z[f"{name}/in"])
    q = fb.quantize_coordinates(pc, int(Z[f"{name}/bits"]))
    assert q.bit_depth == int(Z[f"{name}/bits"])
    assert q.coords.dtype == np.int64 and np.array_equal(q.coords, Z[f"{name}/out"])
    assert np.array_equal(q.colors, pc.colors)


@pytest.mark.gpu
def test_quantize_large_matches_oracle(gpu_ready):
    rng = np.random.default_rng(5)
    g = rng.standard_normal((2_000_000, 3)) * np.array([3.0, 0.01, 700.0]) + 12.5
    q = fb.quantize_coordinates(cloud(g), 16)
    assert np.array_equal(q.coords, O.quantize_coordinates(g, 16))
    gi = rng.integers(-(1 << 20), 1 << 20, size=(1_000_000, 3))
    assert np.array_equal(fb.quantize_coordinates(cloud(gi.astype(np.float64)), 12).coords,
                          O.quantize_coordinates(gi.astype(np.float64), 12))
    pc = fb.PointCloud(gi, np.zeros(gi.shape), None)
    assert np.array_equal(fb.quantize_coordinates(pc, 12).coords, O.quantize_coordinates(gi, 12))


@pytest.mark.gpu
@pytest.mark.parametrize("name", PSNR)
def test_psnr_bit_identical(gpu_ready, name):
    a, b = psnr_inputs(int(name[5:]))
    got = fb.psnr(cloud(np.zeros((a.shape[0], 3)), a), cloud(np.zeros((a.shape[0], 3)), b))
    assert got == float(Z[f"{name}/psnr"])


@pytest.mark.gpu
def test_psnr_cap_and_zero(gpu_ready):
    a = cloud(np.zeros((4, 3)), np.full((4, 3), 7.0))
    assert fb.psnr(a, a) == 100.0 and fb.psnr(a, a, cap_db=42.0) == 42.0
    z = cloud(np.zeros((4, 3)), np.zeros((4, 3)))
    assert fb.psnr(z, z.with_colors(np.full((4, 3), 255.0))) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [7, 8, 129, 1000, 65536 + 3, 1_000_000])
def test_psnr_vs_numpy_sizes(gpu_ready, n):
    rng = np.random.default_rng(n + 1)
    a = rng.uniform(0, 255, size=(n, 3))
    b = np.clip(a + rng.normal(0, 30, size=(n, 3)), 0, 255)
    assert fb.psnr(cloud(np.zeros((n, 3)), a), cloud(np.zeros((n, 3)), b)) == O.psnr(a, b)
