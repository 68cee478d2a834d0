"""Freeze quantize_coordinates / psnr outputs of the UNMODIFIED reference
(`fgbd.cloud`, cloud.py:89-140) into tests/golden/cloud.npz.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cloud_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import fgbd  # noqa: E402  (the reference)

OUT = Path(__file__).resolve().parent


def psnr_inputs(n: int):
    """Deterministic PSNR operands (numpy PCG64 stream, seed = n)."""
    rng = np.random.default_rng(n)
    a = rng.uniform(0, 255, size=(n, 3))
    return a, np.clip(a + rng.normal(0, 9, size=(n, 3)), 0, 255)


def main():
    rng = np.random.default_rng(2024)
    arrays = {}
    quant = {
        "float_normal": (rng.normal(size=(5000, 3)) * np.array([1.0, 1e3, 1e-4]), 10),
        "float_degenerate_axis": (np.column_stack([rng.uniform(-5, 5, 777), np.full(777, 3.25),
                                                   rng.uniform(0, 1, 777)]), 8),
        "float_halves": (np.array([[0.0, 0, 0], [2.0, 2, 2], [0.5, 1.0, 1.5],
                                   [0.25, 0.75, 1.25]]), 2),
        "float_21bit": (rng.uniform(-1e6, 1e6, size=(3000, 3)), 21),
        "int_out_of_range": (rng.integers(-500, 5000, size=(4000, 3)), 9),
        "int_passthrough": (rng.integers(0, 1 << 7, size=(1000, 3)), 7),
        "int_too_big_for_bits": (rng.integers(0, 1 << 12, size=(1000, 3)), 11),
        "single_point": (np.array([[3.5, -2.0, 7.0]]), 5),
    }
    for name, (coords, bits) in quant.items():
        pc = fgbd.PointCloud(coords, np.zeros((coords.shape[0], 3)),
                             None if coords.dtype.kind == "f" else None)
        q = fgbd.quantize_coordinates(pc, bits)
        arrays[f"{name}/in"] = coords
        arrays[f"{name}/bits"] = np.array(bits)
        arrays[f"{name}/out"] = np.asarray(q.coords)
    for n in (1, 2, 3, 5, 43, 128, 129, 1000, 33333, 300000):
        a, b = psnr_inputs(n)  # regenerated from the seed by the tests
        name = f"psnr_{n}"
        arrays[f"{name}/psnr"] = np.array(fgbd.psnr(fgbd.PointCloud(np.zeros((n, 3)), a),
                                                    fgbd.PointCloud(np.zeros((n, 3)), b)))
    np.savez_compressed(OUT / "cloud.npz", **arrays)
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
