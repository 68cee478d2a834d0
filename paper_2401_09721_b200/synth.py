"""Deterministic synthetic frames for tests and benchmarks (host numpy).

Produces byte-identical clouds to the reference generator (synth.py:25-69)
so the B200 path and the CPU reference see the same inputs; the golden
fixtures pin this with SHA-256 digests (tests/test_oracle.py).

kinds:
  constant  uniform random voxels (Philox(seed)), mid-grey everywhere
  grid      first n points of the k^3 raster lattice, mid-grey
  ramp      lattice, colour 120 + 16 * coord / (k - 1) per channel
  two-tone  lattice, tone B inside the slab k//3 <= x < 2k//3, tone A outside
"""

from __future__ import annotations

import numpy as np

from .cloud import MAX_BIT_DEPTH, PointCloud
from .errors import CloudError

KINDS = ("constant", "ramp", "two-tone", "grid")
MID_GRAY = (128.0, 128.0, 128.0)
TONE_A = (192.0, 64.0, 64.0)
TONE_B = (64.0, 64.0, 192.0)


def lattice_side(n: int) -> int:
    k = max(1, int(round(n ** (1.0 / 3.0))))
    while k ** 3 < n:
        k += 1
    while k > 1 and (k - 1) ** 3 >= n:
        k -= 1
    return k


def _raster_lattice(n: int):
    """(x, y, z) of the first n raster positions of a k^3 cube, x fastest."""
    k = lattice_side(n)
    i = np.arange(n, dtype=np.int64)
    x = i % k
    y = (i // k) % k
    z = i // (k * k)
    return np.stack([x, y, z], axis=1), k


def generate_cloud(kind: str, n: int, bits: int | None = None, seed: int = 0):
    """Return (PointCloud, labels-or-None); labels only for two-tone."""
    if n < 1:
        raise CloudError(f"n must be >= 1, got {n}")
    if kind not in KINDS:
        raise CloudError(f"unknown synthetic kind {kind!r}; choose from {KINDS}")
    if kind == "constant":
        b = 10 if bits is None else int(bits)
        if not 1 <= b <= MAX_BIT_DEPTH:
            raise CloudError(f"bits must be in [1, {MAX_BIT_DEPTH}], got {bits}")
        gen = np.random.Generator(np.random.Philox(int(seed)))
        coords = gen.integers(0, 1 << b, size=(n, 3), dtype=np.int64)
        return PointCloud(coords, np.full((n, 3), MID_GRAY[0]), b), None

    coords, k = _raster_lattice(n)
    b = max(1, (k - 1).bit_length()) if bits is None else int(bits)
    if k > (1 << b):
        raise CloudError(f"lattice of side {k} does not fit in {b} bits")
    if kind == "grid":
        return PointCloud(coords, np.full((n, 3), MID_GRAY[0]), b), None
    if kind == "ramp":
        span = float(max(k - 1, 1))
        return PointCloud(coords, 120.0 + 16.0 * coords.astype(np.float64) / span, b), None
    inside = (coords[:, 0] >= k // 3) & (coords[:, 0] < 2 * k // 3)
    colors = np.where(inside[:, None], np.array(TONE_B), np.array(TONE_A))
    return PointCloud(coords, colors.astype(np.float64), b), inside.astype(np.int64)
