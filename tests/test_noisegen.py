"""add_gaussian_noise on the device (reference
cloud.py:111-123): the same variates as numpy's Generator(Philox(seed)).normal,
bit for bit.

CPU: the oracle's restatement of numpy's Philox4x64-10 + ziggurat, with the
tables of csrc/ziggurat_tables.cuh, reproduces numpy exactly (so the header
holds numpy's tables and the restated algorithm is numpy's).  GPU: the
device stream equals numpy's for sizes from 1 value to 3M values."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O

HEADER = Path(__file__).resolve().parent.parent / "paper_2401_09721_b200" / "csrc" / "ziggurat_tables.cuh"


def tables():
    src = HEADER.read_text()
    ki = [int(v, 16) for v in re.findall(r"0x([0-9a-f]{16})ull", src)]
    fl = [float.fromhex(v) for v in re.findall(r"(-?0x[0-9a-f.]+p[-+]\d+)", src)]
    assert len(ki) == 256 and len(fl) == 512
    return ki, fl[:256], fl[256:]


@pytest.mark.parametrize("seed", [0, 1, 7, 2024])
def test_oracle_stream_is_numpys(seed):
    ki, wi, fi = tables()
    raw = np.random.Philox(seed).random_raw(11)
    st0 = np.random.Philox(seed).state["state"]
    st = O.PhiloxStream(st0["counter"], st0["key"])
    assert [st.next_u64() for _ in range(11)] == [int(v) for v in raw]
    colors = np.random.default_rng(seed).uniform(0, 255, size=(4000, 3))
    got = O.gaussian_noise(colors, 12.5, seed, ki, wi, fi)
    ref = np.clip(colors + np.random.Generator(np.random.Philox(seed)).normal(0.0, 12.5, colors.shape),
                  0.0, 255.0)
    assert np.array_equal(got, ref)


def test_tables_match_numpy_build():
    """Regenerate the header's tables from numpy's libnpyrandom.a."""
    import shutil
    import subprocess
    import sys

    if not all(shutil.which(t) for t in ("ar", "nm", "objcopy")):
        pytest.skip("binutils not available")
    root = HEADER.parent.parent.parent
    before = HEADER.read_text()
    try:
        subprocess.run([sys.executable, str(root / "tools" / "gen_ziggurat_tables.py")], check=True,
                       capture_output=True)
        assert HEADER.read_text() == before
    finally:
        HEADER.write_text(before)


def test_sigma_checks_host():
    pc, _ = fb.generate_cloud("ramp", 50, seed=0)
    with pytest.raises(fb.CloudError):
        fb.add_gaussian_noise(pc, -1.0, device=True)
    assert fb.add_gaussian_noise(pc, 0.0, device=True) is pc


@pytest.mark.gpu
@pytest.mark.parametrize("n,sigma,seed", [(1, 10.0, 0), (7, 3.0, 5), (1000, 10.0, 1), (33333, 25.0, 9),
                                          (100_000, 0.5, 3), (200_000, 255.0, 4),
                                          (1_000_000, 10.0, 1)])
def test_device_noise_matches_numpy(gpu_ready, n, sigma, seed):
    pc, _ = fb.generate_cloud("ramp", n, seed=0)
    host = fb.add_gaussian_noise(pc, sigma, seed)
    dev = fb.add_gaussian_noise(pc, sigma, seed, device=True)
    bad = np.flatnonzero(host.colors.reshape(-1) != dev.colors.reshape(-1))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}"
    assert np.array_equal(host.coords, dev.coords)


@pytest.mark.gpu
def test_device_noise_many_seeds(gpu_ready):
    # ~800 exponential-tail draws per 3M values: many seeds cover the rare paths
    pc, _ = fb.generate_cloud("two-tone", 300_000, seed=0)
    for seed in range(12):
        host = fb.add_gaussian_noise(pc, 10.0, seed)
        dev = fb.add_gaussian_noise(pc, 10.0, seed, device=True)
        assert np.array_equal(host.colors, dev.colors), seed


def _glibc_log1p_model(x: float) -> float:
    """The operation order csrc/noisegen.cu's glibc_log1p uses (fdlibm
    reduction, Estrin polynomial with fused multiply-adds), in Python: fma is
    evaluated exactly with fractions and rounded once.  Main branch only."""
    import math
    import struct
    from fractions import Fraction as Fr

    def fma(a, b, c):
        return float(Fr(a) * Fr(b) + Fr(c))

    def hiword(v):
        return struct.unpack("<q", struct.pack("<d", v))[0] >> 32

    def with_hi(v, h):
        b = struct.unpack("<Q", struct.pack("<d", v))[0]
        return struct.unpack("<d", struct.pack("<Q", (b & 0xFFFFFFFF) | (h << 32)))[0]

    lp = [6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,
          2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,
          1.479819860511658591e-01]
    hx = hiword(x)
    k, hu, f, c = 1, 0, 0.0, 0.0
    if hx < 0x3FDA827A and (hx > 0 or hx <= -1076707645):
        k, f, hu = 0, x, 1
    if k:
        u = 1.0 + x
        hu = hiword(u)
        k = (hu >> 20) - 1023
        c = (1.0 - (u - x) if k > 0 else x - (u - 1.0)) / u
        hu &= 0x000FFFFF
        if hu < 0x6A09E:
            u = with_hi(u, hu | 0x3FF00000)
        else:
            k += 1
            u = with_hi(u, hu | 0x3FE00000)
            hu = (0x00100000 - hu) >> 2
        f = u - 1.0
    if hu == 0:
        return math.log1p(x)  # |f| < 2^-20: not modelled here
    hfsq = 0.5 * f * f
    s = f / (2.0 + f)
    z = s * s
    z2 = z * z
    z4 = z2 * z2
    z6 = z4 * z2
    r = fma(z, lp[0], z2 * fma(z, lp[2], lp[1]))
    r = fma(z4, fma(z, lp[4], lp[3]), r)
    r = fma(z6, fma(z, lp[6], lp[5]), r)
    t = s * (hfsq + r)
    if k == 0:
        return f - (hfsq - t)
    return k * 6.93147180369123816490e-01 - ((hfsq - (t + (k * 1.90821492927058770002e-10 + c))) - f)


def test_log1p_model_matches_host_libm():
    """The device log1p's operation order reproduces the host libm's log1p
    (which numpy's ziggurat tail calls) on the arguments the tail uses."""
    import math
    import random

    rng = random.Random(5)
    for _ in range(20000):
        u = rng.getrandbits(53) * 2.0 ** -53
        assert _glibc_log1p_model(-u) == math.log1p(-u), u
