"""Large frames against the oracle: the largest sizes the CPU oracle finishes
in seconds.  A 4M-point lattice (k = 159, b = 8) with its rows shuffled, and
a 2M-point random cloud at b = 10 (64-bit sort keys are not needed, but
4 radix passes and scattered gathers are).  q and S must be identical;
sigma_est, colours and the criterion trace within the parity tolerances."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O

pytestmark = pytest.mark.gpu

COLOR_ATOL = 1e-4 * 255.0


@pytest.mark.parametrize("kind,n,shuffle", [("ramp", 4_000_000, True), ("constant", 2_000_000, False)])
def test_large_frame_matches_oracle(gpu_ready, kind, n, shuffle):
    clean, _ = fb.generate_cloud(kind, n, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    if shuffle:
        p = np.random.default_rng(5).permutation(n)
        noisy = fb.PointCloud(np.array(noisy.coords)[p], np.array(noisy.colors)[p], noisy.bit_depth)
    out, rep = fb.denoise(noisy)
    ref = O.denoise(noisy.coords, noisy.colors, noisy.bit_depth, O.OracleConfig())
    assert rep.selected_q == ref.selected_q
    assert rep.device["steps"] == ref.steps
    assert rep.sigma_est == pytest.approx(ref.sigma_est, rel=1e-10)
    assert rep.masked_fraction == ref.masked_fraction
    assert np.max(np.abs(out.colors - ref.colors)) <= COLOR_ATOL
    np.testing.assert_allclose(rep.device["trace"], ref.trace, rtol=1e-6, atol=1e-6)
