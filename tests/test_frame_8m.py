"""BASELINE.json configs[4] at full size: the 8M-point frame (lattice k=200,
b=8, sigma=10) against fixtures frozen from the UNMODIFIED reference
(tests/golden/make_golden.py --only-8m; ~90 s of reference time per frame).

`denoise` on one GPU and `denoise_slab` with P = 2, 4, 8 slab ranks (block
groups on this GPU, the same peer-memory protocol the P-GPU run uses) must
give the reference's q and S exactly, sigma_est within 1e-10, the
reference's FSLR included count, PSNR within 0.01 dB and output sums within
1e-9; the slab colours must equal the single-GPU colours bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from conftest import golden_case, golden_names, regen_input

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIGMA_RTOL = 1e-10
PSNR_TOL = 0.01
CRIT_ATOL = 1e-6
CRIT_RTOL = 1e-6

NAMES = golden_names("x8m_")


@pytest.fixture(scope="module", params=NAMES)
def frame(request):
    rec, _ = golden_case(request.param)
    clean, noisy = regen_input(rec)
    out, rep = fb.denoise(noisy)
    return rec, clean, noisy, out, rep


def _check(rec, clean, out, rep):
    r = rec["report"]
    assert rep.selected_q == r["selected_q"]
    assert rep.device["steps"] == rec["steps"]
    assert rep.sigma_est == pytest.approx(r["sigma_est"], rel=SIGMA_RTOL)
    assert rep.masked_fraction == r["masked_fraction"]
    assert rep.eligible_count == r["eligible_count"]
    assert rep.device["n_edges"] == rec["graph"]["n_edges"]
    assert rep.device["sigma_g"] == pytest.approx(rec["graph"]["sigma_g"], rel=1e-12)
    assert rep.device["included_count"] == rec["included_count"]
    np.testing.assert_allclose(rep.device["trace"], rec["trace"], rtol=CRIT_RTOL, atol=CRIT_ATOL)
    assert abs(fb.psnr(clean, out) - rec["psnr_out"]) <= PSNR_TOL
    assert out.colors.sum() == pytest.approx(rec["out_sum"], rel=1e-9)
    assert (out.colors ** 2).sum() == pytest.approx(rec["out_sumsq"], rel=1e-9)
    assert out.colors.min() >= 0.0 and out.colors.max() <= 255.0


def test_denoise_8m_matches_reference(gpu_ready, frame):
    rec, clean, noisy, out, rep = frame
    _check(rec, clean, out, rep)


@pytest.mark.parametrize("ranks,exchange", [(2, False), (4, False), (8, False), (8, True)])
def test_denoise_slab_8m_matches_reference(gpu_ready, frame, ranks, exchange):
    from paper_2401_09721_b200.slab import denoise_slab

    rec, clean, noisy, out, rep = frame
    b, rb = denoise_slab(noisy, emulate_ranks=ranks, emulate_exchange=exchange)
    _check(rec, clean, b, rb)
    assert np.array_equal(b.colors, out.colors)
