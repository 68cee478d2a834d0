"""The NE-GBP finish on the device (FGBD_FLAG_DEVICE_NE, k_finish_noise:
covariance -> Jacobi -> tail rule -> sigma, csrc/noise.cu) against the host
C++ finish of the default path: the same moments in, bit-identical
eigenvalues, tail choices, sigma_est and q out, including glibc's hypot
reproduced on the device.  Errors keep their class and message.  The
k_mask path (FGBD_MASK_FOLD=0) is checked the same way against the folded
mask."""

from __future__ import annotations

import os
import threading

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from paper_2401_09721_b200.filtering import denoise_frame

pytestmark = pytest.mark.gpu


def _in_thread(fn, env=None):
    """Run fn in a fresh thread (its own device context, created under env)."""
    box = {}

    def run():
        old = {k: os.environ.get(k) for k in (env or {})}
        os.environ.update(env or {})
        try:
            box["r"] = fn()
        except Exception as e:  # noqa: BLE001
            box["e"] = e
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v

    t = threading.Thread(target=run)
    t.start()
    t.join()
    if "e" in box:
        raise box["e"]
    return box["r"]


CASES = [("ramp", 30_000, 10.0, {}), ("two-tone", 40_000, 20.0, {}),
         ("constant", 25_000, 15.0, {}), ("ramp", 30_000, 3.0, {"patch_size": 4}),
         ("two-tone", 30_000, 10.0, {"tau_divisor": "count_plus_one"}),
         ("constant", 20_000, 30.0, {"criterion_mode": "per_channel", "patch_size": 5}),
         ("grid", 8_000, 0.0, {})]


@pytest.mark.parametrize("kind,n,sigma,kw", CASES)
def test_device_finish_matches_host_finish(gpu_ready, kind, n, sigma, kw):
    clean, _ = fb.generate_cloud(kind, n, seed=2)
    pc = fb.add_gaussian_noise(clean, sigma, seed=5) if sigma else clean
    cfg = fb.FilterConfig(**kw)
    dev = denoise_frame(pc, cfg, device_ne=True)
    host = fb.denoise(pc, cfg)
    nofold = _in_thread(lambda: fb.denoise(pc, cfg), {"FGBD_MASK_FOLD": "0"})
    assert nofold[1].selected_q == host[1].selected_q
    assert nofold[1].masked_fraction == host[1].masked_fraction
    assert np.max(np.abs(nofold[0].colors - host[0].colors)) <= 1e-9
    (a, ra), (b, rb) = dev, host
    assert ra.sigma_est == rb.sigma_est
    assert ra.device["eigenvalues"] == rb.device["eigenvalues"]
    assert ra.device["m"] == rb.device["m"] and ra.device["tau"] == rb.device["tau"]
    assert ra.device["fallback"] == rb.device["fallback"]
    assert ra.device["jacobi_direct_off"] == rb.device["jacobi_direct_off"]
    assert ra.selected_q == rb.selected_q and ra.device["steps"] == rb.device["steps"]
    assert ra.masked_fraction == rb.masked_fraction
    assert ra.eligible_count == rb.eligible_count
    np.testing.assert_allclose(ra.device["trace"], rb.device["trace"], rtol=1e-12, atol=1e-12)
    assert np.max(np.abs(a.colors - b.colors)) <= 1e-9


def test_device_finish_errors_match_host(gpu_ready):
    """patch_size beyond 1 + max degree, and a patch size the tail rule
    rejects: same class and message on both finishes."""
    pc = fb.PointCloud([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]],
                       [[10, 20, 30], [20, 30, 40], [30, 40, 50], [40, 50, 60]], 2)
    for cfg in (fb.FilterConfig(patch_size=7), fb.FilterConfig(patch_size=2)):
        errs = []
        for dev_ne in (True, False):
            try:
                denoise_frame(pc, cfg, device_ne=dev_ne)
                errs.append(None)
            except ValueError as e:
                errs.append((type(e), str(e)))
        assert errs[0] is not None and errs[0] == errs[1]
