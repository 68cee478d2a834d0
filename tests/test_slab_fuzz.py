"""Seeded randomized parity of the partitioned slab path:
`denoise_slab(emulate_ranks=P)` -- every rank sorts, estimates and filters
only its z-slab, cross-slab neighbours come from the peers' block lists --
against `denoise` on the whole frame: q, S, sigma_g, the edge count and the
colours must be identical (bit for bit), on random kinds, sizes, bit depths,
point orders, duplicates, FilterConfig knobs and rank counts."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from paper_2401_09721_b200.slab import denoise_slab

pytestmark = pytest.mark.gpu


def make_case(seed):
    rng = np.random.default_rng(7000 + seed)
    kind = ["ramp", "two-tone", "constant", "grid"][seed % 4]
    n = int(rng.integers(3_000, 60_000))
    bits = None if kind != "constant" else int(rng.integers(5, 16))
    clean, _ = fb.generate_cloud(kind, n, bits=bits, seed=int(rng.integers(0, 100)))
    sigma = float(rng.choice([3.0, 10.0, 25.0]))
    noisy = fb.add_gaussian_noise(clean, sigma, seed=int(rng.integers(0, 100)))
    g, y = np.array(noisy.coords), np.array(noisy.colors)
    if seed % 3 == 1:
        p = rng.permutation(n)
        g, y = g[p], y[p]
    if seed % 5 == 2:  # duplicated points scattered through the input
        k = int(rng.integers(2, 40))
        src = rng.integers(0, n, size=k)
        dst = rng.integers(0, n, size=k)
        g[dst] = g[src]
    pc = fb.PointCloud(g, y, noisy.bit_depth)
    cfg = fb.FilterConfig(
        q_max=int(rng.choice([1, 5, 20, 64])), fslr_enabled=bool(rng.random() < 0.8),
        patch_size=int(rng.integers(3, 8)), criterion_mode=str(rng.choice(["pooled", "per_channel"])),
        early_exit=bool(rng.random() < 0.8),
        tau_divisor=str(rng.choice(["count", "count_plus_one"])))
    ranks = int(rng.integers(2, 7))
    return pc, cfg, ranks


@pytest.mark.parametrize("seed", range(32))
def test_slab_matches_denoise(gpu_ready, seed):
    pc, cfg, ranks = make_case(seed)
    z_planes = len(np.unique(np.asarray(pc.coords)[:, 2]))
    ranks = min(ranks, z_planes)
    try:
        a, ra = fb.denoise(pc, cfg)
    except ValueError as e:
        with pytest.raises(type(e)):
            denoise_slab(pc, cfg, emulate_ranks=ranks)
        return
    # odd seeds run the filter's per-step cross-rank exchange (the P-GPU
    # protocol: rank totals in peer slots, release/acquire ticks)
    b, rb = denoise_slab(pc, cfg, emulate_ranks=ranks, emulate_exchange=bool(seed & 1))
    assert rb.selected_q == ra.selected_q
    assert rb.device["steps"] == ra.device["steps"]
    assert rb.device["sigma_g"] == ra.device["sigma_g"]
    assert rb.device["n_edges"] == ra.device["n_edges"]
    assert rb.device["max_degree"] == ra.device["max_degree"]
    assert rb.masked_fraction == ra.masked_fraction
    assert rb.sigma_est == pytest.approx(ra.sigma_est, rel=1e-12)
    assert np.array_equal(a.colors, b.colors)
    # the cached path with the selected q
    c, _ = fb.denoise(pc, cfg, cached_q=ra.selected_q, cached_sigma_est=ra.sigma_est)
    d, _ = denoise_slab(pc, cfg, cached_q=ra.selected_q, cached_sigma_est=ra.sigma_est,
                        emulate_ranks=ranks, emulate_exchange=bool(seed & 1))
    assert np.array_equal(c.colors, d.colors)


def test_slab_rejects_deep_grids(gpu_ready):
    clean, _ = fb.generate_cloud("constant", 5000, bits=16, seed=0)
    with pytest.raises(ValueError):
        denoise_slab(clean, emulate_ranks=2)
