"""Brute-force kNN graph and bench-graph against graphs
and rows produced by the unmodified reference (tests/golden/make_knn_golden.py).

CPU: the oracle restatement reproduces every reference graph (pins it), and
argument errors.  GPU: the device builder is bit-identical to the reference
on every fixture (exact ties by index, duplicates, float and 17-bit
coordinates, the generic-k kernel), a 200k-point cloud is checked row by row
against the oracle on sampled vertices, and bench-graph rows reproduce the
reference's degree / overlap columns.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
INDEX = json.loads((GOLD / "knn_index.json").read_text())
_ARR = np.load(GOLD / "knn.npz")
ARR = {k: _ARR[k] for k in _ARR.files}
FIELDS = ("indptr", "indices", "csr_edge", "edge_u", "edge_v", "edge_sqdist")


def cloud(meta) -> fb.PointCloud:
    p = meta["params"]
    if p is not None:
        return fb.generate_cloud(p["kind"], p["n"], bits=p["bits"], seed=p["seed"])[0]
    coords = ARR[f"{meta['cloud']}/coords"]
    colors = np.full((coords.shape[0], 3), 100.0)
    return fb.PointCloud(coords, colors, meta["bit_depth"])


def assert_graph(g, key):
    for f in FIELDS:
        got, want = np.asarray(getattr(g, f)), ARR[f"{key}/{f}"]
        assert got.dtype == want.dtype and np.array_equal(got, want), f


@pytest.mark.parametrize("key", sorted(INDEX["graphs"]))
def test_oracle_knn_matches_reference(key):
    meta = INDEX["graphs"][key]
    pc = cloud(meta)
    if pc.n_points > 1000 and meta["k"] != 6:
        pytest.skip("oracle is O(n^2) in Python; one k per large cloud")
    assert_graph(O.build_knn_brute(pc.coords, meta["k"]), key)


@pytest.mark.parametrize("k", sorted(INDEX["errors"]))
def test_knn_argument_errors(k):
    cls, msg = INDEX["errors"][k]
    pc, _ = fb.generate_cloud("constant", 10, bits=4, seed=0)
    with pytest.raises(fb.GraphError) as ei:
        fb.build_knn_brute(pc, int(k))
    assert type(ei.value).__name__ == cls and str(ei.value) == msg


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(INDEX["graphs"]))
def test_device_knn_bit_identical(gpu_ready, key):
    meta = INDEX["graphs"][key]
    g = fb.build_knn_brute(cloud(meta), meta["k"])
    assert g.n_edges == meta["n_edges"]
    assert_graph(g, key)


@pytest.mark.gpu
def test_device_knn_large_sampled(gpu_ready):
    """200k random voxels: every sampled vertex's row is the union of its own
    k nearest and the vertices that count it among theirs."""
    pc, _ = fb.generate_cloud("constant", 200_000, bits=10, seed=9)
    k = 6
    g = fb.build_knn_brute(pc, k)
    rng = np.random.default_rng(0)
    sample = rng.choice(pc.n_points, 60, replace=False)
    mine = O.knn_rows(pc.coords, k, sample)
    for r, i in enumerate(sample):
        row = set(g.neighbors(int(i)).tolist())
        assert set(mine[r].tolist()) <= row
        others = np.array(sorted(row - set(mine[r].tolist())), np.int64)
        if others.size:
            theirs = O.knn_rows(pc.coords, k, others)
            assert all(int(i) in t for t in theirs.tolist())
    assert np.array_equal(np.diff(g.indptr), np.bincount(
        np.concatenate([g.edge_u, g.edge_v]), minlength=g.n))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(INDEX["bench"]))
def test_bench_graph_rows(gpu_ready, name):
    meta = INDEX["bench"][name]
    rows = fb.run_graph_bench(meta["sizes"], k=meta["k"], bits=meta["bits"], seed=meta["seed"])
    for got, want in zip(rows, meta["rows"]):
        assert got.n == want["n"]
        assert got.mean_degree == want["mean_degree"]
        assert got.overlap == want["overlap"]
        assert got.slg_s > 0 and got.bf_knn_s > 0
    csv = fb.rows_to_csv(rows)
    assert csv.splitlines()[0] == "n,slg_s,bf_knn_s,mean_degree,overlap"
    assert len(csv.splitlines()) == 1 + len(rows)


@pytest.mark.gpu
def test_device_stages_reject_foreign_graphs(gpu_ready):
    """The device noise / q-scan stages run on the scan-line graph: a kNN
    graph is refused loudly, the SLG rebuilt from plain arrays is accepted."""
    pc, _ = fb.generate_cloud("ramp", 2000, seed=0)
    pc = fb.add_gaussian_noise(pc, 10.0, seed=1)
    knn = fb.build_knn_brute(pc, 6)
    with pytest.raises(fb.GraphError, match="scan-line graph"):
        fb.estimate_noise_from_patches(fb.extract_patches(pc, knn, 3))
    slg = fb.build_weighted_slg(pc)
    plain = fb.Graph(slg.n, slg.indptr, slg.indices, slg.csr_edge, slg.edge_u, slg.edge_v,
                     slg.edge_sqdist, slg.sigma_g, slg.edge_weights)
    a = fb.estimate_noise_from_patches(fb.extract_patches(pc, slg, 7))
    b = fb.estimate_noise_from_patches(fb.extract_patches(pc, plain, 7))
    assert a.sigma_est == b.sigma_est
    bent = fb.Graph(slg.n, slg.indptr, slg.indices, slg.csr_edge, slg.edge_u, slg.edge_v,
                    slg.edge_sqdist, slg.sigma_g, slg.edge_weights * 0.5)
    with pytest.raises(fb.GraphError, match="scan-line graph"):
        fb.select_q(pc, bent, a.sigma_est, fb.FilterConfig())
    # any CSR graph filters
    wk = fb.apply_gaussian_weights(knn, fb.compute_sigma_g(pc, knn))
    out = fb.apply_filter(wk, pc.colors, 2)
    ok = O.OracleGraph(knn.n, knn.indptr, knn.indices, knn.csr_edge, knn.edge_u, knn.edge_v,
                       knn.edge_sqdist, wk.sigma_g, np.asarray(wk.edge_weights))
    want = O.EllOperator(ok).step(O.EllOperator(ok).step(pc.colors))
    assert np.array_equal(out, want)
