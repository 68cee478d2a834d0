"""CPU suite: pin the oracle (oracle/fgbd_oracle.py) to the reference.

1. SPEC.md known-answer examples (the reference's only golden vectors).
2. Oracle vs fixtures frozen from the unmodified reference
   (tests/golden/make_golden.py): structure, weights, patches, eigenvalues,
   mask, criterion trace, q, S and output colours -- bit-exact, because the
   oracle evaluates the same floating-point expressions in the same order.
3. The synthetic generator in the package reproduces the reference's bytes.
"""

from __future__ import annotations

import math

from pathlib import Path

import numpy as np
import pytest

from conftest import cfg_kwargs, custom_input, digest, golden_case, golden_names, regen_input
from oracle import fgbd_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def psnr_inputs(n: int):
    """Same operands as tests/golden/make_cloud_golden.py (seed = n)."""
    rng = np.random.default_rng(n)
    a = rng.uniform(0, 255, size=(n, 3))
    return a, np.clip(a + rng.normal(0, 9, size=(n, 3)), 0, 255)

# ---------------------------------------------------------------------------
# SPEC known answers
# ---------------------------------------------------------------------------


def test_spec_scanline_codes():
    g = np.array([[1, 2, 3]])
    assert O.scanline_codes(g, 4, 1)[0] == 801
    assert O.scanline_codes(g, 4, 2)[0] == 306
    assert O.scanline_codes(g, 4, 3)[0] == 531
    z = np.zeros((1, 3), np.int64)
    assert all(O.scanline_codes(z, 4, l)[0] == 0 for l in (1, 2, 3))


def test_spec_radix_argsort():
    assert O.radix_argsort(np.array([5, 2, 9], np.uint64)).tolist() == [1, 0, 2]
    assert O.radix_argsort(np.full(17, 7, np.uint64)).tolist() == list(range(17))
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 2 ** 63, size=100_000, dtype=np.uint64)
    keys[::7] = keys[3]  # ties
    assert np.array_equal(O.radix_argsort(keys), np.argsort(keys, kind="stable"))


def test_spec_slg_small():
    g2 = O.build_slg(np.array([[0, 0, 0], [1, 1, 1]]), 1)
    assert list(zip(g2.edge_u, g2.edge_v)) == [(0, 1)]
    assert g2.degrees().tolist() == [1, 1]
    g3 = O.build_slg(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]]), 2)
    assert list(zip(g3.edge_u, g3.edge_v)) == [(0, 1), (1, 2)]
    assert g3.degrees().max() == 2


def test_spec_sigma_and_weights():
    g = O.build_slg(np.array([[0, 0, 0], [1, 0, 0], [4, 0, 0]]), 3)
    assert O.compute_sigma_g(g) == 2.0
    g1 = O.build_weighted_slg(np.array([[0, 0, 0], [1, 0, 0]]), 1)
    assert g1.edge_weights[0] == pytest.approx(math.exp(-1))  # SPEC: e^-1
    gd = O.build_slg(np.array([[0, 0, 0], [0, 0, 0], [2, 0, 0]]), 2)
    O.apply_gaussian_weights(gd, 1.0)
    assert gd.edge_weights[0] == 1.0                          # coincident -> 1


def test_spec_filter_step_two_nodes():
    g = O.build_weighted_slg(np.array([[0, 0, 0], [1, 0, 0]]), 1)
    out = O.EllOperator(g).step(np.array([[0.0], [100.0]]))
    assert out[:, 0].tolist() == [50.0, 50.0]


def test_spec_patch_order():
    coords = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]])
    g = O.build_weighted_slg(coords, 2)
    colors = np.array([[10.0, 0, 0], [20.0, 0, 0], [30.0, 0, 0]])
    vec, elig = O.extract_patches(colors, g, 3)
    row = int(np.flatnonzero(elig == 1)[0])
    assert vec[0, row].tolist() == [20.0, 10.0, 30.0]


def test_spec_covariance_eigen_tail():
    x = np.array([[0.0, 0.0], [2.0, 2.0]])
    assert O.patch_covariance(x).tolist() == [[1.0, 1.0], [1.0, 1.0]]
    assert O.symmetric_eigenvalues(np.diag([2.0, 1.0])).tolist() == [2.0, 1.0]
    lam = O.symmetric_eigenvalues(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert lam == pytest.approx([2.0, 0.0], abs=1e-12)
    m, tau, fb = O.select_tail(np.array([50, 2.0, 1.0, 0.9, 0.8, 0.7, 0.6]))
    assert (m, fb) == (1, False) and tau == pytest.approx(1.0)
    m, tau, fb = O.select_tail(np.full(7, 4.0))
    assert (m, fb) == (3, True) and tau == 4.0


def test_spec_criterion_and_spectral():
    y = np.array([[10.0]])
    x = np.array([[6.0]])
    assert O.selection_criterion(y, x, np.ones(1, bool), 8.0) == 0.0
    assert O.selection_criterion(y, y, np.ones(1, bool), 0.0) == 0.0


def test_spec_psnr_and_quantize():
    a = np.full((4, 3), 7.0)
    assert O.psnr(a, a) == 100.0
    assert O.psnr(np.zeros((4, 3)), np.full((4, 3), 255.0)) == 0.0
    q = O.quantize_coordinates(np.array([[0.0, 0, 0], [1.0, 0, 0]]), 4)
    assert q[:, 0].tolist() == [0, 15] and q[:, 1].tolist() == [0, 0]
    assert O.quantize_coordinates(np.array([[0, 1, 2], [3, 4, 5]]), 3) is None


def test_oracle_quantize_and_psnr_match_reference_fixture():
    """Pinned to outputs of the reference's cloud.py (tests/golden/cloud.npz)."""
    z = np.load(GOLDEN / "cloud.npz")
    for name in sorted({k.split("/")[0] for k in z.files if k.endswith("/in")}):
        got = O.quantize_coordinates(z[f"{name}/in"], int(z[f"{name}/bits"]))
        want = z[f"{name}/out"]
        assert np.array_equal(z[f"{name}/in"] if got is None else got, want), name
    for name in sorted({k.split("/")[0] for k in z.files if k.endswith("/psnr")}):
        a, b = psnr_inputs(int(name.split("_")[1]))
        assert O.psnr(a, b) == float(z[f"{name}/psnr"]), name


def test_eigensolver_suite_oracle():
    """SPEC acceptance 7: trace identity + characteristic polynomial residual."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        a = rng.standard_normal((7, 7))
        s = (a + a.T) / 2
        lam = O.symmetric_eigenvalues(s)
        assert np.all(np.diff(lam) <= 1e-12)
        assert lam.sum() == pytest.approx(np.trace(s), rel=1e-9, abs=1e-9)
        norm = np.linalg.norm(s)
        for l in lam:
            assert abs(np.linalg.det(s - l * np.eye(7))) < 1e-6 * norm ** 7


# ---------------------------------------------------------------------------
# oracle vs the reference's frozen outputs
# ---------------------------------------------------------------------------

FULL = [n for n in golden_names("s5k_")] + [n for n in golden_names("rand_")] + \
    [n for n in golden_names("tiny_")]


def _oracle_cfg(rec):
    c = cfg_kwargs(rec)
    return O.OracleConfig(**c) if c else O.OracleConfig()


@pytest.mark.parametrize("name", FULL)
def test_oracle_graph_matches_reference(name):
    rec, arr = golden_case(name)
    pc = custom_input(arr, rec) if "coords" in arr else regen_input(rec)[1]
    b = rec["bit_depth"]
    for line in (1, 2, 3):
        assert np.array_equal(O.sort_permutation(pc.coords, b, line), arr[f"perm{line}"])
    g = O.build_slg(pc.coords, b)
    for key in ("indptr", "indices", "csr_edge", "edge_u", "edge_v", "edge_sqdist"):
        assert np.array_equal(getattr(g, key), arr[key]), key
    if g.n_edges:
        sg = O.compute_sigma_g(g)
        assert sg == rec["graph"]["sigma_g"]
        O.apply_gaussian_weights(g, sg)
        assert np.array_equal(g.edge_weights, arr["edge_weights"])
        assert np.array_equal(g.weighted_degrees(), arr["weighted_degrees"])


@pytest.mark.parametrize("name", [n for n in FULL if "patch_vectors" in golden_case(n)[1]])
def test_oracle_patches_match_reference(name):
    rec, arr = golden_case(name)
    pc = custom_input(arr, rec) if "coords" in arr else regen_input(rec)[1]
    g = O.build_weighted_slg(pc.coords, rec["bit_depth"])
    vec, elig = O.extract_patches(pc.colors, g, 7)
    assert np.array_equal(elig, arr["patch_point_index"])
    assert np.array_equal(vec, arr["patch_vectors"])
    assert np.array_equal(O.fslr_stat(vec), arr["fslr_stat"])
    est = O.estimate_noise_from_patches(vec)
    assert est.sigma_est == rec["noise"]["sigma_est"]
    assert np.array_equal(est.eigenvalues, np.array(rec["noise"]["eigenvalues"]))


def _check_denoise(rec, arr, res):
    rep = rec["report"]
    assert res.selected_q == rep["selected_q"]
    if not rec.get("cached_q") and rec.get("cached_q") != 0:
        assert res.steps == rec["steps"]
    assert res.sigma_est == rep["sigma_est"]
    assert res.masked_fraction == rep["masked_fraction"]
    if "criterion_value" in rep:
        assert res.criterion_value == rep["criterion_value"]
        assert res.converged == rep["converged"]
        assert res.trace == rec["trace"]
    if "include_bits" in arr:
        assert np.array_equal(np.packbits(res.include), arr["include_bits"])
    if "out_colors" in arr:
        assert np.array_equal(res.colors, arr["out_colors"])
    if "out_colors_f32" in arr:
        assert np.array_equal(res.colors.astype(np.float32), arr["out_colors_f32"])
    if "sha_out_colors" in rec:
        assert digest(res.colors) == rec["sha_out_colors"]


DENOISE_CASES = [n for n in golden_names(require=["report"])
                 if not n.startswith(("x1m_", "checker"))]


@pytest.mark.parametrize("name", DENOISE_CASES)
def test_oracle_denoise_matches_reference(name):
    rec, arr = golden_case(name)
    pc = custom_input(arr, rec) if "coords" in arr else regen_input(rec)[1]
    res = O.denoise(pc.coords, pc.colors, rec["bit_depth"], _oracle_cfg(rec),
                    cached_q=rec.get("cached_q"), cached_sigma_est=rec.get("cached_sigma"))
    _check_denoise(rec, arr, res)


@pytest.mark.parametrize("name", [n for n in golden_names(require=["denoise_error"])])
def test_oracle_errors_match_reference(name):
    rec, arr = golden_case(name)
    pc = custom_input(arr, rec) if "coords" in arr else regen_input(rec)[1]
    with pytest.raises(O.OracleError) as ei:
        O.denoise(pc.coords, pc.colors, rec["bit_depth"], _oracle_cfg(rec))
    assert str(ei.value) in rec["denoise_error"]


def test_oracle_all_excluded_fallback():
    rec, arr = golden_case("checker_all_excluded")
    with pytest.warns(UserWarning, match="excluded every point"):
        res = O.denoise(arr["coords"], arr["noisy_colors"], 3, O.OracleConfig(patch_size=3))
    assert res.all_excluded_fallback and rec["all_excluded_warning"]
    assert res.selected_q == rec["report"]["selected_q"]
    assert res.trace == rec["trace"]
    assert np.array_equal(res.colors, arr["out_colors"])


@pytest.mark.parametrize("name", golden_names(require=["sha_noisy_colors"]))
def test_generator_reproduces_reference_inputs(name):
    regen_input(golden_case(name)[0])


def test_oracle_ell_step_equals_scipy_csr():
    """The ELL restatement of filter_step is bit-identical to scipy's CSR matvec."""
    sparse = pytest.importorskip("scipy.sparse")
    rec, arr = golden_case("s5k_constant_s10")
    pc = regen_input(rec)[1]
    g = O.build_weighted_slg(pc.coords, rec["bit_depth"])
    w = sparse.csr_matrix((g.csr_weights(), g.indices, g.indptr), shape=(g.n, g.n))
    d = g.weighted_degrees()[:, None]
    ref = (d * pc.colors + w @ pc.colors) / (2.0 * d)
    assert np.array_equal(O.EllOperator(g).step(pc.colors), ref)


def test_ell_view_equals_csr_matvec():
    """The oracle's step calls scipy's CSR matvec; the padded-row (ELL)
    accumulation in slot order from 0.0 gives the same bits."""
    rng = np.random.default_rng(4)
    coords = rng.integers(0, 16, size=(3000, 3))
    g = O.build_weighted_slg(coords, 4)
    op = O.EllOperator(g)
    f = rng.uniform(0, 255, size=(3000, 3))
    idx, w = op.dense_rows()
    acc = np.zeros_like(f)
    for s in range(idx.shape[1]):
        acc = acc + w[:, s, None] * f[idx[:, s]]
    assert np.array_equal(acc, op.W @ f)
