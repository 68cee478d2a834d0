"""Freeze golden vectors by running the UNMODIFIED reference `fgbd` here.

Run in the build container only (the reference tree does not exist on the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--skip-1m]

Writes tests/golden/*.npz plus index.json.  Every fixture records the
generator parameters and SHA-256 digests of the input arrays, so a test can
regenerate the input with `paper_2401_09721_b200.synth` and prove it is the
same byte stream before comparing outputs.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
import warnings
from pathlib import Path

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

import fgbd  # noqa: E402  (the reference)
import fgbd.filtering as ref_filtering  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype("<i8")
    elif a.dtype.kind == "f":
        a = a.astype("<f8")
    elif a.dtype.kind == "b":
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


def make_input(kind, n, bits, seed, sigma, noise_seed):
    clean, _ = fgbd.generate_cloud(kind, n, bits=bits, seed=seed)
    noisy = fgbd.add_gaussian_noise(clean, sigma, seed=noise_seed) if sigma > 0 else clean
    return clean, noisy


def run_reference(noisy, cfg, cached_q=None, cached_sigma=None):
    """denoise() with the criterion curve and the number of filter steps recorded."""
    trace = []
    steps = [0]
    real_crit = ref_filtering.selection_criterion
    real_step = ref_filtering.filter_step
    in_select = [False]

    def crit(*a, **k):
        v = real_crit(*a, **k)
        if in_select[0]:
            trace.append(v)
        return v

    def step(*a, **k):
        if in_select[0]:
            steps[0] += 1
        return real_step(*a, **k)

    real_select = ref_filtering.select_q

    def select(*a, **k):
        in_select[0] = True
        try:
            return real_select(*a, **k)
        finally:
            in_select[0] = False

    ref_filtering.selection_criterion = crit
    ref_filtering.filter_step = step
    ref_filtering.select_q = select
    try:
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            t0 = time.perf_counter()
            out, rep = ref_filtering.denoise(noisy, cfg, cached_q=cached_q,
                                             cached_sigma_est=cached_sigma)
            dt = time.perf_counter() - t0
        warned = any("excluded every point" in str(x.message) for x in w)
    finally:
        ref_filtering.selection_criterion = real_crit
        ref_filtering.filter_step = real_step
        ref_filtering.select_q = real_select
    return out, rep, np.array(trace), steps[0], warned, dt


def graph_record(noisy, full: bool):
    g = fgbd.build_slg(noisy)
    sg = fgbd.compute_sigma_g(noisy, g) if g.n_edges else 0.0
    rec = {
        "n_edges": int(g.n_edges),
        "nnz": int(g.indices.size),
        "max_degree": int(np.diff(g.indptr).max(initial=0)),
        "sigma_g": float(sg),
        "sha_indptr": digest(g.indptr),
        "sha_indices": digest(g.indices),
        "sha_csr_edge": digest(g.csr_edge),
        "sha_edge_u": digest(g.edge_u),
        "sha_edge_v": digest(g.edge_v),
        "sha_edge_sqdist": digest(g.edge_sqdist),
    }
    arrays = {}
    if full:
        arrays = dict(indptr=g.indptr, indices=g.indices, csr_edge=g.csr_edge,
                      edge_u=g.edge_u, edge_v=g.edge_v, edge_sqdist=g.edge_sqdist)
        for line in (1, 2, 3):
            arrays[f"perm{line}"] = fgbd.sort_permutation(fgbd.scanline_codes(noisy, line))
        if g.n_edges:
            gw = fgbd.apply_gaussian_weights(g, sg)
            arrays["edge_weights"] = gw.edge_weights
            arrays["weighted_degrees"] = gw.weighted_degrees()
    return rec, arrays


def noise_record(noisy, cfg, full: bool):
    g = fgbd.build_weighted_slg(noisy)
    patches = fgbd.extract_patches(noisy, g, cfg.patch_size)
    est = fgbd.estimate_noise_from_patches(patches, cfg.tau_divisor)
    rec = {
        "sigma_est": float(est.sigma_est),
        "per_channel_sigma": est.per_channel_sigma.tolist(),
        "eigenvalues": est.eigenvalues.tolist(),
        "m": est.m.tolist(),
        "tau": est.tau.tolist(),
        "fallback": est.fallback.tolist(),
        "eligible_count": int(est.eligible_count),
        "covariance": [fgbd.patch_covariance(patches, c).tolist() for c in range(3)],
    }
    stat = patches.vectors.std(axis=2).mean(axis=0)
    arrays = {}
    if full:
        arrays["patch_point_index"] = patches.point_index
        arrays["patch_vectors"] = patches.vectors
        arrays["fslr_stat"] = stat
    return rec, arrays


def case(name, kind, n, sigma, *, bits=None, seed=0, noise_seed=1, cfg=None,
         full=False, colors="f32", cached_q=None, cached_sigma=None, index=None):
    cfg = cfg or fgbd.FilterConfig()
    clean, noisy = make_input(kind, n, bits, seed, sigma, noise_seed)
    rec = {
        "name": name, "kind": kind, "n": n, "bits": bits, "seed": seed,
        "sigma": sigma, "noise_seed": noise_seed,
        "bit_depth": int(noisy.bit_depth),
        "cfg": {k: getattr(cfg, k) for k in (
            "q_max", "epsilon", "fslr_enabled", "patch_size", "reestimate_interval",
            "fslr_sigma_floor", "criterion_mode", "early_exit", "tau_divisor")},
        "cached_q": cached_q, "cached_sigma": cached_sigma,
        "sha_coords": digest(noisy.coords),
        "sha_clean_colors": digest(clean.colors),
        "sha_noisy_colors": digest(noisy.colors),
    }
    arrays = {}
    grec, garr = graph_record(noisy, full)
    rec["graph"] = grec
    arrays.update(garr)
    if cached_q is None and n >= 2:
        try:
            nrec, narr = noise_record(noisy, cfg, full)
            rec["noise"] = nrec
            arrays.update(narr)
        except ValueError as e:
            rec["noise_error"] = f"{type(e).__name__}: {e}"
    try:
        out, rep, trace, steps, warned, dt = run_reference(noisy, cfg, cached_q, cached_sigma)
    except ValueError as e:
        rec["denoise_error"] = f"{type(e).__name__}: {e}"
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        index[name] = rec
        print(f"{name}: error {rec['denoise_error']}")
        return
    rec["report"] = {k: v for k, v in rep.to_dict().items() if k != "stage_timings"}
    rec["steps"] = int(steps)
    rec["trace"] = trace.tolist()
    rec["all_excluded_warning"] = bool(warned)
    rec["ref_seconds"] = dt
    rec["psnr_noisy"] = float(fgbd.psnr(clean, noisy))
    rec["psnr_out"] = float(fgbd.psnr(clean, out))
    rec["sha_out_colors"] = digest(out.colors)
    rec["out_sum"] = float(np.sum(out.colors, dtype=np.float64))
    rec["out_sumsq"] = float(np.sum(out.colors.astype(np.float64) ** 2))
    if cached_q is None and n >= 2 and "noise" in rec:
        g = fgbd.build_weighted_slg(noisy)
        patches = fgbd.extract_patches(noisy, g, cfg.patch_size)
        if cfg.fslr_enabled:
            try:
                mask = fgbd.fslr_mask(patches, rec["noise"]["sigma_est"], cfg.fslr_sigma_floor)
                inc = mask.include
            except fgbd.AllPointsExcludedError:
                inc = np.ones(n, bool)
        else:
            inc = np.ones(n, bool)
        arrays["include_bits"] = np.packbits(inc)
        rec["included_count"] = int(inc.sum())
    if colors == "f64":
        arrays["out_colors"] = out.colors
    elif colors == "f32":
        arrays["out_colors_f32"] = out.colors.astype(np.float32)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    index[name] = rec
    print(f"{name}: q={rep.selected_q} S={steps} sigma_est={rep.sigma_est:.6f} "
          f"E={grec['n_edges']} t={dt:.2f}s warn={warned}")


def checker_case(index):
    """Checkerboard lattice + weak noise, D=3: FSLR excludes every point."""
    k = 8
    i = np.arange(k ** 3)
    coords = np.stack([i % k, (i // k) % k, i // (k * k)], axis=1)
    par = (coords.sum(axis=1) % 2).astype(np.float64)
    colors = np.repeat((par * 255.0)[:, None], 3, axis=1)
    clean = fgbd.PointCloud(coords, colors, 3)
    noisy = fgbd.add_gaussian_noise(clean, 1.0, seed=7)
    cfg = fgbd.FilterConfig(patch_size=3)
    out, rep, trace, steps, warned, _ = run_reference(noisy, cfg)
    np.savez_compressed(OUT / "checker_all_excluded.npz", coords=coords,
                        noisy_colors=noisy.colors, out_colors=out.colors)
    index["checker_all_excluded"] = {
        "name": "checker_all_excluded", "bit_depth": 3, "cfg_patch_size": 3,
        "report": {k2: v for k2, v in rep.to_dict().items() if k2 != "stage_timings"},
        "steps": int(steps), "trace": trace.tolist(), "all_excluded_warning": bool(warned),
    }
    print(f"checker: q={rep.selected_q} warn={warned} masked={rep.masked_fraction}")


def custom_case(name, coords, colors, bits, index, cfg=None):
    """Hand-built tiny clouds: full arrays of everything."""
    cfg = cfg or fgbd.FilterConfig()
    pc = fgbd.PointCloud(np.asarray(coords), np.asarray(colors, float), bits)
    rec = {"name": name, "bit_depth": bits, "n": pc.n_points,
           "cfg": {k: getattr(cfg, k) for k in (
               "q_max", "epsilon", "fslr_enabled", "patch_size", "reestimate_interval",
               "fslr_sigma_floor", "criterion_mode", "early_exit", "tau_divisor")}}
    grec, garr = graph_record(pc, True)
    rec["graph"] = grec
    arrays = dict(coords=pc.coords, colors=pc.colors, **garr)
    try:
        out, rep, trace, steps, warned, _ = run_reference(pc, cfg)
        rec["report"] = {k: v for k, v in rep.to_dict().items() if k != "stage_timings"}
        rec["steps"] = int(steps)
        rec["trace"] = trace.tolist()
        arrays["out_colors"] = out.colors
    except ValueError as e:
        rec["denoise_error"] = f"{type(e).__name__}: {e}"
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    index[name] = rec
    print(f"{name}: {rec.get('report', rec.get('denoise_error'))}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-1m", action="store_true")
    ap.add_argument("--only-8m", action="store_true",
                    help="add the configs[4] 8M frames to the existing index.json")
    args = ap.parse_args()
    index: dict = {}
    if args.only_8m:
        main_8m()
        return

    # warm the numba JIT so recorded times are not compile times
    w, _ = fgbd.generate_cloud("ramp", 1000)
    fgbd.denoise(fgbd.add_gaussian_noise(w, 10, seed=1))

    rng = np.random.default_rng(2024)
    # tiny hand-built clouds (SPEC examples and degenerate inputs)
    custom_case("tiny_two_points", [[0, 0, 0], [1, 1, 1]], [[0, 0, 0], [100, 100, 100]], 1, index)
    custom_case("tiny_collinear", [[0, 0, 0], [1, 0, 0], [2, 0, 0]],
                [[10, 20, 30], [20, 30, 40], [30, 40, 50]], 2, index)
    custom_case("tiny_duplicates", rng.integers(0, 2, size=(12, 3)),
                rng.uniform(0, 255, size=(12, 3)), 1, index)
    custom_case("tiny_collinear_d3", [[0, 0, 0], [1, 0, 0], [2, 0, 0]],
                [[10, 20, 30], [20, 30, 40], [30, 40, 50]], 2, index,
                cfg=fgbd.FilterConfig(patch_size=3))
    custom_case("tiny_duplicates_d3", rng.integers(0, 2, size=(12, 3)),
                rng.uniform(0, 255, size=(12, 3)), 1, index,
                cfg=fgbd.FilterConfig(patch_size=3))
    custom_case("rand_b4_500", rng.integers(0, 16, size=(500, 3)),
                np.clip(128 + 20 * rng.standard_normal((500, 3)), 0, 255), 4, index)
    custom_case("rand_b3_1000_dups", rng.integers(0, 8, size=(1000, 3)),
                np.clip(100 + 30 * rng.standard_normal((1000, 3)), 0, 255), 3, index)
    custom_case("rand_b12_3000", rng.integers(0, 4096, size=(3000, 3)),
                np.clip(128 + 10 * rng.standard_normal((3000, 3)), 0, 255), 12, index)
    custom_case("rand_b21_2000", rng.integers(0, 1 << 21, size=(2000, 3)),
                np.clip(128 + 10 * rng.standard_normal((2000, 3)), 0, 255), 21, index)
    checker_case(index)

    # small synthetic frames with every array frozen
    for kind in ("ramp", "two-tone", "constant"):
        case(f"s5k_{kind}_s10", kind, 5000, 10.0, full=True, colors="f64", index=index)
    case("s5k_grid_s0", "grid", 5000, 0.0, full=True, colors="f64", index=index)
    case("s5k_constant_b6_s10", "constant", 5000, 10.0, bits=6, full=True, colors="f64", index=index)

    # 20k sigma sweep (config 3 at desk scale)
    for kind in ("ramp", "two-tone", "constant"):
        for sigma in (5.0, 10.0, 20.0, 30.0):
            case(f"m20k_{kind}_s{int(sigma)}", kind, 20000, sigma, index=index)
        case(f"m20k_{kind}_s10_seed1", kind, 20000, 10.0, seed=1, noise_seed=2,
             colors=None, index=index)
    # FilterConfig variants (every knob of filtering.py:33-59)
    variants = {
        "per_channel": fgbd.FilterConfig(criterion_mode="per_channel"),
        "count_plus_one": fgbd.FilterConfig(tau_divisor="count_plus_one"),
        "no_fslr": fgbd.FilterConfig(fslr_enabled=False),
        "no_early_exit": fgbd.FilterConfig(early_exit=False),
        "qmax5": fgbd.FilterConfig(q_max=5),
        "qmax0": fgbd.FilterConfig(q_max=0),
        "patch4": fgbd.FilterConfig(patch_size=4),
        "patch3": fgbd.FilterConfig(patch_size=3),
        "patch2": fgbd.FilterConfig(patch_size=2),
        "patch8": fgbd.FilterConfig(patch_size=8),
        "floor100": fgbd.FilterConfig(fslr_sigma_floor=100.0),
        "eps": fgbd.FilterConfig(epsilon=5.0),
    }
    for vname, cfg in variants.items():
        case(f"v20k_two-tone_s20_{vname}", "two-tone", 20000, 20.0, cfg=cfg, index=index)
    case("v20k_constant_s20_per_channel", "constant", 20000, 20.0,
         cfg=variants["per_channel"], index=index)
    case("c20k_ramp_s10_cached7", "ramp", 20000, 10.0, cached_q=7, cached_sigma=9.5,
         index=index)
    case("c20k_ramp_s10_cached0", "ramp", 20000, 10.0, cached_q=0, index=index)

    # config 1: 100k on CPU
    for kind in ("ramp", "two-tone", "constant"):
        case(f"l100k_{kind}_s10", kind, 100_000, 10.0, colors=None, index=index)

    if not args.skip_1m:
        # config 2 / 3: 1M frames, scalars + digests only
        for kind in ("ramp", "two-tone", "constant"):
            case(f"x1m_{kind}_s10", kind, 1_000_000, 10.0, colors=None, index=index)
        for sigma in (5.0, 20.0, 30.0):
            case(f"x1m_ramp_s{int(sigma)}", "ramp", 1_000_000, sigma, colors=None, index=index)
        case("x1m_ramp_s10_cached64", "ramp", 1_000_000, 10.0, cached_q=64,
             cached_sigma=10.0, colors=None, index=index)

    meta = {
        "generated_by": "tests/golden/make_golden.py",
        "reference": REF_SRC,
        "numpy": np.__version__,
        "cases": index,
    }
    (OUT / "index.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


def main_8m():
    """configs[4]: the 8M frame (k=200 lattice, b=8), scalars + digests only.

    The reference takes ~2-3 min per frame here.  Appended to index.json so
    the smaller fixtures are not regenerated.
    """
    meta = json.loads((OUT / "index.json").read_text())
    index = meta["cases"]
    w, _ = fgbd.generate_cloud("ramp", 1000)
    fgbd.denoise(fgbd.add_gaussian_noise(w, 10, seed=1))
    case("x8m_ramp_s10", "ramp", 8_000_000, 10.0, colors=None, index=index)
    case("x8m_two-tone_s10", "two-tone", 8_000_000, 10.0, colors=None, index=index)
    (OUT / "index.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
