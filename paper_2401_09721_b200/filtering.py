"""The drop-in: `denoise` plus the filter/selection stage API.

Mirrors reference filtering.py (FilterConfig, FslrMask, DenoiseReport,
filter_step, apply_filter, spectral_response, fslr_mask,
selection_criterion, select_q, denoise) with the same names, defaults,
validation messages and exception classes.  All arithmetic runs in the
B200 library; `denoise` is one C-ABI call (`fgbd_denoise`) that keeps the
frame in HBM from the host->device copy of its inputs to the copy of the
clipped result.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cloud import PointCloud
from .errors import AllPointsExcludedError, FilterError, GraphError
from .graph import Graph, _require_quantized, ensure_device_graph
from .noise import NoiseEstimate, PatchSet, _device_noise, _to_estimate


@dataclass(frozen=True)
class FilterConfig:
    """Knobs for filter selection and the denoise pipeline (filtering.py:33-59).

    epsilon only sets the report's `converged` flag; None means 1e-3 sigma^2.
    """

    q_max: int = 64
    epsilon: float | None = None
    fslr_enabled: bool = True
    patch_size: int = 7
    reestimate_interval: int = 10
    fslr_sigma_floor: float = 0.5
    criterion_mode: str = "pooled"
    early_exit: bool = True
    tau_divisor: str = "count"

    def __post_init__(self):
        if self.q_max < 0:
            raise FilterError(f"q_max must be >= 0, got {self.q_max}")
        if self.reestimate_interval < 1:
            raise FilterError(f"reestimate_interval must be >= 1, got {self.reestimate_interval}")
        if self.patch_size < 2:
            raise FilterError(f"patch_size must be >= 2, got {self.patch_size}")
        if self.criterion_mode not in ("pooled", "per_channel"):
            raise FilterError(f"unknown criterion_mode {self.criterion_mode!r}")


@dataclass(frozen=True)
class FslrMask:
    include: np.ndarray

    def __post_init__(self):
        inc = np.ascontiguousarray(np.asarray(self.include, bool))
        inc.flags.writeable = False
        object.__setattr__(self, "include", inc)

    @property
    def included_count(self) -> int:
        return int(self.include.sum())

    @property
    def n_points(self) -> int:
        return int(self.include.shape[0])

    @classmethod
    def all_points(cls, n: int) -> "FslrMask":
        return cls(np.ones(n, bool))


@dataclass
class DenoiseReport:
    """Outcome summary of one denoise run (filtering.py:86-116).

    `device` carries B200 diagnostics (steps S, sigma_g, edge count, the
    criterion trace, per-channel eigen data, kernel launch count); it is not
    part of `to_dict()`, which stays identical to the reference's.
    """

    selected_q: int
    sigma_est: float
    masked_fraction: float
    stage_timings: dict[str, float] = field(default_factory=dict)
    psnr_db: float | None = None
    criterion_value: float | None = None
    converged: bool | None = None
    cached: bool = False
    eligible_count: int | None = None
    device: dict | None = field(default=None, repr=False, compare=False)

    def to_dict(self) -> dict:
        out = {
            "selected_q": self.selected_q,
            "sigma_est": self.sigma_est,
            "masked_fraction": self.masked_fraction,
            "stage_timings": dict(self.stage_timings),
            "cached": self.cached,
        }
        for key in ("psnr_db", "criterion_value", "converged", "eligible_count"):
            val = getattr(self, key)
            if val is not None:
                out[key] = val
        return out


def _signal(signal, n) -> tuple[np.ndarray, bool]:
    f = np.asarray(signal, np.float64)
    flat = f.ndim == 1
    if flat:
        f = f[:, None]
    if f.shape[0] != n:
        raise FilterError(f"signal has {f.shape[0]} rows for a {n}-vertex graph")
    return f, flat


def apply_filter(g: Graph, signal: np.ndarray, q: int) -> np.ndarray:
    """q random-walk steps (filtering.py:158-165) on the device.

    Uses the graph's fp64 per-slot weights verbatim (weight injection), so
    the result is bit-identical to the reference's scipy evaluation.
    """
    if q < 0:
        raise FilterError(f"q must be >= 0, got {q}")
    if not g.is_weighted:
        raise FilterError("filter_step requires a weighted graph")
    f, flat = _signal(signal, g.n)
    if q == 0:
        out = np.array(f, np.float64)
        return out[:, 0] if flat else out
    cols = f.shape[1]
    # the device kernel filters (N, 3) signals; pad / split other widths
    chunks = []
    for c0 in range(0, cols, 3):
        blk = np.zeros((g.n, 3))
        w = min(3, cols - c0)
        blk[:, :w] = f[:, c0:c0 + w]
        out = np.empty((g.n, 3))
        ctx = nat.context()
        slot_w = np.ascontiguousarray(g.csr_weights())
        ctx.check(ctx.lib.fgbd_filter_steps_csr(ctx.handle, nat.ptr(g.indptr), nat.ptr(g.indices),
                                                nat.ptr(slot_w), g.n, g.indices.size,
                                                nat.ptr(blk), int(q), nat.ptr(out), 0),
                  "filter_step")
        chunks.append(out[:, :w])
    res = np.concatenate(chunks, axis=1)
    return res[:, 0] if flat else res


def filter_step(g: Graph, signal: np.ndarray) -> np.ndarray:
    """out_i = (d_i f_i + sum_j w_ij f_j) / (2 d_i) (filtering.py:132-155)."""
    if not g.is_weighted:
        raise FilterError("filter_step requires a weighted graph")
    return apply_filter(g, signal, 1)


def spectral_response(lam, q: int):
    """(1 - lambda/2)^q -- analysis utility, not on the device path (filtering.py:168-172)."""
    if q < 0:
        raise FilterError(f"q must be >= 0, got {q}")
    return (1.0 - np.asarray(lam, np.float64) / 2.0) ** q


def fslr_mask(patches: PatchSet, sigma_est: float, sigma_floor: float = 0.5) -> FslrMask:
    """Exclude points whose mean patch std exceeds 2 sigma (filtering.py:175-194)."""
    n = patches.n_points
    if sigma_est < sigma_floor:
        return FslrMask.all_points(n)
    _device_noise(patches, "count")  # device FSLR statistic for this patch set
    ctx = nat.context()
    inc = np.empty(n, np.uint8)
    allx = nat.c_i32()
    rc = ctx.lib.fgbd_fslr_mask(ctx.handle, float(sigma_est), float(sigma_floor),
                                nat.ptr(inc), allx)
    if allx.value:
        raise AllPointsExcludedError(
            "the variance threshold excluded every point; fall back to "
            "unmasked selection (disable the mask or raise sigma_floor)")
    ctx.check(rc, "fslr_mask")
    return FslrMask(inc.astype(bool))


def selection_criterion(y: np.ndarray, x_q: np.ndarray, mask: FslrMask, sigma_est: float,
                        mode: str = "pooled") -> float:
    """Eq. (6): |sigma^2 - per-entry power removed| over included points."""
    y = np.asarray(y, np.float64)
    x = np.asarray(x_q, np.float64)
    if y.ndim == 1:
        y, x = y[:, None], x[:, None]
    if y.shape != x.shape:
        raise FilterError(f"signal shapes differ: {y.shape} vs {x.shape}")
    if mode not in ("pooled", "per_channel"):
        raise FilterError(f"unknown criterion mode {mode!r}")
    if mask.included_count < 1:
        raise FilterError("criterion needs at least one included point")
    if y.shape[1] != 3:
        raise NotImplementedError("the device criterion is defined for (N, 3) colour signals")
    ctx = nat.context()
    y = np.ascontiguousarray(y)
    x = np.ascontiguousarray(x)
    inc = np.ascontiguousarray(mask.include, np.uint8)
    out = nat.c_f64()
    ctx.check(ctx.lib.fgbd_selection_criterion(ctx.handle, nat.ptr(y), nat.ptr(x), nat.ptr(inc),
                                               y.shape[0], float(sigma_est),
                                               0 if mode == "pooled" else 1, out, 0),
              "selection_criterion")
    return float(out.value)


def select_q(pc_noisy: PointCloud, g: Graph, sigma_est: float, cfg: FilterConfig,
             mask: FslrMask | None = None) -> tuple[int, np.ndarray]:
    """Device-resident q scan (filtering.py:225-256)."""
    if sigma_est < 0:
        raise FilterError(f"sigma_est must be >= 0, got {sigma_est}")
    ctx = ensure_device_graph(pc_noisy, g)
    n = pc_noisy.n_points
    inc = None if mask is None else np.ascontiguousarray(mask.include, np.uint8)
    q = nat.c_i32()
    x = np.empty((n, 3))
    rep = nat.Report()
    ctx.check(ctx.lib.fgbd_select_q(ctx.handle, nat.ptr(pc_noisy.colors), nat.ptr(inc),
                                    float(sigma_est), nat.make_config(cfg), q, nat.ptr(x),
                                    rep, 0), "select_q")
    return int(q.value), x


def _device_info(r: nat.Report, patch: int) -> dict:
    nt = int(r.n_trace)
    return {
        "steps": int(r.steps),
        "sigma_g": float(r.sigma_g),
        "n_edges": int(r.n_edges),
        "max_degree": int(r.max_degree),
        "included_count": int(r.included_count),
        "all_excluded_fallback": bool(r.all_excluded_fallback),
        "per_channel_sigma": list(r.per_channel_sigma),
        "eigenvalues": [[r.eigenvalues[c][k] for k in range(patch)] for c in range(3)],
        "m": list(r.tail_m),
        "tau": list(r.tail_tau),
        "fallback": [bool(v) for v in r.tail_fallback],
        "trace": [r.trace[k] for k in range(nt)],
        "gpu_launches": int(r.gpu_launches),
        "t_total": float(r.t_total),
        "t_lf_steps": float(r.t_lf_steps),
        "t_h2d": float(r.t_h2d),
        "t_d2h": float(r.t_d2h),
        "graph_reused": bool(r.graph_reused),
        # True per channel where the reference would have raised "Jacobi did
        # not converge" (noise.py:180-185) and this build returned the
        # eigenvalues instead
        "jacobi_direct_off": [bool(v) for v in r.jacobi_direct_off],
    }


def denoise(pc_noisy: PointCloud, cfg: FilterConfig = FilterConfig(),
            cached_q: int | None = None,
            cached_sigma_est: float | None = None) -> tuple[PointCloud, DenoiseReport]:
    """SLG -> NE-GBP -> FSLR + q selection -> low-pass filter, on one B200.

    Same contract as the reference (filtering.py:259-328): N < 2 returns the
    input unchanged; `cached_q` skips estimation and selection; geometry is
    never modified; an all-excluded FSLR mask warns and selects unmasked.
    """
    return denoise_frame(pc_noisy, cfg, cached_q, cached_sigma_est)


def denoise_frame(pc_noisy: PointCloud, cfg: FilterConfig = FilterConfig(),
                  cached_q: int | None = None, cached_sigma_est: float | None = None,
                  reuse_graph: bool = False, static_geometry: bool = False,
                  device_ne: bool = False) -> tuple[PointCloud, DenoiseReport]:
    """`denoise` for one frame of a sequence.  With `reuse_graph`, a frame
    whose coordinates are byte-identical to the previous frame handled by
    this thread's device context reuses that scan-line graph instead of
    rebuilding it (verified on the device; results are identical).  With
    `static_geometry` the caller GUARANTEES the coordinates equal those of
    the graph this thread's context holds: they are not uploaded or compared
    (FGBD_FLAG_STATIC_GEOMETRY); without a held graph it acts as reuse_graph.
    `device_ne` finishes NE-GBP on the device (FGBD_FLAG_DEVICE_NE, same bits):
    no host round trip, so concurrent frames overlap better."""
    n = pc_noisy.n_points
    if n < 2:
        return pc_noisy, DenoiseReport(
            selected_q=0, sigma_est=0.0, masked_fraction=0.0,
            stage_timings={"graph_construction": 0.0, "noise_estimation": 0.0,
                           "low_pass_filter": 0.0})
    bits = _require_quantized(pc_noisy)
    cfg = _check_call(cfg, cached_q)
    ctx = nat.context()
    out = nat.pinned_output((n, 3), np.float64)  # full-rate D2H, recycled
    rep = nat.Report()
    cq = -1 if cached_q is None else int(cached_q)
    cs = float("nan") if cached_sigma_est is None else float(cached_sigma_est)
    ctx.graph_token = None  # the call rebuilds the device graph, even when it fails
    ctx.check(ctx.lib.fgbd_denoise(ctx.handle, nat.ptr(pc_noisy.coords), nat.ptr(pc_noisy.colors),
                                   n, bits, nat.make_config(cfg), cq, cs, nat.ptr(out), rep,
                                   (nat.FLAG_REUSE_GRAPH if reuse_graph else 0)
                                   | (nat.FLAG_STATIC_GEOMETRY if static_geometry else 0)
                                   | (nat.FLAG_DEVICE_NE if device_ne else 0)),
              "denoise")
    report = _report_from(rep, cfg, cached_q, cached_sigma_est)
    out.flags.writeable = False
    return PointCloud._trusted(pc_noisy.coords, out, pc_noisy.bit_depth), report


def _check_call(cfg: FilterConfig, cached_q) -> FilterConfig:
    """Argument errors denoise raises (filtering.py:315, noise.py:205); an
    unknown divisor rule only matters when noise is estimated."""
    if cached_q is not None and cached_q < 0:
        raise FilterError(f"cached_q must be >= 0, got {cached_q}")
    if cfg.tau_divisor not in ("count", "count_plus_one"):
        from .errors import NoiseEstimationError
        if cached_q is None:
            raise NoiseEstimationError(f"unknown divisor rule {cfg.tau_divisor!r}")
        cfg = FilterConfig(**{**cfg.__dict__, "tau_divisor": "count"})
    return cfg


def _report_from(rep, cfg: FilterConfig, cached_q, cached_sigma_est) -> DenoiseReport:
    """DenoiseReport of one device frame (filtering.py:300-328 field rules)."""
    timings = {"graph_construction": float(rep.t_graph_construction),
               "noise_estimation": float(rep.t_noise_estimation),
               "low_pass_filter": float(rep.t_low_pass_filter)}
    info = _device_info(rep, cfg.patch_size)
    if cached_q is None:
        if rep.all_excluded_fallback:
            warnings.warn("variance mask excluded every point; selecting unmasked")
        return DenoiseReport(
            selected_q=int(rep.selected_q), sigma_est=float(rep.sigma_est),
            masked_fraction=float(rep.masked_fraction), stage_timings=timings,
            criterion_value=float(rep.criterion_value), converged=bool(rep.converged),
            eligible_count=int(rep.eligible_count), device=info)
    return DenoiseReport(
        selected_q=int(cached_q),
        sigma_est=float(cached_sigma_est) if cached_sigma_est is not None else 0.0,
        masked_fraction=0.0, stage_timings=timings, cached=True, device=info)
