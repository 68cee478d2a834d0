"""Spatial slab partition of one frame over P GPUs.

The frame is cut into P z-slabs of about N/P points each (whole z planes;
the scan-line-1 code is z-major, so a slab is a contiguous range of the
global line-1 order).  Rank r uploads, sorts, estimates and filters ONLY its
own points; cross-slab work goes over peer memory (csrc/slab.cu):

* scan-line graph: per-line block lists (first/last point of each run that
  shares the line's key above z) are published; each rank derives its exact
  cross-slab neighbours -- wraparounds included -- from its peers' lists;
* sigma_g: exact fixed-point shares, all-gathered (the single-GPU bits);
* NE-GBP moments and the FSLR sums: all-gathered and summed in rank order, so
  every rank runs the same host Jacobi and selects the same q;
* the q scan: halo signals are P2P loads from the owner's buffers, the
  criterion is all-reduced through peer slots + flags every step.

`denoise_slab(pc, cfg, process_group=pg)` is a collective: every rank of the
process group (one process per GPU) passes the same frame; with
output="full" every rank gets the whole denoised frame, with output="local"
it gets (global indices, colours) of its own points only -- the partitioned
path, which uploads and downloads 1/P of the frame.

`denoise_slab(pc, cfg, emulate_ranks=P)` runs the P ranks' protocol on this
process's GPU (the test harness).  Either way q, S and the colours equal
`denoise(pc)` bit for bit (csrc/graph.cu fx52: sigma_g is partition-exact).
"""

from __future__ import annotations

import ctypes as C
import threading
import warnings
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .cloud import PointCloud
from .errors import FilterError, NoiseEstimationError
from .filtering import DenoiseReport, FilterConfig, _device_info
from .graph import _require_quantized

MAX_RANKS = 16
MAX_SLAB_BITS = 15
_cache = threading.local()
_part_cache: dict = {}
_part_lock = threading.Lock()


@dataclass(frozen=True)
class SlabPartition:
    """z-slab split of one frame: rank r owns the points with
    zcut[r] <= z < zcut[r+1], i.e. the global line-1 rows
    [starts[r], starts[r+1]).  `order` lists the points rank by rank in
    increasing index (None when the input is already z-sorted, so every
    rank's points are the contiguous index range [starts[r], starts[r+1]))."""

    world: int
    zcut: np.ndarray
    counts: np.ndarray
    starts: np.ndarray
    order: np.ndarray | None

    def own_index(self, rank: int) -> np.ndarray:
        a, b = int(self.starts[rank]), int(self.starts[rank + 1])
        return np.arange(a, b, dtype=np.int64) if self.order is None else self.order[a:b]


def slab_partition(pc: PointCloud, world: int) -> SlabPartition:
    """Equal-count z-slabs (whole z planes) of a quantized cloud.

    Every rank computes the same partition from the same frame.  Cached per
    coordinate array, so a static-geometry sequence pays for it once.
    """
    world = int(world)
    if not 1 <= world <= MAX_RANKS:
        raise ValueError(f"slab ranks must be in [1, {MAX_RANKS}], got {world}")
    key = (id(pc.coords), world)
    with _part_lock:
        hit = _part_cache.get(key)
        if hit is not None and hit[0]() is pc.coords:
            return hit[1]
    b = _require_quantized(pc)
    n = pc.n_points
    z = np.asarray(pc.coords)[:, 2]
    hist = np.bincount(z, minlength=1 << b)
    cum = np.cumsum(hist)
    zcut = np.zeros(world + 1, np.int64)
    zcut[world] = 1 << b
    for r in range(1, world):
        target = (n * r) // world
        zcut[r] = max(int(np.searchsorted(cum, target, side="left")) + 1, int(zcut[r - 1]) + 1)
    zcut = np.minimum(zcut, 1 << b)
    below = np.concatenate([[0], cum])  # points with z < zc
    starts = below[zcut]
    counts = np.diff(starts)
    if np.any(counts < 1):
        raise FilterError(f"cannot cut this frame into {world} non-empty z-slabs")
    order = None
    if n > 1 and not bool(np.all(z[1:] >= z[:-1])):
        slab_id = np.searchsorted(zcut, z, side="right") - 1
        order = np.argsort(slab_id, kind="stable").astype(np.int64)
    part = SlabPartition(world, zcut, counts.astype(np.int64), starts.astype(np.int64), order)
    with _part_lock:
        if len(_part_cache) > 64:
            _part_cache.clear()
        _part_cache[key] = (weakref.ref(pc.coords), part)
    return part


def exchange_handles(handle: bytes, process_group) -> list[bytes]:
    """All-gather every rank's IPC handle (control plane, once per shape)."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(process_group)
    dist.all_gather_object(out, handle, group=process_group)
    return out


class _Slab:
    def __init__(self, ctx, world, rank, n_total, max_own, flags, process_group=None):
        self.ctx = ctx
        self.h = ctx.lib.fgbd_slab_create(ctx.handle, world, rank, n_total, max_own, flags)
        if not self.h:
            ctx.check(nat.E_ARG, "slab create")
        if not flags & nat.SLAB_EMULATED:
            size = ctx.lib.fgbd_slab_handle_size()
            mine = (C.c_uint8 * size)()
            ctx.check(ctx.lib.fgbd_slab_export(ctx.handle, self.h, mine), "slab export")
            allh = exchange_handles(bytes(mine), process_group)
            flat = (C.c_uint8 * (size * world)).from_buffer_copy(b"".join(allh))
            ctx.check(ctx.lib.fgbd_slab_import(ctx.handle, self.h, flat), "slab import")

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.fgbd_slab_destroy(self.ctx.handle, self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _slab_for(ctx, world, rank, n_total, max_own, flags, pg):
    key = (id(ctx), world, rank, n_total, flags)
    slabs = getattr(_cache, "slabs", None)
    if slabs is None:
        slabs = _cache.slabs = {}
    s = slabs.get(key)
    if s is not None and s[1] < max_own:
        slabs.pop(key)[0].close()
        s = None
    if s is None:
        for k in [k for k in slabs if k[0] == id(ctx)]:
            slabs.pop(k)[0].close()
        s = slabs[key] = (_Slab(ctx, world, rank, n_total, max_own, flags, pg), max_own)
    return s[0]


def denoise_slab(pc_noisy: PointCloud, cfg: FilterConfig = FilterConfig(),
                 cached_q: int | None = None, cached_sigma_est: float | None = None, *,
                 process_group=None, emulate_ranks: int | None = None,
                 output: str = "full", partition: SlabPartition | None = None,
                 emulate_exchange: bool = False):
    """`denoise` with the frame split into z-slabs over P ranks.

    Returns (PointCloud, DenoiseReport) like `denoise`; with output="local"
    (multi-GPU only) returns (own global indices, own colours, report).
    `emulate_exchange` runs the filter's per-step cross-rank exchange of the
    P-GPU protocol in the emulation too (testing).
    """
    n = pc_noisy.n_points
    if n < 2:
        from .filtering import denoise

        return denoise(pc_noisy, cfg, cached_q, cached_sigma_est)
    bits = _require_quantized(pc_noisy)
    if bits > MAX_SLAB_BITS:
        raise ValueError(f"slab partition supports bit depths up to {MAX_SLAB_BITS}, got {bits}")
    if cached_q is not None and cached_q < 0:
        raise FilterError(f"cached_q must be >= 0, got {cached_q}")
    if cfg.tau_divisor not in ("count", "count_plus_one") and cached_q is None:
        raise NoiseEstimationError(f"unknown divisor rule {cfg.tau_divisor!r}")
    if output not in ("full", "local"):
        raise ValueError(f"output must be 'full' or 'local', got {output!r}")
    if emulate_ranks is not None:
        world, rank, emulated = int(emulate_ranks), 0, True
    else:
        import torch.distributed as dist

        world, rank, emulated = dist.get_world_size(process_group), \
            dist.get_rank(process_group), False
    if not 1 <= world <= MAX_RANKS:
        raise ValueError(f"slab ranks must be in [1, {MAX_RANKS}], got {world}")
    part = partition if partition is not None else slab_partition(pc_noisy, world)
    if part.world != world:
        raise ValueError(f"partition is for {part.world} ranks, not {world}")
    ctx = nat.context()
    flags = nat.SLAB_EMULATED if emulated else (nat.SLAB_FULL_OUTPUT if output == "full" else 0)
    if emulated and emulate_exchange:
        flags |= nat.SLAB_EXCHANGE
    max_own = int(part.counts.max())
    slab = _slab_for(ctx, world, rank, n, max_own, flags, process_group)
    coords, colors = pc_noisy.coords, pc_noisy.colors
    counts = np.ascontiguousarray(part.counts, np.int64)
    if emulated:
        lo, hi = 0, n
    else:
        lo, hi = int(part.starts[rank]), int(part.starts[rank + 1])
    if part.order is None:
        own_c, own_y, gidx, base = coords[lo:hi], colors[lo:hi], None, lo
    else:
        sel = part.order[lo:hi]
        own_c = np.ascontiguousarray(coords[sel])
        own_y = np.ascontiguousarray(colors[sel])
        gidx, base = sel.astype(np.uint32), 0
    full_out = emulated or output == "full"
    rows = n if full_out and not emulated else hi - lo
    out = nat.pinned_output((rows, 3), np.float64)
    rep = nat.Report()
    cq = -1 if cached_q is None else int(cached_q)
    cs = float("nan") if cached_sigma_est is None else float(cached_sigma_est)
    ctx.graph_token = None  # the slab ranks reuse this context's graph scratch
    ctx.check(ctx.lib.fgbd_denoise_slab(
        ctx.handle, slab.h, nat.ptr(np.ascontiguousarray(own_c)),
        nat.ptr(np.ascontiguousarray(own_y)), None if gidx is None else nat.ptr(gidx), base,
        nat.ptr(counts), bits, nat.make_config(cfg), cq, cs, nat.ptr(out), rep, 0),
        "denoise_slab")
    report = _report(rep, cfg, cached_q, cached_sigma_est, world)
    if not full_out:
        idx = np.arange(lo, hi, dtype=np.int64) if part.order is None else part.order[lo:hi]
        colors_out = np.array(out)
        return idx, colors_out, report
    if emulated and part.order is not None:
        full = np.empty((n, 3), np.float64)
        full[part.order] = out
        out = full
    out.flags.writeable = False
    return PointCloud._trusted(pc_noisy.coords, out, pc_noisy.bit_depth), report


def _report(rep, cfg, cached_q, cached_sigma_est, world) -> DenoiseReport:
    timings = {"graph_construction": float(rep.t_graph_construction),
               "noise_estimation": float(rep.t_noise_estimation),
               "low_pass_filter": float(rep.t_low_pass_filter)}
    info = _device_info(rep, cfg.patch_size)
    info["slab_ranks"] = world
    # per rank run here: device seconds of [upload + own sort + block lists,
    # cross-slab neighbours + rows, NE-GBP + FSLR, output + download]
    info["slab_rank_seconds"] = [[float(rep.t_slab_rank[r][k]) for k in range(4)]
                                 for r in range(world)]
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
