"""Spatial slab partition of one frame over P GPUs.

`denoise_slab(pc, cfg, process_group=pg)` is a collective: every rank of the
process group (one process per GPU) passes the same frame and gets the full
denoised frame back.  Every rank builds the whole scan-line graph and runs
NE-GBP (pure functions of the frame: identical on all ranks); the q scan is
split into row slabs [n*r/P, n*(r+1)/P), and the fused filter kernel reads
foreign neighbours straight from the owner GPU's memory (CUDA IPC + NVLink
peer access) and all-reduces the criterion through peer-memory slots and
flags (csrc/slab.cu).  The only host-side collective is the one-time
exchange of IPC handles.

`denoise_slab(pc, cfg, emulate_ranks=P)` runs the same protocol with the P
ranks as block groups of one cooperative launch on this process's GPU; its
result is bit-identical to the P-GPU run and to the single-GPU `denoise`
colours (the partition only regroups the criterion sums).
"""

from __future__ import annotations

import ctypes as C
import threading
import warnings

import numpy as np

from . import _native as nat
from .cloud import PointCloud
from .errors import FilterError, NoiseEstimationError
from .filtering import DenoiseReport, FilterConfig, _device_info
from .graph import _require_quantized

MAX_RANKS = 16
_cache = threading.local()


def slab_bounds(n: int, world: int) -> list[int]:
    """Row ranges of the ranks: rank r owns [b[r], b[r+1]) (csrc/slab.cu slab_lo)."""
    return [(n * r) // world for r in range(world + 1)]


def exchange_handles(handle: bytes, process_group) -> list[bytes]:
    """All-gather every rank's IPC handle (control plane, once per shape)."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(process_group)
    dist.all_gather_object(out, handle, group=process_group)
    return out


class _Slab:
    def __init__(self, ctx, world, rank, n, emulated, process_group=None):
        self.ctx = ctx
        self.h = ctx.lib.fgbd_slab_create(ctx.handle, world, rank, n, 1 if emulated else 0)
        if not self.h:
            ctx.check(nat.E_ARG, "slab create")
        if not emulated:
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


def _slab_for(ctx, world, rank, n, emulated, pg):
    key = (id(ctx), world, rank, n, emulated)
    slabs = getattr(_cache, "slabs", None)
    if slabs is None:
        slabs = _cache.slabs = {}
    s = slabs.get(key)
    if s is None:
        for k in [k for k in slabs if k[0] == id(ctx)]:
            slabs.pop(k).close()
        s = slabs[key] = _Slab(ctx, world, rank, n, emulated, pg)
    return s


def denoise_slab(pc_noisy: PointCloud, cfg: FilterConfig = FilterConfig(),
                 cached_q: int | None = None, cached_sigma_est: float | None = None, *,
                 process_group=None, emulate_ranks: int | None = None
                 ) -> tuple[PointCloud, DenoiseReport]:
    """`denoise` with the filter loop split into spatial slabs over P ranks."""
    n = pc_noisy.n_points
    if n < 2:
        from .filtering import denoise

        return denoise(pc_noisy, cfg, cached_q, cached_sigma_est)
    bits = _require_quantized(pc_noisy)
    if cached_q is not None and cached_q < 0:
        raise FilterError(f"cached_q must be >= 0, got {cached_q}")
    if cfg.tau_divisor not in ("count", "count_plus_one"):
        raise NoiseEstimationError(f"unknown divisor rule {cfg.tau_divisor!r}")
    if emulate_ranks is not None:
        world, rank, emulated = int(emulate_ranks), 0, True
    else:
        import torch.distributed as dist

        world, rank, emulated = dist.get_world_size(process_group), \
            dist.get_rank(process_group), False
    if not 1 <= world <= MAX_RANKS:
        raise ValueError(f"slab ranks must be in [1, {MAX_RANKS}], got {world}")
    ctx = nat.context()
    slab = _slab_for(ctx, world, rank, n, emulated, process_group)
    out = nat.pinned_output((n, 3), np.float64)
    rep = nat.Report()
    cq = -1 if cached_q is None else int(cached_q)
    cs = float("nan") if cached_sigma_est is None else float(cached_sigma_est)
    ctx.check(ctx.lib.fgbd_denoise_slab(ctx.handle, slab.h, nat.ptr(pc_noisy.coords),
                                        nat.ptr(pc_noisy.colors), n, bits, nat.make_config(cfg),
                                        cq, cs, nat.ptr(out), rep, 0), "denoise_slab")
    ctx.graph_token = None
    timings = {"graph_construction": float(rep.t_graph_construction),
               "noise_estimation": float(rep.t_noise_estimation),
               "low_pass_filter": float(rep.t_low_pass_filter)}
    info = _device_info(rep, cfg.patch_size)
    info["slab_ranks"] = world
    if cached_q is None:
        if rep.all_excluded_fallback:
            warnings.warn("variance mask excluded every point; selecting unmasked")
        report = DenoiseReport(
            selected_q=int(rep.selected_q), sigma_est=float(rep.sigma_est),
            masked_fraction=float(rep.masked_fraction), stage_timings=timings,
            criterion_value=float(rep.criterion_value), converged=bool(rep.converged),
            eligible_count=int(rep.eligible_count), device=info)
    else:
        report = DenoiseReport(
            selected_q=int(cached_q),
            sigma_est=float(cached_sigma_est) if cached_sigma_est is not None else 0.0,
            masked_fraction=0.0, stage_timings=timings, cached=True, device=info)
    out.flags.writeable = False
    return PointCloud._trusted(pc_noisy.coords, out, pc_noisy.bit_depth), report
