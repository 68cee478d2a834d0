"""NE-GBP stage API (reference noise.py), backed by the B200 library.

The device computes patch moments and the FSLR statistic in one pass; the
7x7 covariance eigenproblem and the tail rule run in host C++ inside the
same library (fgbd_symmetric_eigenvalues / fgbd_select_tail).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

import ctypes as C
import numpy as np

from . import _native as nat
from .cloud import PointCloud
from .errors import NoiseEstimationError
from .graph import Graph, ensure_device_graph

CHANNEL_NAMES = ("R", "G", "B")
JACOBI_MAX_SWEEPS = 50
SYMMETRY_RTOL = 1e-9
OFFDIAG_RTOL = 1e-12


def _channel_index(c) -> int:
    if isinstance(c, str):
        if c.upper() not in CHANNEL_NAMES:
            raise NoiseEstimationError(f"unknown channel {c!r}")
        return CHANNEL_NAMES.index(c.upper())
    c = int(c)
    if not 0 <= c <= 2:
        raise NoiseEstimationError(f"channel index must be 0..2, got {c}")
    return c


@dataclass(frozen=True, eq=False)
class PatchSet:
    """Distance-sorted patches of one cloud on one graph (noise.py:30-48).

    The device never materialises patches on the denoise path; `vectors`
    and `point_index` are pulled from the device on first access.
    """

    pc: PointCloud
    graph: Graph | None
    patch_size: int
    n_points: int
    _cache: dict = field(default_factory=dict, repr=False)

    def _pull(self):
        if "vectors" not in self._cache:
            ctx = ensure_device_graph(self.pc, self.graph)
            ne = nat.c_i64()
            ctx.check(ctx.lib.fgbd_extract_patches(ctx.handle, nat.ptr(self.pc.colors),
                                                   self.patch_size, None, None, ne, 0),
                      "extract_patches")
            idx = np.empty(ne.value, np.int64)
            vec = np.empty((3, ne.value, self.patch_size), np.float64)
            ctx.check(ctx.lib.fgbd_extract_patches(ctx.handle, nat.ptr(self.pc.colors),
                                                   self.patch_size, nat.ptr(idx), nat.ptr(vec),
                                                   ne, 0), "extract_patches")
            idx.flags.writeable = False
            vec.flags.writeable = False
            self._cache["vectors"], self._cache["point_index"] = vec, idx
        return self._cache["vectors"], self._cache["point_index"]

    @property
    def vectors(self) -> np.ndarray:
        return self._pull()[0]

    @property
    def point_index(self) -> np.ndarray:
        return self._pull()[1]

    @property
    def eligible_count(self) -> int:
        if "ne" not in self._cache:
            if self.graph is not None:
                self._cache["ne"] = int((self.graph.degrees() >= self.patch_size - 1).sum())
            else:
                self._cache["ne"] = int(self.point_index.shape[0])
        return self._cache["ne"]

    def channel(self, c) -> np.ndarray:
        return self.vectors[_channel_index(c)]


@dataclass(frozen=True)
class NoiseEstimate:
    sigma_est: float
    per_channel_sigma: np.ndarray
    eigenvalues: np.ndarray
    m: np.ndarray
    tau: np.ndarray
    fallback: np.ndarray
    eligible_count: int
    # per channel: the reference would have raised "Jacobi did not converge"
    # here (noise.py:180-185); see DESIGN.md section 1.  Not a reference field.
    jacobi_direct_off: tuple = field(default=(False, False, False), compare=False, repr=False)


class TailSelection(NamedTuple):
    m: int
    tau: float
    fallback: bool


def extract_patches(pc: PointCloud, g: Graph, patch_size: int) -> PatchSet:
    """Validate like noise.py:89-97 and bind the patch set to (pc, g)."""
    d = int(patch_size)
    if d < 2:
        raise NoiseEstimationError(f"patch_size must be >= 2, got {patch_size}")
    max_deg = int(g.degrees().max(initial=0))
    if d > 1 + max_deg:
        raise NoiseEstimationError(
            f"patch_size {d} exceeds 1 + max degree ({1 + max_deg}) of this graph")
    return PatchSet(pc, g, d, pc.n_points)


def _device_noise(patches: PatchSet, divisor: str, want_stat: bool = False):
    ctx = ensure_device_graph(patches.pc, patches.graph)
    out = nat.Noise()
    div = {"count": 0, "count_plus_one": 1}.get(divisor)
    if div is None:
        raise NoiseEstimationError(f"unknown divisor rule {divisor!r}")
    stat = np.empty(patches.n_points, np.float64) if want_stat else None
    ctx.check(ctx.lib.fgbd_estimate_noise(ctx.handle, nat.ptr(patches.pc.colors),
                                          patches.patch_size, div, out, nat.ptr(stat), 0),
              "estimate_noise")
    return out, stat


def patch_covariance(patches: PatchSet, channel) -> np.ndarray:
    """Population covariance of one channel's patches (noise.py:122-130)."""
    c = _channel_index(channel)
    if patches.eligible_count < 2:
        raise NoiseEstimationError(f"need at least 2 patches, have {patches.eligible_count}")
    out, _ = _device_noise(patches, "count")
    d = patches.patch_size
    return np.array([[out.covariance[c][i][j] for j in range(d)] for i in range(d)])


def symmetric_eigenvalues(s: np.ndarray, max_sweeps: int = JACOBI_MAX_SWEEPS) -> np.ndarray:
    """Cyclic Jacobi eigenvalues, descending (noise.py:133-185), host C++."""
    s = np.ascontiguousarray(np.asarray(s, np.float64))
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise NoiseEstimationError(f"matrix must be square, got {s.shape}")
    if max_sweeps != JACOBI_MAX_SWEEPS:
        raise NotImplementedError("the device library fixes max_sweeps at 50")
    lib = nat.load_library()
    out = np.empty(s.shape[0])
    err = C.create_string_buffer(256)
    rc = lib.fgbd_symmetric_eigenvalues(nat.ptr(s), s.shape[0], nat.ptr(out), err, 256)
    if rc:
        raise NoiseEstimationError(err.value.decode())
    return out


def select_tail(eigenvalues: np.ndarray, divisor: str = "count") -> TailSelection:
    """Smallest m with mean(tail) > median(tail), else m = D // 2 (noise.py:188-216)."""
    lam = np.ascontiguousarray(np.asarray(eigenvalues, np.float64))
    div = {"count": 0, "count_plus_one": 1}.get(divisor)
    if lam.size >= 3 and div is None:
        raise NoiseEstimationError(f"unknown divisor rule {divisor!r}")
    lib = nat.load_library()
    m, fb, tau = nat.c_i32(), nat.c_i32(), nat.c_f64()
    err = C.create_string_buffer(256)
    rc = lib.fgbd_select_tail(nat.ptr(lam), lam.size, div if div is not None else 0, m, tau, fb,
                              err, 256)
    if rc:
        raise NoiseEstimationError(err.value.decode())
    return TailSelection(int(m.value), float(tau.value), bool(fb.value))


def _to_estimate(out: nat.Noise) -> NoiseEstimate:
    d = out.patch_size
    return NoiseEstimate(
        sigma_est=float(out.sigma_est),
        per_channel_sigma=np.array(out.per_channel_sigma[:]),
        eigenvalues=np.array([[out.eigenvalues[c][k] for k in range(d)] for c in range(3)]),
        m=np.array(out.m[:], np.int64),
        tau=np.array(out.tau[:]),
        fallback=np.array([bool(x) for x in out.fallback]),
        eligible_count=int(out.eligible_count),
        jacobi_direct_off=tuple(bool(x) for x in out.jacobi_direct_off),
    )


def estimate_noise_from_patches(patches: PatchSet, divisor: str = "count") -> NoiseEstimate:
    """Covariance -> eigenvalues -> tail -> sigma per channel, pooled (noise.py:219-243)."""
    out, _ = _device_noise(patches, divisor)
    return _to_estimate(out)


def estimate_noise(pc: PointCloud, g: Graph, patch_size: int = 7,
                   divisor: str = "count") -> NoiseEstimate:
    return estimate_noise_from_patches(extract_patches(pc, g, patch_size), divisor)
