"""Scan-line graph stage API (reference graph.py), backed by the B200 library.

`denoise` never goes through these functions -- it keeps the graph in HBM
as an ELL structure.  They exist so callers of the reference's stage API
(`build_slg`, `compute_sigma_g`, ...) can switch too; each one runs its
arithmetic on the device through the C ABI and returns arrays in the
reference's `Graph` conventions (graph.py:40-107).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .cloud import MAX_BIT_DEPTH, PointCloud
from .errors import GraphError

_LINE_AXES = {1: (2, 1, 0), 2: (0, 2, 1), 3: (1, 0, 2)}  # graph.py:25
_tokens = itertools.count(1)


def _ro(a, dtype):
    a = np.ascontiguousarray(np.asarray(a, dtype))
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class ScanLineCodes:
    """One 3b-bit raster-scan code per point for a single scan line."""

    codes: np.ndarray
    line: int
    bit_depth: int

    def __post_init__(self):
        object.__setattr__(self, "codes", _ro(self.codes, np.uint64))


@dataclass(frozen=True, eq=False)
class Graph:
    """CSR adjacency + unique edge list in the reference's conventions.

    `_token` ties a graph built here to the device copy a context holds, so
    follow-up stage calls on the same graph do not rebuild it.
    """

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    csr_edge: np.ndarray
    edge_u: np.ndarray
    edge_v: np.ndarray
    edge_sqdist: np.ndarray
    sigma_g: float | None = None
    edge_weights: np.ndarray | None = None
    _token: int = 0
    _bits: int = 0
    _slg: bool = False  # built here as the scan-line graph of its cloud

    def __post_init__(self):
        for name in ("indptr", "indices", "csr_edge", "edge_u", "edge_v"):
            object.__setattr__(self, name, _ro(getattr(self, name), np.int64))
        object.__setattr__(self, "edge_sqdist", _ro(self.edge_sqdist, np.float64))
        if self.edge_weights is not None:
            object.__setattr__(self, "edge_weights", _ro(self.edge_weights, np.float64))

    @property
    def n_edges(self) -> int:
        return int(self.edge_u.shape[0])

    @property
    def is_weighted(self) -> bool:
        return self.edge_weights is not None

    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def weighted_degrees(self) -> np.ndarray:
        """(sum over j > i) + (sum over j < i) of incident weights (graph.py:78-85)."""
        if self.edge_weights is None:
            raise GraphError("graph has no weights; run apply_gaussian_weights first")
        w = self.edge_weights
        return (np.bincount(self.edge_u, weights=w, minlength=self.n)
                + np.bincount(self.edge_v, weights=w, minlength=self.n))

    def csr_weights(self) -> np.ndarray:
        if self.edge_weights is None:
            raise GraphError("graph has no weights; run apply_gaussian_weights first")
        return self.edge_weights[self.csr_edge]

    def neighbors(self, i: int) -> np.ndarray:
        return self.indices[self.indptr[i]:self.indptr[i + 1]]

    def edge_set(self) -> set[tuple[int, int]]:
        return set(zip(self.edge_u.tolist(), self.edge_v.tolist()))

    def edge_list_text(self) -> str:
        """One "i j w" line per unique edge, ascending (i, j)."""
        w = self.edge_weights if self.edge_weights is not None else np.ones(self.n_edges)
        rows = [f"{u} {v} {repr(float(x))}"
                for u, v, x in zip(self.edge_u.tolist(), self.edge_v.tolist(), w.tolist())]
        return "\n".join(rows) + ("\n" if rows else "")


def _require_quantized(pc: PointCloud) -> int:
    if not pc.is_quantized:
        raise GraphError("graph construction requires integer voxel coordinates; "
                         "run quantize_coordinates first")
    b = int(pc.bit_depth)
    if b > MAX_BIT_DEPTH:
        raise GraphError(f"bit depth {b} exceeds {MAX_BIT_DEPTH} (64-bit code overflow)")
    return b


def scanline_codes(pc: PointCloud, line: int) -> ScanLineCodes:
    """Eqs. (1)-(3) evaluated on the device (graph.py:122-136)."""
    b = _require_quantized(pc)
    if line not in _LINE_AXES:
        raise GraphError(f"line must be 1, 2 or 3, got {line}")
    ctx = nat.context()
    n = pc.n_points
    codes = np.empty(n, np.uint64)
    ctx.graph_token = None  # the sort scratch is shared with the held SLG
    ctx.check(ctx.lib.fgbd_scan_line(ctx.handle, nat.ptr(pc.coords), n, b, line,
                                     nat.ptr(codes), None, 0), "scanline_codes")
    return ScanLineCodes(codes, line, b)


def radix_argsort(keys: np.ndarray, key_bits: int = 64) -> np.ndarray:
    """Stable LSD radix argsort on the device (graph.py:154-171)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    if not 1 <= key_bits <= 64:
        raise ValueError(f"key_bits must be in [1, {64}], got {key_bits}")
    n = keys.size
    if n < 2:
        return np.arange(n, dtype=np.int64)
    ctx = nat.context()
    perm = np.empty(n, np.int64)
    ctx.graph_token = None  # the sort scratch is shared with the held SLG
    ctx.check(ctx.lib.fgbd_radix_argsort(ctx.handle, nat.ptr(keys), n, int(key_bits),
                                         nat.ptr(perm), 0), "radix_argsort")
    return perm


def sort_permutation(codes: ScanLineCodes) -> np.ndarray:
    """Stable rank order under one scan-line code (graph.py:174-176)."""
    return radix_argsort(codes.codes, key_bits=3 * codes.bit_depth)


def _device_build(pc: PointCloud, weights64: bool = False) -> tuple[nat.Context, object]:
    b = _require_quantized(pc)
    ctx = nat.context()
    ctx.graph_token = None
    info = nat.GraphInfo()
    flags = nat.FLAG_WEIGHTS_F64 if weights64 else 0
    ctx.check(ctx.lib.fgbd_build_graph(ctx.handle, nat.ptr(pc.coords), pc.n_points, b,
                                       info, flags), "build_slg")
    return ctx, info


def _export(ctx, info, weighted: bool, bits: int) -> Graph:
    n, e, nnz = int(info.n), int(info.n_edges), int(info.nnz)
    indptr = np.zeros(n + 1, np.int64)
    indices = np.empty(nnz, np.int64)
    csr_edge = np.empty(nnz, np.int64)
    eu = np.empty(e, np.int64)
    ev = np.empty(e, np.int64)
    sq = np.empty(e, np.float64)
    w = np.empty(e, np.float64) if weighted else None
    ctx.check(ctx.lib.fgbd_graph_export(ctx.handle, nat.ptr(indptr), nat.ptr(indices),
                                        nat.ptr(csr_edge), nat.ptr(eu), nat.ptr(ev),
                                        nat.ptr(sq), nat.ptr(w), None), "graph export")
    tok = next(_tokens)
    ctx.graph_token = tok
    sg = float(info.sigma_g) if weighted else None
    return Graph(n, indptr, indices, csr_edge, eu, ev, sq, sg, w, _token=tok, _bits=bits,
                 _slg=True)


def build_slg(pc: PointCloud) -> Graph:
    """Scan-line graph: three device radix sorts + per-point dedup (graph.py:211-224)."""
    ctx, info = _device_build(pc)
    g = _export(ctx, info, weighted=False, bits=int(pc.bit_depth))
    object.__setattr__(g, "_sigma_dev", float(info.sigma_g))
    return g


def build_weighted_slg(pc: PointCloud) -> Graph:
    """Scan-line graph with Gaussian weights at the mean-edge-length scale."""
    ctx, info = _device_build(pc)
    if info.n_edges == 0:
        raise GraphError("cannot compute a distance scale on an edgeless graph")
    return _export(ctx, info, weighted=True, bits=int(pc.bit_depth))


def compute_sigma_g(pc: PointCloud, g: Graph) -> float:
    """Mean Euclidean length over the unique edges (graph.py:227-233), on device."""
    if g.n_edges == 0:
        raise GraphError("cannot compute a distance scale on an edgeless graph")
    ctx = nat.context()
    sg = nat.c_f64()
    ctx.check(ctx.lib.fgbd_edge_weights(ctx.handle, nat.ptr(g.edge_sqdist), g.n_edges,
                                        float("nan"), sg, None, 0), "compute_sigma_g")
    return float(sg.value)


def apply_gaussian_weights(g: Graph, sigma_g: float) -> Graph:
    """w = exp(-sqdist / sigma_g^2) per unique edge (Eq. 4, graph.py:236-245)."""
    if not sigma_g > 0:
        raise GraphError(f"sigma_g must be positive, got {sigma_g}")
    ctx = nat.context()
    w = np.empty(g.n_edges, np.float64)
    if g.n_edges:
        ctx.check(ctx.lib.fgbd_edge_weights(ctx.handle, nat.ptr(g.edge_sqdist), g.n_edges,
                                            float(sigma_g), None, nat.ptr(w), 0),
                  "apply_gaussian_weights")
    return Graph(g.n, g.indptr, g.indices, g.csr_edge, g.edge_u, g.edge_v, g.edge_sqdist,
                 float(sigma_g), w, _token=g._token, _bits=g._bits, _slg=g._slg)


def ensure_device_graph(pc: PointCloud, g: Graph | None, weights64: bool = False):
    """Make the calling thread's context hold the SLG of `pc`.

    Reuses the held copy when `g` is the graph this context built last;
    otherwise rebuilds it on the device from the cloud (the SLG is a pure
    function of the coordinates).  The device noise estimator and q scan run
    on the scan-line graph only: a graph built elsewhere (by hand, from
    fixtures) is accepted when it IS that graph -- same edges, and weights
    at its sigma_g equal to the device's -- and rejected loudly otherwise
    (`apply_filter` / `filter_step` take any CSR graph).
    """
    ctx = nat.context()
    if g is not None and g._token and ctx.graph_token == g._token and not weights64:
        return ctx
    if g is not None and g.n != pc.n_points:
        raise GraphError(f"graph has {g.n} vertices for a {pc.n_points}-point cloud")
    ctx.graph_token = None  # a failed rebuild leaves no valid graph behind
    ctx, info = _device_build(pc, weights64)
    if g is not None and not g._slg:
        _check_is_slg(ctx, info, g)
    ctx.graph_token = g._token if g is not None and g._token else None
    return ctx


def _check_is_slg(ctx, info, g: Graph) -> None:
    same = int(info.n_edges) == g.n_edges
    if same and g.n_edges:
        eu = np.empty(g.n_edges, np.int64)
        ev = np.empty(g.n_edges, np.int64)
        w = np.empty(g.n_edges, np.float64) if g.is_weighted else None
        ctx.check(ctx.lib.fgbd_graph_export(ctx.handle, None, None, None, nat.ptr(eu),
                                            nat.ptr(ev), None, nat.ptr(w), None), "graph export")
        same = np.array_equal(eu, g.edge_u) and np.array_equal(ev, g.edge_v)
        if same and w is not None:
            same = g.sigma_g == float(info.sigma_g) and np.allclose(
                w, g.edge_weights, rtol=1e-12, atol=0.0)
    if not same:
        raise GraphError("this stage runs on the device scan-line graph of the cloud; the "
                         "given graph differs from it (other graphs: apply_filter/filter_step)")


def build_knn_brute(pc: PointCloud, k: int) -> Graph:
    """Exact k-nearest-neighbour graph by exhaustive search on the device
    (graph.py:254-298): ties by point index, directed neighbour sets
    symmetrised by union.  The bench-graph baseline (paper Table 3), off the
    denoise path; integer or float coordinates."""
    n = pc.n_points
    k = int(k)
    if not 1 <= k < n:
        raise GraphError(f"k must satisfy 1 <= k < n_points, got k={k}, n={n}")
    ctx = nat.context()
    e = nat.c_i64()
    q = pc.is_quantized
    ctx.graph_token = None  # the sort scratch was shared with the held SLG
    ctx.check(ctx.lib.fgbd_knn_build(ctx.handle, nat.ptr(pc.coords) if q else None,
                                     None if q else nat.ptr(pc.coords), n, k,
                                     int(pc.bit_depth) if q else 0, e, 0), "build_knn_brute")
    m = int(e.value)
    indptr = np.empty(n + 1, np.int64)
    indices = np.empty(2 * m, np.int64)
    csr_edge = np.empty(2 * m, np.int64)
    eu = np.empty(m, np.int64)
    ev = np.empty(m, np.int64)
    sq = np.empty(m, np.float64)
    ctx.check(ctx.lib.fgbd_knn_export(ctx.handle, nat.ptr(indptr), nat.ptr(indices),
                                      nat.ptr(csr_edge), nat.ptr(eu), nat.ptr(ev), nat.ptr(sq)),
              "knn export")
    return Graph(n, indptr, indices, csr_edge, eu, ev, sq)
