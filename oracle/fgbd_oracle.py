"""CPU oracle for the FGBD denoise hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/fgbd/{graph,noise,filtering}.py`).  It exists to
check the CUDA product path and to serve as the timed CPU baseline
(`bench.py` cpu_baseline leg / `--impl reference`).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU legs may import it; the
product package `paper_2401_09721_b200` never does (it fails loudly when its
CUDA library is missing instead of falling back here).

Parity pinning: the outputs of this restatement are checked against golden
vectors produced by running the unmodified reference in the build container
(`tests/golden/make_golden.py`, fixtures under `tests/golden/`), and against
the SPEC.md known-answer examples (`tests/test_oracle.py`).

The restatement is deliberately *structurally different* from the reference
where the reference's structure is an implementation accident:

* the scan-line graph is built per point from rank neighbours (the shape the
  GPU uses) instead of `np.unique` over packed pair keys, and the edge list /
  `csr_edge` are derived as the row-major upper triangle -- the test suite
  proves this equals the reference's lexicographic edge list;
* the random-walk step accumulates `acc += w * f_j` over each row's
  neighbours in ascending column order from 0.0 with no FMA -- the order of
  the reference's scipy CSR matvec, which the oracle also calls (an
  explicit ELL view, `EllOperator.dense_rows`, gives the same bits).

Everything operates on plain numpy arrays: coords (N, 3) int64, colors
(N, 3) float64 in [0, 255].
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

# graph.py:25 -- (high, mid, low) coordinate axis of each scan-line code
LINE_AXES = {1: (2, 1, 0), 2: (0, 2, 1), 3: (1, 0, 2)}

JACOBI_MAX_SWEEPS = 50     # noise.py:21
SYMMETRY_RTOL = 1e-9       # noise.py:22
OFFDIAG_RTOL = 1e-12       # noise.py:23


class OracleError(ValueError):
    """Raised where the reference raises one of its ValueError subclasses."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # "graph" | "noise" | "filter" | "all_excluded"


# --------------------------------------------------------------------------
# a2/a3: scan-line codes and the stable LSD radix argsort
# --------------------------------------------------------------------------

def scanline_codes(coords: np.ndarray, bit_depth: int, line: int) -> np.ndarray:
    """Eqs. (1)-(3): code = hi << 2b | mid << b | lo  (graph.py:122-136)."""
    hi, mid, lo = LINE_AXES[line]
    g = np.asarray(coords).astype(np.uint64)
    b = np.uint64(bit_depth)
    return (g[:, hi] << (b + b)) | (g[:, mid] << b) | g[:, lo]


def radix_argsort(keys: np.ndarray, key_bits: int = 64) -> np.ndarray:
    """Stable LSD radix argsort, 8-bit digits, ceil(key_bits/8) passes.

    Restates graph.py:139-171: each pass is a stable counting sort of the
    current order by one byte of the key.  A stable numpy sort of the byte
    column is exactly a stable counting pass.
    """
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n = keys.size
    order = np.arange(n, dtype=np.int64)
    if n < 2:
        return order
    for shift in range(0, key_bits, 8):
        digit = (keys[order] >> np.uint64(shift)) & np.uint64(0xFF)
        order = order[np.argsort(digit.astype(np.uint16), kind="stable")]
    return order


def sort_permutation(coords, bit_depth, line):
    """graph.py:174-176."""
    return radix_argsort(scanline_codes(coords, bit_depth, line), 3 * bit_depth)


# --------------------------------------------------------------------------
# a4/a5: scan-line graph in the reference's conventions
# --------------------------------------------------------------------------

@dataclass
class OracleGraph:
    n: int
    indptr: np.ndarray      # (N+1,) int64
    indices: np.ndarray     # (nnz,) int64, ascending within each row
    csr_edge: np.ndarray    # (nnz,) int64 -> unique edge id
    edge_u: np.ndarray      # (E,) int64, edge_u < edge_v, lexicographic
    edge_v: np.ndarray
    edge_sqdist: np.ndarray  # (E,) float64 (exact integers)
    sigma_g: float | None = None
    edge_weights: np.ndarray | None = None

    @property
    def n_edges(self):
        return int(self.edge_u.size)

    def degrees(self):
        return np.diff(self.indptr)

    def weighted_degrees(self):
        """graph.py:78-85: bincount over edge_u plus bincount over edge_v.

        Per vertex i that is (sum over j>i, ascending j) + (sum over j<i,
        ascending j), each partial starting from 0.0.
        """
        w = self.edge_weights
        return (np.bincount(self.edge_u, weights=w, minlength=self.n)
                + np.bincount(self.edge_v, weights=w, minlength=self.n))

    def csr_weights(self):
        return self.edge_weights[self.csr_edge]


def _rows_from_candidates(cand: np.ndarray, n: int):
    """Sort + dedup up to 6 candidate neighbours per point (-1 = none)."""
    big = np.int64(n)  # sentinel sorts after every real index
    c = np.where(cand < 0, big, cand)
    c.sort(axis=1)
    dup = np.zeros_like(c, dtype=bool)
    dup[:, 1:] = c[:, 1:] == c[:, :-1]
    c[dup] = big
    c.sort(axis=1)
    valid = c < big
    deg = valid.sum(axis=1)
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=indptr[1:])
    return indptr, c[valid].astype(np.int64)


def build_slg(coords: np.ndarray, bit_depth: int) -> OracleGraph:
    """Scan-line graph (graph.py:179-224), built per point.

    Under scan line l, point perm_l[k] is adjacent to perm_l[k-1] and
    perm_l[k+1].  The union over l=1..3 with duplicates removed, rows sorted
    by index, is exactly the reference's CSR; unique edges are the upper
    triangle (j > i) enumerated row-major, which is the lexicographic order
    `np.unique(lo * n + hi)` produces.
    """
    coords = np.asarray(coords, np.int64)
    n = coords.shape[0]
    if n >= 2 ** 31:
        raise OracleError("graph", "point count exceeds the 2^31 edge-encoding limit")
    if n < 2:
        e = np.empty(0, np.int64)
        return OracleGraph(n, np.zeros(n + 1, np.int64), e, e, e, e, np.empty(0))
    cand = np.full((n, 6), -1, np.int64)
    for li, line in enumerate((1, 2, 3)):
        perm = sort_permutation(coords, bit_depth, line)
        cand[perm[1:], 2 * li] = perm[:-1]     # predecessor on the scan line
        cand[perm[:-1], 2 * li + 1] = perm[1:]  # successor on the scan line
    indptr, indices = _rows_from_candidates(cand, n)
    row = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    upper = indices > row
    edge_u = row[upper]
    edge_v = indices[upper]
    # edge id of every slot: upper slots are numbered in order; a lower slot
    # (i, j<i) is edge (j, i), found by binary search in the sorted key list.
    ukey = edge_u * n + edge_v
    skey = np.where(upper, row * n + indices, indices * n + row)
    csr_edge = np.searchsorted(ukey, skey).astype(np.int64)
    d = (coords[edge_u] - coords[edge_v]).astype(np.float64)
    sqdist = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]
    return OracleGraph(n, indptr, indices, csr_edge, edge_u, edge_v, sqdist)


def compute_sigma_g(g: OracleGraph) -> float:
    """graph.py:227-233: mean Euclidean length of the unique edges."""
    if g.n_edges == 0:
        raise OracleError("graph", "cannot compute a distance scale on an edgeless graph")
    return float(np.mean(np.sqrt(g.edge_sqdist)))


def apply_gaussian_weights(g: OracleGraph, sigma_g: float) -> OracleGraph:
    """Eq. (4), graph.py:236-245: w = exp(-sqdist / sigma_g^2)."""
    if not sigma_g > 0:
        raise OracleError("graph", f"sigma_g must be positive, got {sigma_g}")
    g.sigma_g = float(sigma_g)
    g.edge_weights = np.exp(-g.edge_sqdist / float(sigma_g) ** 2)
    return g


def build_weighted_slg(coords, bit_depth) -> OracleGraph:
    g = build_slg(coords, bit_depth)
    return apply_gaussian_weights(g, compute_sigma_g(g))


def quantize_coordinates(coords: np.ndarray, bits: int):
    """cloud.py:89-108: per-axis affine map of [min, max] onto [0, 2^b - 1],
    rint; integer clouds already on the grid pass through (returns None)."""
    g = np.asarray(coords)
    if np.issubdtype(g.dtype, np.integer) and g.min() >= 0 and g.max() < (1 << bits):
        return None
    lo = g.min(axis=0).astype(np.float64)
    span = g.max(axis=0).astype(np.float64) - lo
    scale = np.where(span > 0, ((1 << bits) - 1) / np.where(span > 0, span, 1.0), 0.0)
    return np.rint((g - lo) * scale).astype(np.int64)


def psnr(ref_colors: np.ndarray, test_colors: np.ndarray, cap_db: float = 100.0) -> float:
    """cloud.py:126-140: pooled MSE over all 3N values (numpy's pairwise
    summation in np.mean), 10 log10(255^2 / MSE), cap at zero error."""
    diff = np.asarray(ref_colors, np.float64) - np.asarray(test_colors, np.float64)
    mse = float(np.mean(diff * diff))
    if mse == 0.0:
        return float(cap_db)
    return float(10.0 * np.log10(255.0 ** 2 / mse))


# --------------------------------------------------------------------------
# add_gaussian_noise (cloud.py:111-123): numpy's Generator(Philox(seed)).normal
# restated -- Philox4x64-10 (numpy/random/src/philox/philox.h) and the
# 256-level ziggurat of random_standard_normal (distributions.c).  The third-
# party algorithm here is numpy's (2.3.5 in this image); the tables are read
# from numpy's own libnpyrandom.a (tools/gen_ziggurat_tables.py).  Pure Python:
# small cases only.
# --------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def philox4x64_10(ctr, key):
    c, k = list(ctr), list(key)
    for r in range(10):
        if r:
            k = [(k[0] + 0x9E3779B97F4A7C15) & _M64, (k[1] + 0xBB67AE8584CAA73B) & _M64]
        p0, p1 = 0xD2E7470EE14C6C93 * c[0], 0xCA5A826395121157 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & _M64, (p0 >> 64) ^ c[3] ^ k[1], p0 & _M64]
    return c


class PhiloxStream:
    """numpy's Philox draws from a BitGenerator state (counter, key)."""

    def __init__(self, counter, key):
        self.ctr = [int(v) for v in counter]
        self.key = [int(v) for v in key]
        self.buf: list = []

    def next_u64(self) -> int:
        if not self.buf:
            self.ctr[0] = (self.ctr[0] + 1) & _M64
            i = 0
            while self.ctr[i] == 0 and i < 3:
                i += 1
                self.ctr[i] = (self.ctr[i] + 1) & _M64
            self.buf = philox4x64_10(self.ctr, self.key)
        return self.buf.pop(0)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def standard_normal(st: PhiloxStream, ki, wi, fi) -> float:
    while True:
        r = st.next_u64()
        idx = r & 0xFF
        r >>= 8
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if r & 1:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-st.next_double())
                yy = -math.log1p(-st.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
        elif (fi[idx - 1] - fi[idx]) * st.next_double() + fi[idx] < math.exp(-0.5 * x * x):
            return x


def gaussian_noise(colors: np.ndarray, sigma: float, seed: int, ki, wi, fi) -> np.ndarray:
    """clip(colors + (0 + sigma z), 0, 255) in C order, z from seed's stream."""
    st0 = np.random.Philox(int(seed)).state["state"]
    st = PhiloxStream(st0["counter"], st0["key"])
    flat = np.asarray(colors, np.float64).reshape(-1)
    out = np.empty_like(flat)
    for k in range(flat.size):
        out[k] = min(max(flat[k] + (0.0 + sigma * standard_normal(st, ki, wi, fi)), 0.0), 255.0)
    return out.reshape(np.shape(colors))


def knn_rows(coords: np.ndarray, k: int, queries=None, chunk: int = 256) -> np.ndarray:
    """Exact k nearest neighbours (graph.py:254-285) for the given query rows.

    The reference scans j ascending and inserts on a strict `<`, so its row
    is the k smallest (squared distance, index) pairs, j != i.  Restated as a
    lexicographic selection over fp64 distances ((dx*dx + dy*dy) + dz*dz).
    """
    g = np.asarray(coords, np.float64)
    n = g.shape[0]
    if not 1 <= k < n:
        raise OracleError("graph", f"k must satisfy 1 <= k < n_points, got k={k}, n={n}")
    q = np.arange(n) if queries is None else np.asarray(queries, np.int64)
    out = np.empty((q.size, k), np.int64)
    idx = np.arange(n)
    for s0 in range(0, q.size, chunk):
        qs = q[s0:s0 + chunk]
        d = g[None, :, :] - g[qs, None, :]
        d2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        d2[np.arange(qs.size), qs] = np.inf  # never its own neighbour
        for r in range(qs.size):
            order = np.lexsort((idx, d2[r]))
            out[s0 + r] = order[:k]
    return out


def graph_from_pairs(coords: np.ndarray, u: np.ndarray, v: np.ndarray) -> OracleGraph:
    """Undirected union of directed pairs (graph.py:179-208) as an OracleGraph:
    rows are the sorted distinct partners of each vertex; edges the upper
    triangle row-major (== np.unique of lo * n + hi)."""
    g = np.asarray(coords)
    n = g.shape[0]
    u = np.asarray(u, np.int64)
    v = np.asarray(v, np.int64)
    keep = u != v
    src = np.concatenate([u[keep], v[keep]])
    dst = np.concatenate([v[keep], u[keep]])
    key = np.unique(src * n + dst)
    row, indices = key // n, key % n
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(row, minlength=n), out=indptr[1:])
    upper = indices > row
    edge_u, edge_v = row[upper], indices[upper]
    ukey = edge_u * n + edge_v
    skey = np.where(upper, row * n + indices, indices * n + row)
    csr_edge = np.searchsorted(ukey, skey).astype(np.int64)
    d = g[edge_u].astype(np.float64) - g[edge_v].astype(np.float64)
    # np.einsum("ij,ij->i") over 3 terms adds as (x*x + z*z) + y*y (its
    # two-lane inner loop); exact for integer coordinates, visible for floats
    sqdist = (d[:, 0] * d[:, 0] + d[:, 2] * d[:, 2]) + d[:, 1] * d[:, 1]
    return OracleGraph(n, indptr, indices.astype(np.int64), csr_edge, edge_u, edge_v, sqdist)


def build_knn_brute(coords: np.ndarray, k: int) -> OracleGraph:
    """graph.py:288-298 restated: knn_rows + graph_from_pairs."""
    nb = knn_rows(coords, k)
    n = nb.shape[0]
    return graph_from_pairs(coords, np.repeat(np.arange(n), k), nb.reshape(-1))


# --------------------------------------------------------------------------
# a9-a13: NE-GBP
# --------------------------------------------------------------------------

def extract_patches(colors: np.ndarray, g: OracleGraph, patch_size: int):
    """noise.py:82-119.  Returns (vectors (3, ne, D), eligible point ids).

    Patch = own value, then the D-1 nearest graph neighbours ordered by
    (squared distance, index).
    """
    d = int(patch_size)
    if d < 2:
        raise OracleError("noise", f"patch_size must be >= 2, got {patch_size}")
    deg = g.degrees()
    max_deg = int(deg.max(initial=0))
    if d > 1 + max_deg:
        raise OracleError("noise", f"patch_size {d} exceeds 1 + max degree ({1 + max_deg}) of this graph")
    elig = np.flatnonzero(deg >= d - 1)
    ne = elig.size
    width = max(max_deg, 1)
    col = np.arange(width)[None, :]
    ln = deg[elig][:, None]
    ok = col < ln
    pos = g.indptr[elig][:, None] + np.minimum(col, np.maximum(ln - 1, 0))
    nbr = np.where(ok, g.indices[pos] if g.indices.size else 0, np.int64(g.n))
    slot_d = g.edge_sqdist[g.csr_edge] if g.csr_edge.size else np.empty(0)
    dist = np.where(ok, slot_d[pos] if slot_d.size else 0.0, np.inf)
    order = np.lexsort((nbr, dist), axis=1)[:, : d - 1]
    pick = np.take_along_axis(nbr, order, axis=1)
    vec = np.empty((3, ne, d))
    for c in range(3):
        vec[c, :, 0] = colors[elig, c]
        vec[c, :, 1:] = colors[:, c][pick]
    return vec, elig


def patch_covariance(x: np.ndarray) -> np.ndarray:
    """noise.py:122-130: population covariance of one channel's (ne, D) patches."""
    ne = x.shape[0]
    if ne < 2:
        raise OracleError("noise", f"need at least 2 patches, have {ne}")
    xc = x - x.mean(axis=0)
    s = (xc.T @ xc) / ne
    return (s + s.T) * 0.5


# noise.py:152's off-diagonal norm is a difference of two sums and cannot
# resolve below ~sqrt(ulp(|a|^2)); the reference then reports non-convergence
# for matrices whose off-diagonal entries are exactly zero.  The CUDA path
# accepts such a matrix; tests set this flag to compute
# the result it must match.  Default False: the oracle is the reference.
JACOBI_DIRECT_OFF_FALLBACK = False


def symmetric_eigenvalues(s: np.ndarray, max_sweeps: int = JACOBI_MAX_SWEEPS) -> np.ndarray:
    """Cyclic Jacobi, descending eigenvalues (noise.py:133-185).

    Rotation (p<q): t from theta = (a_qq - a_pp) / (2 a_pq),
    c = 1/sqrt(1+t^2), s = t c; columns then rows are rotated and a_pq is
    zeroed.  Converged when the off-diagonal Frobenius norm <= 1e-12 ||S||.
    """
    s = np.asarray(s, np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise OracleError("noise", f"matrix must be square, got {s.shape}")
    scale = np.abs(s).max()
    if scale > 0 and np.abs(s - s.T).max() > SYMMETRY_RTOL * scale:
        raise OracleError("noise", "matrix is not symmetric within tolerance")
    a = np.array((s + s.T) * 0.5)
    n = a.shape[0]
    fro = np.linalg.norm(a)
    if fro == 0.0 or n == 1:
        return np.sort(np.diag(a))[::-1]
    tol = OFFDIAG_RTOL * fro

    def off_norm():
        return math.sqrt(max(float(np.sum(a * a) - np.sum(np.diag(a) ** 2)), 0.0))

    for _ in range(max_sweeps):
        if off_norm() <= tol:
            return np.sort(np.diag(a))[::-1]
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = a[p, q]
                if apq == 0.0:
                    continue
                gap = a[q, q] - a[p, p]
                if abs(apq) < 1e-36 * abs(gap):
                    t = apq / gap
                else:
                    th = gap / (2.0 * apq)
                    t = np.sign(th) / (abs(th) + np.hypot(th, 1.0))
                    if t == 0.0:
                        t = 1.0
                c = 1.0 / np.sqrt(t * t + 1.0)
                sn = t * c
                cp, cq = a[:, p].copy(), a[:, q].copy()
                a[:, p] = c * cp - sn * cq
                a[:, q] = sn * cp + c * cq
                rp, rq = a[p, :].copy(), a[q, :].copy()
                a[p, :] = c * rp - sn * rq
                a[q, :] = sn * rp + c * rq
                a[p, q] = a[q, p] = 0.0
    if off_norm() <= tol:
        return np.sort(np.diag(a))[::-1]
    if JACOBI_DIRECT_OFF_FALLBACK and math.sqrt(float(np.sum((a - np.diag(np.diag(a))) ** 2))) <= tol:
        return np.sort(np.diag(a))[::-1]
    raise OracleError("noise", f"Jacobi did not converge in {max_sweeps} sweeps")


def select_tail(lam: np.ndarray, divisor: str = "count"):
    """noise.py:188-216 -> (m, tau, fallback)."""
    lam = np.asarray(lam, np.float64)
    d = lam.size
    if d < 3:
        raise OracleError("noise", f"need at least 3 eigenvalues, got {d}")
    if divisor not in ("count", "count_plus_one"):
        raise OracleError("noise", f"unknown divisor rule {divisor!r}")
    extra = 0 if divisor == "count" else 1
    for m in range(1, d - 1):
        tail = lam[m:]
        tau = float(tail.sum() / (tail.size + extra))
        if tau > float(np.median(tail)):
            return m, tau, False
    m = d // 2
    tail = lam[m:]
    return m, float(tail.sum() / (tail.size + extra)), True


@dataclass
class OracleNoise:
    sigma_est: float
    per_channel_sigma: np.ndarray
    eigenvalues: np.ndarray
    m: np.ndarray
    tau: np.ndarray
    fallback: np.ndarray
    eligible_count: int


def estimate_noise_from_patches(vec: np.ndarray, divisor: str = "count") -> OracleNoise:
    """noise.py:219-243."""
    d = vec.shape[2]
    lam = np.empty((3, d))
    m = np.empty(3, np.int64)
    tau = np.empty(3)
    fb = np.empty(3, bool)
    sig = np.empty(3)
    for c in range(3):
        lam[c] = symmetric_eigenvalues(patch_covariance(vec[c]))
        m[c], tau[c], fb[c] = select_tail(lam[c], divisor)
        sig[c] = math.sqrt(max(tau[c], 0.0))
    return OracleNoise(float(sig.mean()), sig, lam, m, tau, fb, int(vec.shape[1]))


# --------------------------------------------------------------------------
# a14: FSLR
# --------------------------------------------------------------------------

def fslr_stat(vec: np.ndarray) -> np.ndarray:
    """Mean over channels of the population std of each patch (filtering.py:186)."""
    return vec.std(axis=2).mean(axis=0)


def fslr_mask(vec, elig, n, sigma_est, sigma_floor=0.5) -> np.ndarray:
    """filtering.py:175-194 -> include (N,) bool.  Raises all_excluded."""
    if sigma_est < sigma_floor:
        return np.ones(n, bool)
    inc = np.ones(n, bool)
    inc[elig[fslr_stat(vec) > 2.0 * sigma_est]] = False
    if not inc.any():
        raise OracleError("all_excluded", "the variance threshold excluded every point")
    return inc


# --------------------------------------------------------------------------
# a15-a18: random-walk low-pass filter and q selection
# --------------------------------------------------------------------------

class EllOperator:
    """The random-walk step operator of one weighted graph.

    Row i's neighbours are kept in ascending column order.  The product
    `sum_j w_ij f_j` accumulates `acc = acc + w * f_j` in that slot order
    from acc = 0.0 -- scipy's csr_matvecs loop, which this restatement calls
    for speed (the timed CPU baseline should not be slower than the
    reference's own scipy matvec).  `dense_rows()` gives the padded-row
    (ELL) view with (index 0, weight 0.0) padding for inspection; adding a
    +0.0 product leaves a finite accumulator unchanged, so both views give
    the same bits.
    """

    def __init__(self, g: OracleGraph):
        from scipy import sparse

        self.graph = g
        self.W = sparse.csr_matrix((g.csr_weights(), g.indices, g.indptr), shape=(g.n, g.n))
        self.d = g.weighted_degrees()
        self.width = int(g.degrees().max(initial=0))

    def dense_rows(self):
        g = self.graph
        deg = g.degrees()
        width = max(self.width, 1)
        idx = np.zeros((g.n, width), np.int64)
        w = np.zeros((g.n, width), np.float64)
        col = np.arange(width)[None, :]
        ok = col < deg[:, None]
        pos = (g.indptr[:-1][:, None] + col)[ok]
        idx[ok] = g.indices[pos]
        w[ok] = g.csr_weights()[pos]
        return idx, w

    def step(self, f: np.ndarray) -> np.ndarray:
        """filtering.py:132-155: out = (d f + W f) / (2 d); d == 0 passes through."""
        acc = self.W @ f
        dcol = self.d[:, None] if f.ndim == 2 else self.d
        with np.errstate(invalid="ignore", divide="ignore"):
            out = (dcol * f + acc) / (2.0 * dcol)
        iso = self.d == 0.0
        if iso.any():
            out[iso] = f[iso]
        return out


def selection_criterion(y, x, include, sigma_est, mode="pooled") -> float:
    """Eq. (6), filtering.py:197-222."""
    count = int(include.sum())
    if count < 1:
        raise OracleError("filter", "criterion needs at least one included point")
    sv2 = float(sigma_est) ** 2
    if mode == "pooled":
        lost = (np.sum(y[include] ** 2) - np.sum(x[include] ** 2)) / (count * y.shape[1])
        return float(abs(sv2 - lost))
    if mode == "per_channel":
        lost = (np.sum(y[include] ** 2, axis=0) - np.sum(x[include] ** 2, axis=0)) / count
        return float(np.mean(np.abs(sv2 - lost)))
    raise OracleError("filter", f"unknown criterion mode {mode!r}")


def select_q(y, op: EllOperator, sigma_est, include, q_max=64, mode="pooled",
             early_exit=True, trace=None):
    """filtering.py:225-256.  Returns (q, x_q, steps_executed).

    `trace`, when a list, receives the criterion value of every q visited.
    """
    if sigma_est < 0:
        raise OracleError("filter", f"sigma_est must be >= 0, got {sigma_est}")
    x = y.copy()
    best_q, best_x = 0, x.copy()
    best = selection_criterion(y, x, include, sigma_est, mode)
    if trace is not None:
        trace.append(best)
    prev, streak, steps = best, 0, 0
    for q in range(1, q_max + 1):
        if best == 0.0:
            break
        x = op.step(x)
        steps += 1
        crit = selection_criterion(y, x, include, sigma_est, mode)
        if trace is not None:
            trace.append(crit)
        if crit < best:
            best_q, best, best_x = q, crit, x.copy()
        streak = streak + 1 if crit > prev else 0
        prev = crit
        if early_exit and streak >= 3:
            break
    return best_q, best_x, steps


@dataclass
class OracleConfig:
    """Mirror of FilterConfig (filtering.py:33-59)."""
    q_max: int = 64
    epsilon: float | None = None
    fslr_enabled: bool = True
    patch_size: int = 7
    reestimate_interval: int = 10
    fslr_sigma_floor: float = 0.5
    criterion_mode: str = "pooled"
    early_exit: bool = True
    tau_divisor: str = "count"


@dataclass
class OracleResult:
    colors: np.ndarray
    selected_q: int
    sigma_est: float
    masked_fraction: float
    criterion_value: float | None = None
    converged: bool | None = None
    cached: bool = False
    eligible_count: int | None = None
    steps: int = 0
    all_excluded_fallback: bool = False
    noise: OracleNoise | None = None
    include: np.ndarray | None = None
    graph: OracleGraph | None = None
    trace: list = field(default_factory=list)
    stage_timings: dict = field(default_factory=dict)


def denoise(coords, colors, bit_depth, cfg: OracleConfig | None = None,
            cached_q: int | None = None, cached_sigma_est: float | None = None,
            keep_graph: bool = False) -> OracleResult:
    """filtering.py:259-328 on plain arrays."""
    cfg = cfg or OracleConfig()
    coords = np.asarray(coords, np.int64)
    y = np.asarray(colors, np.float64)
    n = coords.shape[0]
    if n < 2:
        return OracleResult(y, 0, 0.0, 0.0)
    t = {}
    t0 = time.perf_counter()
    g = build_weighted_slg(coords, bit_depth)
    op = EllOperator(g)
    t["graph_construction"] = time.perf_counter() - t0
    if cached_q is None:
        t0 = time.perf_counter()
        vec, elig = extract_patches(y, g, cfg.patch_size)
        est = estimate_noise_from_patches(vec, cfg.tau_divisor)
        fallback = False
        if cfg.fslr_enabled:
            try:
                inc = fslr_mask(vec, elig, n, est.sigma_est, cfg.fslr_sigma_floor)
            except OracleError as e:
                if e.kind != "all_excluded":
                    raise
                warnings.warn("variance mask excluded every point; selecting unmasked")
                inc = np.ones(n, bool)
                fallback = True
        else:
            inc = np.ones(n, bool)
        t["noise_estimation"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        trace: list = []
        q, x, steps = select_q(y, op, est.sigma_est, inc, cfg.q_max,
                               cfg.criterion_mode, cfg.early_exit, trace)
        t["low_pass_filter"] = time.perf_counter() - t0
        crit = selection_criterion(y, x, inc, est.sigma_est, cfg.criterion_mode)
        eps = cfg.epsilon if cfg.epsilon is not None else 1e-3 * est.sigma_est ** 2
        res = OracleResult(np.clip(x, 0.0, 255.0), q, est.sigma_est,
                           1.0 - int(inc.sum()) / n, crit, bool(crit <= eps), False,
                           est.eligible_count, steps, fallback, est, inc,
                           trace=trace, stage_timings=t)
    else:
        if cached_q < 0:
            raise OracleError("filter", f"cached_q must be >= 0, got {cached_q}")
        t["noise_estimation"] = 0.0
        t0 = time.perf_counter()
        x = y
        for _ in range(cached_q):
            x = op.step(x)
        t["low_pass_filter"] = time.perf_counter() - t0
        res = OracleResult(np.clip(x, 0.0, 255.0), int(cached_q),
                           float(cached_sigma_est) if cached_sigma_est is not None else 0.0,
                           0.0, cached=True, steps=int(cached_q), stage_timings=t)
    if keep_graph:
        res.graph = g
    return res
