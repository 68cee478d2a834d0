"""CPU: the slab partition's cross-slab protocol (csrc/slab.cu).

Each rank sorts only its own z-slab along the 3 scan lines and publishes,
per line, its block list (first / last point of every run sharing the line's
key above z).  A rank's true scan-line neighbours are the local sort's
neighbours inside a block, and at block ends the last / first point of the
(key, rank)-adjacent block over all ranks (k_resolve, csrc/graph.cu).

This restates that protocol in numpy and checks, for several geometries,
point orders and rank counts, that it reproduces the oracle's scan-line
neighbours (and hence the reference's graph) exactly.  The GPU tests run the
CUDA implementation against the reference fixtures.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O
from paper_2401_09721_b200.slab import slab_partition

LINES = (1, 2, 3)


def _seg_key(code, line, b):
    """Key above z: line 1 -> 0, line 2 (x, z, y) -> x, line 3 (y, x, z) -> (y, x)."""
    if line == 1:
        return np.zeros_like(code)
    return code >> np.uint64(2 * b) if line == 2 else code >> np.uint64(b)


def _blocks(gidx, coords, b, line):
    """Own block list of one line: (key, first gidx, last gidx) in sorted order,
    and the own sorted order (stable in global index)."""
    code = O.scanline_codes(coords, b, line)
    order = np.argsort(code, kind="stable")  # own points are in increasing gidx
    key = _seg_key(code[order], line, b)
    start = np.ones(order.size, bool)
    start[1:] = key[1:] != key[:-1]
    first = np.flatnonzero(start)
    last = np.concatenate([first[1:] - 1, [order.size - 1]])
    return key[first], gidx[order[first]], gidx[order[last]], gidx[order], key


def _protocol_neighbours(coords, b, world):
    """Per line: (prev, next) global neighbour of every point, via the protocol."""
    pc = fb.PointCloud(coords, np.zeros(coords.shape, np.float64), b)
    part = slab_partition(pc, world)
    n = coords.shape[0]
    out = {line: np.full((n, 2), -1, np.int64) for line in LINES}
    lists = {}
    for r in range(world):
        g = part.own_index(r)
        for line in LINES:
            lists[r, line] = _blocks(g, coords[g], b, line)
    for r in range(world):
        for line in LINES:
            keys, fg, lg, sorted_g, skey = lists[r, line]
            nb = out[line]
            # inside blocks: the local sort's neighbours
            same = skey[1:] == skey[:-1]
            nb[sorted_g[1:][same], 0] = sorted_g[:-1][same]
            nb[sorted_g[:-1][same], 1] = sorted_g[1:][same]
            for bi, k in enumerate(keys):
                pred = succ = None  # (key', rank', gidx)
                if bi > 0:
                    pred = (keys[bi - 1], r, lg[bi - 1])
                if bi + 1 < len(keys):
                    succ = (keys[bi + 1], r, fg[bi + 1])
                for s in range(world):
                    if s == r:
                        continue
                    ks, fgs, lgs = lists[s, line][:3]
                    # s < r: largest key' <= k; s > r: largest key' < k
                    p = np.searchsorted(ks, k, side="right" if s < r else "left") - 1
                    if p >= 0 and (pred is None or (ks[p], s) > pred[:2]):
                        pred = (ks[p], s, lgs[p])
                    # s > r: smallest key' >= k; s < r: smallest key' > k
                    q = np.searchsorted(ks, k, side="right" if s < r else "left")
                    if q < len(ks) and (succ is None or (ks[q], s) < succ[:2]):
                        succ = (ks[q], s, fgs[q])
                nb[fg[bi], 0] = -1 if pred is None else pred[2]
                nb[lg[bi], 1] = -1 if succ is None else succ[2]
    return out, part


def _oracle_neighbours(coords, b):
    n = coords.shape[0]
    out = {}
    for line in LINES:
        perm = O.sort_permutation(coords, b, line)
        nb = np.full((n, 2), -1, np.int64)
        nb[perm[1:], 0] = perm[:-1]
        nb[perm[:-1], 1] = perm[1:]
        out[line] = nb
    return out


def _cloud(kind, n, seed, order):
    clean, _ = fb.generate_cloud(kind, n, seed=seed)
    g = np.array(clean.coords)
    if order == "shuffle":
        g = g[np.random.default_rng(seed).permutation(n)]
    elif order == "reverse":
        g = g[::-1].copy()
    return g, clean.bit_depth


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("kind,n,order", [("ramp", 9000, "asis"), ("ramp", 9000, "shuffle"),
                                          ("constant", 6000, "asis"),
                                          ("two-tone", 7000, "reverse")])
def test_protocol_reproduces_scan_line_neighbours(world, kind, n, order):
    coords, b = _cloud(kind, n, 3, order)
    got, part = _protocol_neighbours(coords, b, world)
    want = _oracle_neighbours(coords, b)
    assert int(part.counts.sum()) == n and np.all(part.counts >= 1)
    for line in LINES:
        np.testing.assert_array_equal(got[line], want[line], err_msg=f"line {line}")


def test_protocol_with_duplicates_and_sparse_planes():
    rng = np.random.default_rng(11)
    coords = rng.integers(0, 6, size=(3000, 3))
    coords[:, 2] = rng.choice([0, 1, 4, 5], size=3000)  # empty z planes between slabs
    coords[100:140] = coords[0]                          # duplicates of one point
    got, _ = _protocol_neighbours(coords, 3, 3)
    want = _oracle_neighbours(coords, 3)
    for line in LINES:
        np.testing.assert_array_equal(got[line], want[line])


def test_partition_is_z_slabs_in_line1_order():
    coords, b = _cloud("ramp", 20000, 0, "shuffle")
    pc = fb.PointCloud(coords, np.zeros(coords.shape), b)
    part = slab_partition(pc, 4)
    assert part.order is not None  # shuffled: not z-sorted
    perm1 = O.sort_permutation(coords, b, 1)
    # rank r's points are exactly line-1 ranks [starts[r], starts[r+1])
    for r in range(4):
        want = np.sort(perm1[part.starts[r]:part.starts[r + 1]])
        np.testing.assert_array_equal(part.own_index(r), want)
    assert abs(int(part.counts.max()) - 5000) < 1000
    ordered, b2 = _cloud("ramp", 20000, 0, "asis")
    part2 = slab_partition(fb.PointCloud(ordered, np.zeros(ordered.shape), b2), 4)
    assert part2.order is None  # raster order: contiguous index ranges
    assert slab_partition(fb.PointCloud(ordered, np.zeros(ordered.shape), b2), 4).world == 4


def test_partition_rejects_too_few_planes():
    coords = np.zeros((10, 3), np.int64)
    coords[:, 0] = np.arange(10)
    with pytest.raises(fb.FilterError):
        slab_partition(fb.PointCloud(coords, np.zeros((10, 3)), 4), 2)
