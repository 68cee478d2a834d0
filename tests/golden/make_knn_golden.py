"""Freeze brute-force kNN graphs and bench-graph rows from the UNMODIFIED
reference (`fgbd.build_knn_brute`, `fgbd.bench.run_graph_bench`).

Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_knn_golden.py

Writes tests/golden/knn.npz + knn_index.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import fgbd  # noqa: E402  (the reference)
from fgbd.bench import run_graph_bench  # noqa: E402

OUT = Path(__file__).resolve().parent
FIELDS = ("indptr", "indices", "csr_edge", "edge_u", "edge_v", "edge_sqdist")


def clouds():
    """(name, cloud, params) -- params regenerate synthetic clouds."""
    out = []
    for kind, n, bits, seed in (("constant", 500, 4, 1), ("constant", 2000, 10, 2),
                                ("constant", 1500, 17, 3), ("grid", 343, None, 0),
                                ("ramp", 1000, None, 0)):
        pc, _ = fgbd.generate_cloud(kind, n, bits=bits, seed=seed)
        out.append((f"{kind}_{n}_b{bits}", pc, dict(kind=kind, n=n, bits=bits, seed=seed)))
    rng = np.random.default_rng(7)
    fl = rng.normal(size=(400, 3)) * np.array([1.0, 10.0, 0.1])
    fl[10] = fl[11]  # a coincident pair
    out.append(("float_400", fgbd.PointCloud(fl, np.full((400, 3), 100.0), None), None))
    dup = rng.integers(0, 5, size=(300, 3))  # heavy duplication: many zero distances
    out.append(("dups_300", fgbd.PointCloud(dup, np.full((300, 3), 50.0), 3), None))
    return out


def main():
    arrays, index = {}, {"graphs": {}, "bench": {}}
    for name, pc, params in clouds():
        if params is None:
            arrays[f"{name}/coords"] = np.asarray(pc.coords)
        for k in (1, 6, 11):
            g = fgbd.build_knn_brute(pc, k)
            key = f"{name}/k{k}"
            for f in FIELDS:
                arrays[f"{key}/{f}"] = np.asarray(getattr(g, f))
            index["graphs"][key] = {"cloud": name, "k": k, "params": params,
                                    "bit_depth": pc.bit_depth, "n_edges": g.n_edges}
    for k, bits, sizes in ((6, 10, [300, 1200]), (4, 8, [700])):
        rows = run_graph_bench(sizes, k=k, bits=bits, seed=5)
        index["bench"][f"k{k}_b{bits}"] = {
            "k": k, "bits": bits, "sizes": sizes, "seed": 5,
            "rows": [{"n": r.n, "mean_degree": r.mean_degree, "overlap": r.overlap}
                     for r in rows]}
    errs = {}
    pc, _ = fgbd.generate_cloud("constant", 10, bits=4, seed=0)
    for k in (0, 10, -1):
        try:
            fgbd.build_knn_brute(pc, k)
        except Exception as e:  # noqa: BLE001 -- recording the reference's behaviour
            errs[str(k)] = [type(e).__name__, str(e)]
    index["errors"] = errs
    np.savez_compressed(OUT / "knn.npz", **arrays)
    (OUT / "knn_index.json").write_text(json.dumps(index, indent=1, sort_keys=True))
    print(f"wrote {len(arrays)} arrays, {len(index['graphs'])} graphs")


if __name__ == "__main__":
    main()
