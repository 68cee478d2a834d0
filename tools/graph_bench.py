"""bench-graph on the B200: SLG vs brute-force kNN build time, CSV rows.

    python tools/graph_bench.py --sizes 10000,100000,1000000 [--k 6 --bits 10]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2401_09721_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="10000,100000,1000000")
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--bits", type=int, default=10)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
rows = fb.run_graph_bench([int(s) for s in a.sizes.split(",")], k=a.k, bits=a.bits, seed=a.seed)
print(fb.rows_to_csv(rows), end="")
