"""Diagnostic: where the host time of the public denoise(PointCloud) call
goes (pinned 1M-point frame): wall time per call against the library's own
first-to-last event time, and a cProfile of the Python side."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200 import _native as nat  # noqa: E402


def main():
    clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    c = nat.pinned_empty(noisy.coords.shape, np.int64)
    c[...] = noisy.coords
    y = nat.pinned_empty(noisy.colors.shape, np.float64)
    y[...] = noisy.colors
    pc = fb.PointCloud(c, y, noisy.bit_depth)
    for _ in range(3):
        fb.denoise(pc)
    walls, libs = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        out, rep = fb.denoise(pc)
        walls.append(time.perf_counter() - t0)
        libs.append(rep.device["t_total"])
    print("wall %.3f ms, library events %.3f ms" % (1e3 * np.median(walls), 1e3 * np.median(libs)))
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        fb.denoise(pc)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__":
    main()
