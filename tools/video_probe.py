"""Per-frame timings of the sequence driver (diagnostics)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb
from paper_2401_09721_b200 import _native as nat
from paper_2401_09721_b200.sequence import denoise_sequence

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
pool = []
for s in range(8):
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1 + s)
    c = nat.pinned_empty(noisy.coords.shape, np.int64); c[...] = noisy.coords
    y = nat.pinned_empty(noisy.colors.shape, np.float64); y[...] = noisy.colors
    pool.append(fb.PointCloud(c, y, noisy.bit_depth))
walls = {}
def timed(pc, cfg=fb.FilterConfig(), cached_q=None, cached_sigma_est=None):
    t0 = time.perf_counter()
    r = fb.denoise(pc, cfg, cached_q=cached_q, cached_sigma_est=cached_sigma_est)
    walls[id(r[1])] = (time.perf_counter() - t0, r[1].device["t_total"])
    return r
def sink(i, pc, rep): pass
for rep in range(2):
    walls.clear()
    t0 = time.perf_counter()
    res = denoise_sequence(lambda i: pool[i % 8], n_frames=60, workers=workers, denoise_fn=timed, sink=sink)
    wall = time.perf_counter() - t0
    w = np.array([walls[id(r[1])] for f, r in sorted(res.items())])
    print(f"workers={workers} run{rep}: {60/wall:.1f} fps; per-call wall ms min/med/max "
          f"{1e3*w[:,0].min():.2f}/{1e3*np.median(w[:,0]):.2f}/{1e3*w[:,0].max():.2f}; device ms med "
          f"{1e3*np.median(w[:,1]):.2f}; pool out allocs {nat._pool.allocs} reuses {nat._pool.reuses}")
