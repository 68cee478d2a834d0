"""Timeline of the sequence driver with static-geometry reuse: per-call wall
time split into the library's own phases (diagnostics)."""
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200 import _native as nat  # noqa: E402
from paper_2401_09721_b200.filtering import denoise_frame  # noqa: E402
from paper_2401_09721_b200.sequence import denoise_sequence  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
pool = []
for s in range(8):
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1 + s)
    c = nat.pinned_empty(noisy.coords.shape, np.int64)
    c[...] = noisy.coords
    y = nat.pinned_empty(noisy.colors.shape, np.float64)
    y[...] = noisy.colors
    pool.append(fb.PointCloud(c, y, noisy.bit_depth))
log = []
T0 = [0.0]


def timed(pc, cfg=fb.FilterConfig(), cached_q=None, cached_sigma_est=None):
    t0 = time.perf_counter()
    r = denoise_frame(pc, cfg, cached_q, cached_sigma_est, reuse_graph=True)
    t1 = time.perf_counter()
    d = r[1].device
    log.append((threading.get_ident() % 1000, t0 - T0[0], t1 - T0[0], d["t_total"], d["t_h2d"],
                d["t_d2h"], d["graph_reused"], r[1].cached))
    return r


for rep in range(2):
    log.clear()
    T0[0] = time.perf_counter()
    res = denoise_sequence(lambda i: pool[i % 8], n_frames=60, workers=workers,
                           denoise_fn=timed, sink=lambda i, pc, rep: None)
    wall = time.perf_counter() - T0[0]
    print(f"workers={workers} run{rep}: {60 / wall:.1f} fps")
for row in sorted(log, key=lambda r: r[1])[:16]:
    tid, a, b, tot, h2d, d2h, reused, cached = row
    print(f"thr {tid:3d}  start {1e3*a:7.2f}  end {1e3*b:7.2f}  wall {1e3*(b-a):5.2f}  "
          f"dev_total {1e3*tot:5.2f}  h2d {1e3*h2d:5.2f}  d2h {1e3*d2h:5.2f}  reuse {reused} cached {cached}")
