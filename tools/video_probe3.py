"""Raw C-ABI throughput of cached static-geometry frames: 1..4 host threads,
each calling fgbd_denoise(REUSE) on pinned frames in a tight loop."""
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200 import _native as nat  # noqa: E402

clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
frames = []
for s in range(8):
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1 + s)
    c = nat.pinned_empty(noisy.coords.shape, np.int64)
    c[...] = noisy.coords
    y = nat.pinned_empty(noisy.colors.shape, np.float64)
    y[...] = noisy.colors
    frames.append((c, y, noisy.bit_depth))
cfg = nat.make_config(fb.FilterConfig())


def worker(k, nframes, out_times, q, flags):
    ctx = nat.context()
    out = nat.pinned_empty((1_000_000, 3), np.float64)
    rep = nat.Report()
    t0 = time.perf_counter()
    for f in range(nframes):
        c, y, b = frames[(k + f) % 8]
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, nat.ptr(c), nat.ptr(y), c.shape[0], b, cfg, q,
                                       float("nan"), nat.ptr(out), rep, flags), "denoise")
    out_times[k] = time.perf_counter() - t0


from concurrent.futures import ThreadPoolExecutor

pools = {n: ThreadPoolExecutor(max_workers=n) for n in (1, 2, 3)}
for q in (64, -1):
    for flags, tag in ((nat.FLAG_REUSE_GRAPH, "reuse"), (0, "rebuild")):
        for nthr in (1, 2, 3):
            per = 40
            times = {}
            ex = pools[nthr]
            list(ex.map(lambda k: worker(k, 3, times, q, flags), range(nthr)))  # warm contexts
            t0 = time.perf_counter()
            list(ex.map(lambda k: worker(k, per, times, q, flags), range(nthr)))
            wall = time.perf_counter() - t0
            print(f"q={q:3d} {tag:7s} threads={nthr}: {nthr * per / wall:7.1f} frames/s")
