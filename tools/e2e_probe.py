"""Where does end-to-end time go?  Wall time of the public API vs the raw C call."""

from __future__ import annotations

import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    pcc = nat.pinned_empty(noisy.coords.shape, np.int64)
    pcc[...] = noisy.coords
    pcy = nat.pinned_empty(noisy.colors.shape, np.float64)
    pcy[...] = noisy.colors
    pc = fb.PointCloud(pcc, pcy, noisy.bit_depth)
    ctx = nat.context()
    cfg = nat.make_config(fb.FilterConfig())
    out = nat.pinned_empty((pc.n_points, 3), np.float64)
    for _ in range(3):
        fb.denoise(pc)

    def raw():
        rep = nat.Report()
        t0 = time.perf_counter()
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, nat.ptr(pc.coords), nat.ptr(pc.colors),
                                       pc.n_points, pc.bit_depth, cfg, -1, float("nan"),
                                       nat.ptr(out), rep, 0), "denoise")
        return time.perf_counter() - t0, rep

    walls, devs = [], []
    for _ in range(10):
        w, rep = raw()
        walls.append(w)
        devs.append(rep.t_total)
    print(f"raw C call: wall {1e3 * np.mean(walls):.3f} ms, device events {1e3 * np.mean(devs):.3f} ms")
    walls = []
    for _ in range(10):
        t0 = time.perf_counter()
        o, r = fb.denoise(pc)
        walls.append(time.perf_counter() - t0)
        del o
    print(f"fb.denoise: wall {1e3 * np.mean(walls):.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        o, r = fb.denoise(pc)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(6)
    print("pool allocs", nat._pool.allocs, "reuses", nat._pool.reuses, "free",
          {k: len(v) for k, v in nat._pool.free.items()}, "outstanding", nat._pool.outstanding)
    import gc
    o = None
    gc.collect()
    print("after gc: free", {k: len(v) for k, v in nat._pool.free.items()})


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def torch_variants():
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    pcc = nat.pinned_empty(noisy.coords.shape, np.int64)
    pcc[...] = noisy.coords
    pcy = nat.pinned_empty(noisy.colors.shape, np.float64)
    pcy[...] = noisy.colors
    pc = fb.PointCloud(pcc, pcy, noisy.bit_depth)
    ctx = nat.context()
    stream = torch.cuda.ExternalStream(ctx.lib.fgbd_ctx_stream(ctx.handle))
    flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device="cuda")
    for _ in range(3):
        fb.denoise(pc)
    for mode in ("plain", "sync", "flush+sync", "flush-async"):
        walls, devs = [], []
        for k in range(10):
            if mode in ("flush+sync", "flush-async"):
                with torch.cuda.stream(stream):
                    flush.fill_(k)
            if mode in ("sync", "flush+sync"):
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            o, r = fb.denoise(pc)
            walls.append(time.perf_counter() - t0)
            devs.append(r.device["t_total"])
        print(f"{mode:12s} wall {1e3 * np.mean(walls):.3f} ms  device {1e3 * np.mean(devs):.3f} ms")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "torch":
    torch_variants()
