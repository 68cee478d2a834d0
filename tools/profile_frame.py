"""Small driver for ncu: denoise a few device-resident frames.

    python tools/profile_frame.py [--kind ramp] [--n 1000000] [--frames 3]

Launch order per frame (config 2, ramp, b=7): k_prep, 3 x k_onesweep,
k_neighbors, k_rows, k_expand (side stream), k_noise2 (weights fused),
k_reduce_cols, k_mask, k_lf_run (all S steps), k_compact.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="ramp")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--sigma", type=float, default=10.0)
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--cached", type=int, default=-1)
    ap.add_argument("--no-early-exit", action="store_true")
    ap.add_argument("--order", default="asis",
                    help="permute the points before upload (locality experiments): asis, shuffle, "
                         "morton, line1, brickN (N^3 voxel bricks in row-major brick order, "
                         "line-1 order inside a brick), slabN (z slabs of N, line-1 inside)")
    a = ap.parse_args()
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    clean, _ = fb.generate_cloud(a.kind, a.n, seed=0)
    noisy = fb.add_gaussian_noise(clean, a.sigma, seed=1)
    if a.order != "asis":
        g = np.array(noisy.coords)
        if a.order == "shuffle":
            perm = np.random.default_rng(7).permutation(a.n)
        elif a.order == "line1":
            perm = np.lexsort((g[:, 0], g[:, 1], g[:, 2]))
        elif a.order.startswith("brick"):
            e = int(a.order[5:])
            hi = g // e
            lo = g % e
            perm = np.lexsort((lo[:, 0], lo[:, 1], lo[:, 2], hi[:, 0], hi[:, 1], hi[:, 2]))
        elif a.order.startswith("slab"):
            e = int(a.order[4:])
            perm = np.lexsort((g[:, 0], g[:, 1], g[:, 2] % e, g[:, 2] // e))
        else:  # morton (z-order) of the voxel coordinates
            def spread(v):
                v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
                out = np.zeros_like(v)
                for bit in range(21):
                    out |= ((v >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit)
                return out
            code = spread(g[:, 0]) | (spread(g[:, 1]) << np.uint64(1)) | (spread(g[:, 2]) << np.uint64(2))
            perm = np.argsort(code, kind="stable")
        noisy = fb.PointCloud(g[perm], np.array(noisy.colors)[perm], noisy.bit_depth)
    ctx = nat.context()
    dc = torch.from_numpy(np.array(noisy.coords)).cuda()
    dy = torch.from_numpy(np.array(noisy.colors)).cuda()
    do = torch.empty_like(dy)
    cfg = nat.make_config(fb.FilterConfig(early_exit=not a.no_early_exit))
    for f in range(a.frames):
        rep = nat.Report()
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, dc.data_ptr(), dy.data_ptr(), a.n,
                                       noisy.bit_depth, cfg, a.cached, float("nan"),
                                       do.data_ptr(), rep, nat.FLAG_DEVICE_PTRS), "denoise")
        print(f"frame {f}: q={rep.selected_q} S={rep.steps} launches={rep.gpu_launches} "
              f"GC={rep.t_graph_construction*1e3:.3f}ms NE={rep.t_noise_estimation*1e3:.3f}ms "
              f"LF={rep.t_low_pass_filter*1e3:.3f}ms lf_steps={rep.t_lf_steps*1e3:.3f}ms "
              f"total={rep.t_total*1e3:.3f}ms")


if __name__ == "__main__":
    main()
