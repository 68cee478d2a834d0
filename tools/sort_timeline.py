"""Per-tile timeline of the onesweep radix passes (experiment tool).

    python -c "from paper_2401_09721_b200._build import build; \\
        build(defines=('FGBD_SORT_TLOG=1',), lib='tools/_lib_stlog.so')"
    FGBD_LIB_PATH=tools/_lib_stlog.so python tools/sort_timeline.py [--kind ramp] [--n 1000000]

Per pass and line: kernel span, tile start waves, and the per-tile phases
(load + multisplit, decoupled look-back, scan + reorder + scatter).
"""

from __future__ import annotations

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="ramp")
    ap.add_argument("--n", type=int, default=1_000_000)
    a = ap.parse_args()
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    clean, _ = fb.generate_cloud(a.kind, a.n, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    ctx = nat.context()
    dc = torch.from_numpy(np.array(noisy.coords)).cuda()
    dy = torch.from_numpy(np.array(noisy.colors)).cuda()
    do = torch.empty_like(dy)
    cfg = nat.make_config(fb.FilterConfig())
    for _ in range(3):
        rep = nat.Report()
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, dc.data_ptr(), dy.data_ptr(), a.n,
                                       noisy.bit_depth, cfg, -1, float("nan"),
                                       do.data_ptr(), rep, nat.FLAG_DEVICE_PTRS), "denoise")
    torch.cuda.synchronize()
    print(f"GC={rep.t_graph_construction*1e3:.3f} ms")
    buf = np.zeros((4, 3, 1024, 4), np.uint64)
    fn = ctx.lib.fgbd_debug_stlog
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p]
    assert fn(buf.ctypes.data) == 0
    for p in range(4):
        tiles = int(np.count_nonzero(buf[p, 0, :, 0]))
        if not tiles:
            continue
        t = buf[p, :, :tiles, :].astype(np.int64)
        t0 = t[:, :, 0].min()
        t = (t - t0) / 1e3
        span = t[:, :, 3].max()
        st = t[:, :, 0]
        print(f"pass {p}: tiles/line={tiles} span={span:.2f} us; start: "
              f"p50={np.median(st):.2f} p90={np.percentile(st, 90):.2f} max={st.max():.2f}")
        split = t[:, :, 1] - t[:, :, 0]
        look = t[:, :, 2] - t[:, :, 1]
        tail = t[:, :, 3] - t[:, :, 2]
        for name, v in (("load+split", split), ("look-back", look), ("scan+scatter", tail)):
            print(f"   {name:13s} p10={np.percentile(v, 10):6.2f} p50={np.median(v):6.2f} "
                  f"p90={np.percentile(v, 90):6.2f} max={v.max():6.2f}")
        # look-back wait vs tile index (line 0)
        lb = look[0]
        q = [int(x) for x in np.linspace(0, tiles - 1, 9)]
        print("   look-back by tile index (line 0):", [(k, round(float(lb[k]), 2)) for k in q])


if __name__ == "__main__":
    main()
