"""Per-block timeline of the persistent filter kernel (experiment tool).

    python -c "from paper_2401_09721_b200._build import build; \
        build(defines=('FGBD_LF_TLOG=1',), lib='tools/_lib_tlog.so')"
    FGBD_LIB_PATH=tools/_lib_tlog.so python tools/lf_timeline.py [--kind ramp] [--n 1000000]

For the first 16 steps of the last frame, each block records %globaltimer at
step start (after the grid barrier), sweep end (after its block reduction)
and barrier entry.  Prints, per step: barrier release skew, the sweep-time
distribution over blocks, the critical path, and the barrier latency.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

STEPS, MAXB = 16, 592


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="ramp")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--sigma", type=float, default=10.0)
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    clean, _ = fb.generate_cloud(a.kind, a.n, seed=0)
    noisy = fb.add_gaussian_noise(clean, a.sigma, seed=1)
    ctx = nat.context()
    dc = torch.from_numpy(np.array(noisy.coords)).cuda()
    dy = torch.from_numpy(np.array(noisy.colors)).cuda()
    do = torch.empty_like(dy)
    cfg = nat.make_config(fb.FilterConfig())
    for _ in range(a.frames):
        rep = nat.Report()
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, dc.data_ptr(), dy.data_ptr(), a.n,
                                       noisy.bit_depth, cfg, -1, float("nan"),
                                       do.data_ptr(), rep, nat.FLAG_DEVICE_PTRS), "denoise")
    torch.cuda.synchronize()
    print(f"S={rep.steps} lf_steps={rep.t_lf_steps*1e3:.3f} ms "
          f"({rep.t_lf_steps*1e6/max(rep.steps,1):.2f} us/step)")
    buf = np.zeros((STEPS, MAXB, 3), np.uint64)
    fn = ctx.lib.fgbd_debug_tlog
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p]
    assert fn(buf.ctypes.data) == 0
    nb = int(np.count_nonzero(buf[1, :, 0]))
    t = buf[:, :nb, :].astype(np.int64)
    t0 = t[:, :, 0].min()
    t = (t - t0) / 1e3  # us
    rows = []
    print(f"blocks={nb}")
    print("step  start_min start_skew  sweep_p10 sweep_p50 sweep_p90 sweep_max  "
          "crit_path  decide_max  barrier")
    for c in range(1, STEPS - 1):
        st, sw, br = t[c, :, 0], t[c, :, 1], t[c, :, 2]
        dur = sw - st
        nxt = t[c + 1, :, 0]
        r = dict(step=c, start_min=st.min(), start_skew=st.max() - st.min(),
                 sweep_p10=np.percentile(dur, 10), sweep_p50=np.percentile(dur, 50),
                 sweep_p90=np.percentile(dur, 90), sweep_max=dur.max(),
                 crit_path=sw.max() - st.min(), decide_max=(br - sw).max(),
                 barrier=nxt.min() - br.max(), step_total=nxt.min() - st.min())
        rows.append(r)
        print(f"{c:4d} {r['start_min']:9.2f} {r['start_skew']:9.2f}  {r['sweep_p10']:9.2f} "
              f"{r['sweep_p50']:9.2f} {r['sweep_p90']:9.2f} {r['sweep_max']:9.2f}  "
              f"{r['crit_path']:9.2f} {r['decide_max']:10.2f} {r['barrier']:8.2f}  "
              f"(step {r['step_total']:.2f})")
    # which blocks are slow: sweep time vs block index (SM placement)
    dur = (t[2:STEPS - 1, :, 1] - t[2:STEPS - 1, :, 0]).mean(axis=0)
    order = np.argsort(dur)
    print("fastest blocks:", [(int(b), round(float(dur[b]), 2)) for b in order[:6]])
    print("slowest blocks:", [(int(b), round(float(dur[b]), 2)) for b in order[-6:]])
    q = np.percentile(dur, [0, 25, 50, 75, 100])
    print("mean sweep per block quartiles (us):", np.round(q, 2).tolist())
    # intra-block spread: per-warp sweep end (lane 0 after its last row)
    wb = np.zeros((STEPS, MAXB, 16), np.uint64)
    fw = ctx.lib.fgbd_debug_wlog
    fw.restype = C.c_int
    fw.argtypes = [C.c_void_p]
    assert fw(wb.ctypes.data) == 0
    w = wb[2:STEPS - 1, :nb, :].astype(np.int64)
    nw = int(np.count_nonzero(w[0, 0]))
    w = w[:, :, :nw]
    st = buf[2:STEPS - 1, :nb, 0].astype(np.int64)[:, :, None]
    wdur = (w - st) / 1e3
    spread = wdur.max(axis=2) - wdur.min(axis=2)
    print(f"warps/block={nw}; per-warp sweep (us) p10/p50/p90 = "
          f"{np.percentile(wdur, 10):.2f} / {np.median(wdur):.2f} / {np.percentile(wdur, 90):.2f}; "
          f"intra-block spread (max - min warp) p50 {np.median(spread):.2f}, p90 "
          f"{np.percentile(spread, 90):.2f}; block mean-warp vs max-warp gap "
          f"{np.median(wdur.max(axis=2) - wdur.mean(axis=2)):.2f}")
    if a.json:
        Path(a.json).write_text(json.dumps({"rows": rows, "block_sweep_us": dur.round(3).tolist()},
                                           default=float))


if __name__ == "__main__":
    main()
