"""Host-side latency around one device-resident fgbd_denoise call (diagnostic):
wall time of the ctypes call vs the library's own first-to-last event time,
and the gap between the call's return and an event recorded right after it."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200 import _native as nat  # noqa: E402


def main():
    clean, _ = fb.generate_cloud("ramp", 1_000_000, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    n = noisy.n_points
    ctx = nat.context()
    stream = torch.cuda.ExternalStream(ctx.lib.fgbd_ctx_stream(ctx.handle))
    dev = torch.device("cuda", 0)
    d_coords = torch.from_numpy(np.array(noisy.coords)).to(dev)
    d_colors = torch.from_numpy(np.array(noisy.colors)).to(dev)
    d_out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    cfg = nat.make_config(fb.FilterConfig())
    torch.cuda.synchronize()
    rows = []
    with torch.cuda.stream(stream):
        for k in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t0 = time.perf_counter()
            rep = nat.Report()
            rc = ctx.lib.fgbd_denoise(ctx.handle, d_coords.data_ptr(), d_colors.data_ptr(), n,
                                      noisy.bit_depth, cfg, -1, float("nan"), d_out.data_ptr(),
                                      rep, nat.FLAG_DEVICE_PTRS)
            t1 = time.perf_counter()
            e1.record(stream)
            t2 = time.perf_counter()
            torch.cuda.synchronize()
            assert rc == 0
            rows.append((e0.elapsed_time(e1), 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * rep.t_total,
                         1e3 * rep.t_h2d, 1e3 * rep.t_d2h))
    for r in rows[3:]:
        print("event step %.3f ms | call wall %.3f ms | record %.3f ms | in-library %.3f ms "
              "(entry %.3f, tail %.3f)" % r)


if __name__ == "__main__":
    main()
