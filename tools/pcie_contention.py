"""PCIe copy bandwidth alone and while the filter kernel runs (experiment).

Thread A (optional) loops device-resident cached-q frames (FLAG_DEVICE_PTRS:
no transfers of its own); thread B times 48 MB pinned H2D and 24 MB D2H
copies on its own stream."""
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200 import _native as nat  # noqa: E402

N = 1_000_000
clean, _ = fb.generate_cloud("ramp", N, seed=0)
noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
dc = torch.from_numpy(np.array(noisy.coords)).cuda()
dy = torch.from_numpy(np.array(noisy.colors)).cuda()
do = torch.empty_like(dy)
cfg = nat.make_config(fb.FilterConfig())
stop = threading.Event()


def busy():
    ctx = nat.context()
    rep = nat.Report()
    n = 0
    while not stop.is_set():
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, dc.data_ptr(), dy.data_ptr(), N, noisy.bit_depth,
                                       cfg, 64, float("nan"), do.data_ptr(), rep,
                                       nat.FLAG_DEVICE_PTRS | nat.FLAG_REUSE_GRAPH), "denoise")
        n += 1
    busy.frames = n


def copies(tag):
    h_in = torch.empty(48_000_000 // 8, dtype=torch.float64).pin_memory()
    h_out = torch.empty(24_000_000 // 8, dtype=torch.float64).pin_memory()
    d_in = torch.empty_like(h_in, device="cuda")
    d_out = torch.empty_like(h_out, device="cuda")
    s = torch.cuda.Stream()
    for kind in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for _ in range(20):
                if kind in ("h2d", "both"):
                    d_in.copy_(h_in, non_blocking=True)
                if kind in ("d2h", "both"):
                    h_out.copy_(d_out, non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t0
        mb = 20 * ((48 if kind != "d2h" else 0) + (24 if kind != "h2d" else 0))
        print(f"{tag:10s} {kind:5s} {mb / dt / 1e3:6.1f} GB/s", flush=True)


copies("alone")
t = threading.Thread(target=busy)
t.start()
time.sleep(0.5)
t0 = time.perf_counter()
copies("with-LF")
stop.set()
t.join()
