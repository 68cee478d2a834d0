"""H2D / D2H bandwidth from pinned memory with 1, 2 or 4 concurrent copies."""
import time

import torch

MB = 1 << 20
for size in (24 * MB, 48 * MB):
    h = torch.empty(size, dtype=torch.uint8).pin_memory()
    d = torch.empty(size, dtype=torch.uint8, device="cuda")
    for parts in (2, 1, 4, 1):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        chunk = size // parts
        for direction in ("h2d", "d2h"):
            best = 1e9
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for k, s in enumerate(streams):
                    with torch.cuda.stream(s):
                        if direction == "h2d":
                            d[k * chunk:(k + 1) * chunk].copy_(h[k * chunk:(k + 1) * chunk],
                                                                non_blocking=True)
                        else:
                            h[k * chunk:(k + 1) * chunk].copy_(d[k * chunk:(k + 1) * chunk],
                                                                non_blocking=True)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(f"{size // MB:3d} MB {direction} parts={parts}: {size / best / 1e9:6.1f} GB/s")
# both directions at once
h1 = torch.empty(48 * MB, dtype=torch.uint8).pin_memory()
h2 = torch.empty(24 * MB, dtype=torch.uint8).pin_memory()
d1 = torch.empty(48 * MB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(24 * MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
best = 1e9
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"48 MB h2d + 24 MB d2h concurrently: {best * 1e3:.3f} ms")
