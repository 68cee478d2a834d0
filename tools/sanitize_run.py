"""Small end-to-end workload touching every device entry point: a select
frame, a cached frame and a reused-graph frame per cloud kind, PLY, kNN,
psnr and the device noise generator, on small clouds.  Written for
compute-sanitizer, which this GPU pool does not allow, so it runs plain."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb  # noqa: E402
from paper_2401_09721_b200.filtering import denoise_frame  # noqa: E402
from paper_2401_09721_b200.ply import denoise_ply, save_ply  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for kind in ("ramp", "two-tone", "constant"):
    clean, _ = fb.generate_cloud(kind, n, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    out, rep = fb.denoise(noisy)
    out2, rep2 = fb.denoise(noisy, cached_q=rep.selected_q, cached_sigma_est=rep.sigma_est)
    a = denoise_frame(noisy, reuse_graph=True)
    b = denoise_frame(noisy, reuse_graph=True)
    assert np.array_equal(a[0].colors, b[0].colors)
    print(kind, rep.selected_q, rep.device["steps"], b[1].device["graph_reused"])
src = save_ply(noisy)
denoise_ply(src)
g = fb.build_knn_brute(noisy, 6)
fb.psnr(clean, out)
dev = fb.add_gaussian_noise(clean, 10.0, seed=3, device=True)
assert np.array_equal(dev.colors, fb.add_gaussian_noise(clean, 10.0, seed=3).colors)
print("ok")
