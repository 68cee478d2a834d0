"""Does point order matter?  Same random cloud, original vs raster (line-1) order."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2401_09721_b200 as fb
clean, _ = fb.generate_cloud("constant", 1_000_000, seed=0)
noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
g = noisy.coords
order = np.lexsort((g[:, 0], g[:, 1], g[:, 2]))  # z-major raster = line-1 order
sorted_pc = fb.PointCloud(g[order], noisy.colors[order], noisy.bit_depth)
for name, pc in (("original", noisy), ("raster", sorted_pc)):
    for _ in range(3):
        out, rep = fb.denoise(pc)
    d = rep.device
    print(f"{name:9s} q={rep.selected_q} S={d['steps']} GC={rep.stage_timings['graph_construction']*1e3:.3f} "
          f"NE={rep.stage_timings['noise_estimation']*1e3:.3f} LF={rep.stage_timings['low_pass_filter']*1e3:.3f} "
          f"per-step={d['t_lf_steps']/max(d['steps'],1)*1e6:.1f}us")
