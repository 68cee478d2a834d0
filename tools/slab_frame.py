"""ncu driver: one emulated slab frame (P ranks on this GPU) after a warm-up.

    python tools/slab_frame.py [--n 8000000] [--ranks 8] [--frames 2]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--frames", type=int, default=2)
    a = ap.parse_args()
    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200.slab import denoise_slab

    clean, _ = fb.generate_cloud("ramp", a.n, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    for f in range(a.frames):
        out, rep = denoise_slab(noisy, emulate_ranks=a.ranks)
        print(f"frame {f}: q={rep.selected_q} S={rep.device['steps']} "
              f"lf_steps={1e3 * rep.device['t_lf_steps']:.3f}ms total={1e3 * rep.device['t_total']:.3f}ms")


if __name__ == "__main__":
    main()
