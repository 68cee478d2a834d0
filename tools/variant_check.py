"""Bit-identity of two filter variants on one frame (experiment tool):
    python tools/variant_check.py --n 4000000 --a 0 --b 13"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4_000_000)
    ap.add_argument("--kind", default="ramp")
    ap.add_argument("--a", default="0")
    ap.add_argument("--b", default="13")
    a = ap.parse_args()
    import paper_2401_09721_b200 as fb

    clean, _ = fb.generate_cloud(a.kind, a.n, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    res = {}
    for v in (a.a, a.b):
        os.environ["FGBD_LF_VARIANT"] = v
        import subprocess
        code = (f"import sys, numpy as np; sys.path.insert(0, {str(Path(__file__).resolve().parent.parent)!r}); "
                "import paper_2401_09721_b200 as fb; "
                f"c,_=fb.generate_cloud({a.kind!r},{a.n},seed=0); y=fb.add_gaussian_noise(c,10.0,seed=1); "
                "o,r=fb.denoise(y); "
                f"np.save('/tmp/vc_{v}.npy', o.colors); "
                "print(r.selected_q, r.device['steps'], repr(r.sigma_est), r.masked_fraction, repr(r.criterion_value))")
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                             env=dict(os.environ, FGBD_LF_VARIANT=v))
        print(v, out.stdout.strip(), out.stderr.strip()[-300:])
        res[v] = np.load(f"/tmp/vc_{v}.npy")
    print("colours identical:", bool(np.array_equal(res[a.a], res[a.b])))


if __name__ == "__main__":
    main()
