import sys, os
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np
import paper_2401_09721_b200 as fb
for kind in ('ramp', 'two-tone', 'constant'):
    clean, _ = fb.generate_cloud(kind, 1_000_000, seed=0)
    noisy = fb.add_gaussian_noise(clean, 10.0, seed=1)
    out, rep = fb.denoise(noisy)
    tr = rep.device.get('trace') if isinstance(rep.device, dict) else None
    print(kind, rep.selected_q, rep.device.get('steps'), None if tr is None else np.round(np.array(tr), 6).tolist())
