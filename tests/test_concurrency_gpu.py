"""Several host threads (each with its own device context) denoising
different frames at once -- select-q heads, cached-q frames and graph reuse
mixed, two frame sizes -- give the same bytes as running them one by one.
Frames are ordered on the GPU by a per-device compute-done event and a
cached frame drops the device mutex at enqueue (FGBD_ASYNC_LOCK), so this
is the check that no frame reads or overwrites another frame's work."""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2401_09721_b200 as fb
from paper_2401_09721_b200.filtering import denoise_frame

pytestmark = pytest.mark.gpu


def _jobs():
    jobs = []
    for kind, n in (("ramp", 200_000), ("two-tone", 120_000)):
        clean, _ = fb.generate_cloud(kind, n, seed=0)
        for s in range(4):
            noisy = fb.add_gaussian_noise(clean, 10.0, seed=1 + s)
            jobs.append((noisy, None, s % 2 == 0))
            jobs.append((noisy, 7 + s, s % 2 == 1))  # cached q
    return jobs


def _run(job):
    pc, q, reuse = job
    if q is None:
        out, rep = denoise_frame(pc, reuse_graph=reuse)
    else:
        out, rep = denoise_frame(pc, cached_q=q, cached_sigma_est=10.0, reuse_graph=reuse)
    return np.array(out.colors), rep.selected_q, rep.sigma_est, rep.masked_fraction


def test_threads_match_sequential(gpu_ready):
    jobs = _jobs()
    seq = [_run(j) for j in jobs]
    for workers in (2, 4):
        with ThreadPoolExecutor(max_workers=workers) as ex:
            for rnd in range(2):
                order = np.random.default_rng(rnd).permutation(len(jobs))
                got = dict(zip(order.tolist(), ex.map(_run, [jobs[k] for k in order])))
                for k, ref in enumerate(seq):
                    out, q, s, m = got[k]
                    assert np.array_equal(out, ref[0]), (workers, rnd, k)
                    assert (q, s, m) == ref[1:], (workers, rnd, k)
