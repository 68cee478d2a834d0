"""Frame-sequence driver: schedule properties and the multi-rank exchange.

The per-frame denoise is injected (the CPU oracle adapted to the package's
types) so the multi-process path runs here on CPU with the gloo backend,
world_size 2, exactly as it runs over NCCL with one process per B200.
"""

from __future__ import annotations

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2401_09721_b200 as fb
from oracle import fgbd_oracle as O
from paper_2401_09721_b200.sequence import denoise_sequence, group_heads, plan_sequence


def oracle_denoise(pc, cfg=fb.FilterConfig(), cached_q=None, cached_sigma_est=None):
    ocfg = O.OracleConfig(**{k: getattr(cfg, k) for k in O.OracleConfig.__dataclass_fields__})
    r = O.denoise(pc.coords, pc.colors, pc.bit_depth, ocfg, cached_q, cached_sigma_est)
    rep = fb.DenoiseReport(selected_q=r.selected_q, sigma_est=r.sigma_est,
                           masked_fraction=r.masked_fraction, cached=r.cached)
    return pc.with_colors(r.colors), rep


def make_frames(n_frames=7, n=1500):
    clean, _ = fb.generate_cloud("two-tone", n, seed=0)
    return [fb.add_gaussian_noise(clean, 15.0, seed=1 + f) for f in range(n_frames)]


def sequential_reference(frames, cfg):
    """The reference CLI loop (cli.py:123-136) on the oracle."""
    out, k = {}, cfg.reestimate_interval
    for g in range(0, len(frames), k):
        out[g] = oracle_denoise(frames[g], cfg)
        q, s = out[g][1].selected_q, out[g][1].sigma_est
        for f in range(g + 1, min(g + k, len(frames))):
            out[f] = oracle_denoise(frames[f], cfg, cached_q=q, cached_sigma_est=s)
    return out


@pytest.mark.parametrize("n,k,world", [(1, 10, 1), (7, 3, 2), (20, 10, 4), (300, 10, 8),
                                       (5, 1, 3), (9, 4, 16)])
def test_plan_covers_every_frame_once(n, k, world):
    p1, p2 = plan_sequence(n, k, world)
    heads = sorted(f for r in p1 for f in r)
    assert heads == group_heads(n, k)
    cached = sorted(p.frame for r in p2 for p in r)
    assert sorted(heads + cached) == list(range(n))
    for r in p2:
        for p in r:
            assert p.head == (p.frame // k) * k and p.head != p.frame
    sizes = [len(r) for r in p2]
    assert max(sizes) - min(sizes) <= 1


def test_single_process_matches_reference_loop():
    frames = make_frames()
    cfg = fb.FilterConfig(reestimate_interval=3)
    got = denoise_sequence(frames, cfg, denoise_fn=oracle_denoise, workers=2)
    ref = sequential_reference(frames, cfg)
    assert sorted(got) == sorted(ref)
    for f in ref:
        assert got[f][1].selected_q == ref[f][1].selected_q
        assert got[f][1].cached == ref[f][1].cached
        assert np.array_equal(got[f][0].colors, ref[f][0].colors)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    frames = make_frames()
    cfg = fb.FilterConfig(reestimate_interval=3)
    res = denoise_sequence(lambda i: frames[i], cfg, n_frames=len(frames),
                           process_group=dist.group.WORLD, denoise_fn=oracle_denoise, workers=1)
    with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as fh:
        pickle.dump({f: (pc.colors, rep.selected_q, rep.cached, rep.sigma_est)
                     for f, (pc, rep) in res.items()}, fh)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    frames = make_frames()
    cfg = fb.FilterConfig(reestimate_interval=3)
    ref = sequential_reference(frames, cfg)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        parts = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(2)]
    assert not set(parts[0]) & set(parts[1]), "a frame ran on both ranks"
    merged = {**parts[0], **parts[1]}
    assert sorted(merged) == list(range(len(frames)))
    for f, (colors, q, cached, sigma) in merged.items():
        assert q == ref[f][1].selected_q and cached == ref[f][1].cached
        assert sigma == ref[f][1].sigma_est
        assert np.array_equal(colors, ref[f][0].colors)


def _handle_worker(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_2401_09721_b200.slab import exchange_handles, slab_partition

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    got = exchange_handles(bytes([rank]) * 64, dist.group.WORLD)
    # every rank derives the same z-slab partition from the same frame
    clean, _ = fb.generate_cloud("ramp", 30_000, seed=0)
    g = np.array(clean.coords)[np.random.default_rng(3).permutation(30_000)]
    part = slab_partition(fb.PointCloud(g, np.zeros(g.shape), clean.bit_depth), world)
    own = part.own_index(rank)
    with open(os.path.join(outdir, f"h{rank}.pkl"), "wb") as fh:
        pickle.dump((got, part.counts.tolist(), part.zcut.tolist(), own), fh)
    dist.barrier()
    dist.destroy_process_group()


def test_slab_handle_exchange_gloo():
    """The slab mode's one host-side collective: every rank gets every rank's
    IPC handle in rank order, and all ranks agree on the row ranges."""
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_handle_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        res = [pickle.load(open(os.path.join(d, f"h{r}.pkl"), "rb")) for r in range(2)]
    for got, counts, zcut, _ in res:
        assert got == [bytes([0]) * 64, bytes([1]) * 64]
        assert counts == res[0][1] and zcut == res[0][2] and sum(counts) == 30_000
    own = np.concatenate([res[0][3], res[1][3]])
    assert np.array_equal(np.sort(own), np.arange(30_000))  # the ranks' points partition the frame
