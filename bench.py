"""Benchmark: FGBD denoise of 1M-point frames on B200 (frames/s), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one `denoise` of one 1M-point synthetic frame (BASELINE.json
config 2: the paper's 30 fps case, `ramp` lattice k=100, b=7, Gaussian
colour noise sigma=10, default FilterConfig; q saturates at 64 so S = 64
filter steps, the heaviest LF load).

value      device-resident throughput: inputs already in HBM, the C-ABI call
           `fgbd_denoise(..., FGBD_FLAG_DEVICE_PTRS)`, CUDA events on the
           library's stream, L2 flushed (1 GiB write) between steps and
           excluded from the timed spans.  Whole job = N ranks x K frames /
           max over ranks of the summed step time (frame-parallel, weak).
e2e        the public API `paper_2401_09721_b200.denoise(PointCloud)` with
           inputs in pinned host memory: H2D of coords+colours and D2H of the
           denoised colours inside every timed step.
roofline   dominant kernel k_lf_run (the persistent random-walk step loop): SURVEY 8(d)
           algorithmic bytes per step (52.125 N + 8 nnz) / its mean event-timed
           duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle port (oracle/fgbd_oracle.py, numpy, the
           reference's algorithm) on one frame of the same workload, rank 0, N=1.
--impl reference  times that CPU port on all host cores (one process per
           frame), same metric/config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

KIND, N_POINTS, SIGMA = "ramp", 1_000_000, 10.0
METRIC = "frames/sec at 1M pts/frame (FGBD denoise, 1 frame = 1 step)"
# > 8x the 126 MB L2; the write also keeps the GPU busy while the host
# enters the next call, so host-side entry latency does not show as idle
# device time at the start of a step (the return path still does)
L2_FLUSH_BYTES = 1024 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); without torchrun, N > 1 re-launches this "
                         "script under torch.distributed.run (default: WORLD_SIZE or 1)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--kind", default=KIND)
    ap.add_argument("--points", "--n", dest="n", type=int, default=N_POINTS)
    ap.add_argument("--sigma", type=float, default=SIGMA)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="frame", choices=["frame", "video", "slab", "ply"],
                    help="frame: BASELINE configs[1] (default); video: configs[3]; "
                         "slab: configs[4] (one frame split over the GPUs)")
    ap.add_argument("--frames", type=int, default=300, help="video length (configs[3])")
    ap.add_argument("--slab-ranks", type=int, default=1,
                    help="slab workload at N=1: logical ranks emulated on the one GPU")
    ap.add_argument("--workers", type=int, default=None,
                    help="host threads per GPU (default: video 3, ply 2)")
    ap.add_argument("--static-geometry", action="store_true",
                    help="video: the caller vouches that frames share coordinates "
                         "(FGBD_FLAG_STATIC_GEOMETRY: colours-only uploads)")
    ap.add_argument("--no-reuse", action="store_true",
                    help="video/ply: rebuild the graph of every frame even when the geometry is static")
    return ap.parse_args()


# FGBD_BENCH_SHARED_GPU=1 is a harness check only: every rank runs on GPU 0
# and the ranks meet over gloo, so the N>1 code path (barriers, max over
# ranks, whole-job value) can be exercised on a one-GPU box.  The ranks'
# frames are independent, so no kernel waits on another rank.  Its numbers
# are not bench values (the ranks share one GPU).
SHARED_GPU = os.environ.get("FGBD_BENCH_SHARED_GPU") == "1"


def launch_plan(gpus, env, argv):
    """How to honour `--gpus`: ("run", world) when this process is (one rank
    of) the job, ("relaunch", cmd) when N > 1 ranks must be started first.

    The driver starts N > 1 under torchrun (WORLD_SIZE set); a plain
    `python bench.py --gpus N` starts the ranks itself, so the N it prints is
    the N that ran.  A mismatch between --gpus and WORLD_SIZE is an error.
    """
    ws = env.get("WORLD_SIZE")
    if ws is not None:
        world = int(ws)
        if gpus is not None and gpus != world:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}")
        return "run", world
    world = 1 if gpus is None else int(gpus)
    if world < 1:
        raise SystemExit(f"bench.py: --gpus must be >= 1, got {world}")
    if world == 1:
        return "run", 1
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()),
           # torchrun's parser takes "--n" for an abbreviation of its own options
           *[("--points" + a[3:]) if a == "--n" or a.startswith("--n=") else a for a in argv]]
    return "relaunch", cmd


def dist_env():
    local = int(os.environ.get("LOCAL_RANK", 0))
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            0 if SHARED_GPU else local)


def init_dist(local):
    import torch
    import torch.distributed as dist

    if SHARED_GPU:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def warmup_steps(args):
    """W >= 3 untimed warm-up steps, the same count in both arms."""
    return max(args.warmup, 3)


def make_frame(kind, n, sigma, seed):
    import paper_2401_09721_b200 as fb

    clean, _ = fb.generate_cloud(kind, n, seed=0)
    return clean, fb.add_gaussian_noise(clean, sigma, seed=seed)


def config_block(args, world):
    """Identical in both arms (the driver compares them key for key)."""
    c = {"workload": f"single {args.n:,}-point synthetic '{args.kind}' frame, sigma={args.sigma:g}, "
                     "default FilterConfig (BASELINE.json configs[1])",
         "n_points": args.n, "kind": args.kind, "sigma": args.sigma,
         "parallelism": f"frame-parallel x{world}" if world > 1 else "single GPU",
         "l2": "flushed between timed steps (1 GiB write, untimed)"}
    if SHARED_GPU:
        c["harness_check"] = "FGBD_BENCH_SHARED_GPU: all ranks on GPU 0 over gloo; not a bench value"
    return c


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    """NVML sampler (every 2 ms) of SM clock and throttle reasons.

    `timed` toggles whether samples count: only samples taken while the timed
    steps run are reported (nvidia-smi's 100 ms loop is too coarse for a
    ~20 ms timed region).  Falls back to nvidia-smi if NVML is unavailable.
    """

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.timed = False
        self.run = True
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _loop(self):
        nv = self.nv
        while self.run:
            if self.timed:
                try:
                    mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((mhz, rs))
                except Exception:
                    pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.run = False

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "NVML unavailable"}
        reasons = set()
        for _, rs in self.samples:
            for name, attr in self.REASONS.items():
                if rs & getattr(self.nv, attr):
                    reasons.add(name)
        sm = [m for m, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "NVML, 2 ms period, timed steps only"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args):
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    fb.use_device(local)
    if world > 1:
        import torch.distributed as dist

        init_dist(local)
    clean, noisy = make_frame(args.kind, args.n, args.sigma, seed=1 + rank)
    n = noisy.n_points
    ctx = nat.context()
    stream = torch.cuda.ExternalStream(ctx.lib.fgbd_ctx_stream(ctx.handle), device=local)
    dev = torch.device("cuda", local)
    d_coords = torch.from_numpy(np.array(noisy.coords)).to(dev)
    d_colors = torch.from_numpy(np.array(noisy.colors)).to(dev)
    d_out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    cfg = nat.make_config(fb.FilterConfig())
    torch.cuda.synchronize()

    def step_device():
        rep = nat.Report()
        ctx.check(ctx.lib.fgbd_denoise(ctx.handle, d_coords.data_ptr(), d_colors.data_ptr(), n,
                                       noisy.bit_depth, cfg, -1, float("nan"), d_out.data_ptr(),
                                       rep, nat.FLAG_DEVICE_PTRS), "denoise")
        return rep

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    clk = Clocks(local).__enter__()
    for _ in range(warmup_steps(args)):
        step_device()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    reps = []
    clk.timed = True
    # one stream context for the whole loop: entering it per step cost ~10 us
    # of host time between the frame's return and its end event
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(k)
            ev[k][0].record(stream)
            reps.append(step_device())
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    rep0 = reps[-1]
    S = int(rep0.steps)
    q = int(rep0.selected_q)
    nnz = int(rep0.nnz)
    # dominant kernel: the filter step, event-timed inside the library
    lf_s = float(np.mean([r.t_lf_steps for r in reps])) / max(S, 1)
    frame_bytes = 144.125 * n + 12.0 * nnz + S * (52.125 * n + 8.0 * nnz)
    lf_bytes = 52.125 * n + 8.0 * nnz
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    tf = ROOT / "profiles" / "lf_step_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
    launches = int(sum(r.gpu_launches for r in reps))
    stage = {"graph_construction_ms": 1e3 * float(np.mean([r.t_graph_construction for r in reps])),
             "noise_estimation_ms": 1e3 * float(np.mean([r.t_noise_estimation for r in reps])),
             "low_pass_filter_ms": 1e3 * float(np.mean([r.t_low_pass_filter for r in reps])),
             # the library's own events, first to last (the step also holds
             # the call's host entry / return around them)
             "in_library_ms": 1e3 * float(np.mean([r.t_total for r in reps]))}
    clk.timed = False
    clk.__exit__()
    clocks = clk.summary()

    # e2e: public API, pinned host inputs, H2D + D2H inside each step
    e2e = e2e_pageable = None
    if not args.no_e2e:
        pc_coords = nat.pinned_empty(noisy.coords.shape, np.int64)
        pc_coords[...] = noisy.coords
        pc_colors = nat.pinned_empty(noisy.colors.shape, np.float64)
        pc_colors[...] = noisy.colors
        pc = fb.PointCloud(pc_coords, pc_colors, noisy.bit_depth)
        assert pc.coords.ctypes.data == pc_coords.ctypes.data
        for _ in range(warmup_steps(args)):  # same shape as the timed loop: the
            out, rep = fb.denoise(pc)         # pinned output pool reaches steady state
        barrier()
        t_e2e, dev_t = [], []
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, rep = fb.denoise(pc)
            t_e2e.append(time.perf_counter() - t0)
            dev_t.append((rep.device["t_total"], rep.device["t_h2d"], rep.device["t_d2h"]))
        barrier()
        e2e_s = float(sum(t_e2e))
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": world * args.steps / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": int(pc.coords.nbytes + pc.colors.nbytes),
               "d2h_bytes_per_step": int(out.colors.nbytes),
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "step_ms_min_median_max": [1e3 * min(t_e2e), 1e3 * float(np.median(t_e2e)),
                                          1e3 * max(t_e2e)],
               "breakdown_ms": {"device_events_total": 1e3 * float(np.mean([d[0] for d in dev_t])),
                                "coords_h2d": 1e3 * float(np.mean([d[1] for d in dev_t])),
                                "colors_d2h": 1e3 * float(np.mean([d[2] for d in dev_t]))},
               "path": "paper_2401_09721_b200.denoise(PointCloud) -> fgbd_denoise C-ABI, pinned host inputs"}
        # the same with ordinary (pageable) NumPy inputs, as load_ply /
        # add_gaussian_noise hand them over
        pg_pc = fb.PointCloud(np.array(noisy.coords), np.array(noisy.colors), noisy.bit_depth)
        for _ in range(warmup_steps(args)):
            fb.denoise(pg_pc)
        barrier()
        t_pg = []
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, rep = fb.denoise(pg_pc)
            t_pg.append(time.perf_counter() - t0)
        barrier()
        pg_s = float(sum(t_pg))
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([pg_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pg_s = float(t.item())
        e2e_pageable = {"value": world * args.steps / pg_s, "unit": "frames/s",
                        "h2d_bytes_per_step": int(pg_pc.coords.nbytes + pg_pc.colors.nbytes),
                        "d2h_bytes_per_step": int(out.colors.nbytes),
                        "ms_per_step": 1e3 * pg_s / args.steps,
                        "path": "paper_2401_09721_b200.denoise(PointCloud) with pageable NumPy inputs"}


    # CPU baseline + parity spot check (rank 0, N = 1 only)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import fgbd_oracle as O

        # median of 3 runs of the frame, or of 1 when one run
        # already takes over 10 s, keeping the CPU sample to ~10-30 s
        runs = []
        while True:
            t0 = time.perf_counter()
            ref = O.denoise(noisy.coords, noisy.colors, noisy.bit_depth)
            runs.append(time.perf_counter() - t0)
            if len(runs) == 3 or runs[0] > 10.0:
                break
        t_cpu = float(np.median(runs))
        cpu = {"value": 1.0 / t_cpu, "unit": "frames/s", "cores": 1, "kind": "port",
               "sample": f"median of {len(runs)} run(s) of 1 frame of the same workload "
                         f"({n:,} pts, S={ref.steps}): {', '.join(f'{r:.2f}' for r in runs)} s, "
                         "single-threaded numpy/scipy oracle",
               "stage_s": {k: round(v, 4) for k, v in (ref.stage_timings or {}).items()},
               "host_cores_visible": len(os.sched_getaffinity(0)),
               "thread_env": {k: os.environ.get(k) for k in
                              ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "NUMBA_NUM_THREADS")}}
        out_d = d_out.cpu().numpy()
        parity = {"q_gpu": q, "q_ref": ref.selected_q, "S_gpu": S, "S_ref": ref.steps,
                  "sigma_est_rel": abs(rep0.sigma_est - ref.sigma_est) / ref.sigma_est,
                  "max_abs_color_diff": float(np.max(np.abs(out_d - ref.colors))),
                  "psnr_gpu": fb.psnr(clean, noisy.with_colors(out_d)),
                  "psnr_ref": fb.psnr(clean, noisy.with_colors(ref.colors))}
        parity["dpsnr_db"] = parity["psnr_gpu"] - parity["psnr_ref"]

    if rank == 0:
        ms = total_ms / args.steps
        line = {
            "metric": METRIC, "value": world * args.steps / (total_ms / 1e3), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": warmup_steps(args),
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, world),
            "frame": {"bit_depth": int(noisy.bit_depth), "selected_q": q, "filter_steps_S": S,
                      "n_edges": int(rep0.n_edges)},
            "mpoints_per_s": world * args.steps * n / (total_ms / 1e3) / 1e6,
            "stage_ms": stage,
            "roofline": {"bound": "hbm", "kernel": "k_lf_run",
                         "achieved": lf_bytes / lf_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": lf_bytes / lf_s / 1e9 / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": lf_bytes,
                         "launch_ms": lf_s * 1e3, "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                         if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"},
            # whole-frame algorithmic bytes: GC 88N+8nnz, NE 48N+4nnz,
            # FSLR 8.125N, S x (52.125N + 8nnz)
            "frame_roofline": {
                "bytes_per_frame": frame_bytes,
                "achieved": frame_bytes / (total_ms / args.steps / 1e3) / 1e9, "peak": peak,
                "unit": "GB/s",
                "frac": frame_bytes / (total_ms / args.steps / 1e3) / 1e9 / peak,
                "roofline_fps": peak * 1e9 / frame_bytes},
            "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "gpu_launches": launches, "clocks": clocks,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the CPU port on all host cores
# ---------------------------------------------------------------------------

def _ref_worker(a):
    kind, n, sigma, seed = a
    sys.path.insert(0, str(ROOT))
    from oracle import fgbd_oracle as O

    _, noisy = make_frame(kind, n, sigma, seed)
    t0 = time.perf_counter()
    res = O.denoise(noisy.coords, noisy.colors, noisy.bit_depth)
    return time.perf_counter() - t0, res.selected_q, res.steps


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30
    procs = max(1, min(cores, int(mem_gb // 3), 32))
    env_thr = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    warm = warmup_steps(args)
    walls, qs = [], set()
    with ctx.Pool(procs) as pool:
        for k in range(warm + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_ref_worker, [(args.kind, args.n, args.sigma, 1 + k * procs + i)
                                         for i in range(procs)])
            if k >= warm:
                walls.append(time.perf_counter() - t0)
                qs.update(r[1] for r in res)
    total = float(sum(walls))
    value = procs * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": warm, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(args, 1),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": procs, "kind": "port",
                         "sample": f"each step = {procs} frames denoised concurrently, one "
                                   f"single-threaded process per frame ({cores} cores visible, "
                                   f"thread env {env_thr})"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "selected_q": sorted(qs),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# video workload (BASELINE.json configs[3]): K-frame q reuse, frame-parallel
# ---------------------------------------------------------------------------

def run_video(args):
    if args.workers is None:
        args.workers = 3  # GPU-ordered frames: 3 host threads keep transfers and compute overlapped
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat
    from paper_2401_09721_b200.sequence import denoise_sequence

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    fb.use_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        init_dist(local)
        pg = dist.group.WORLD
    # a pool of distinct noisy frames in pinned memory, cycled over the video
    clean, _ = fb.generate_cloud(args.kind, args.n, seed=0)
    pool = []
    c = nat.pinned_empty(clean.coords.shape, np.int64)  # one capture geometry
    c[...] = clean.coords
    for s in range(8):
        noisy = fb.add_gaussian_noise(clean, args.sigma, seed=1 + s)
        y = nat.pinned_empty(noisy.colors.shape, np.float64)
        y[...] = noisy.colors
        pool.append(fb.PointCloud(c, y, noisy.bit_depth))
    cfg = fb.FilterConfig()
    load = lambda i: pool[i % len(pool)]
    checksum = [0.0]

    compute = []

    def sink(i, pc, rep):  # consume the frame (as a writer would) and release it
        checksum[0] += float(pc.colors[i % pc.n_points, 0])
        compute.append(sum(rep.stage_timings.values()))

    # warm-up: contexts for every worker thread, pinned output pool
    kw = dict(reuse_graph=not args.no_reuse, static_geometry=args.static_geometry)
    denoise_sequence(load, cfg, n_frames=min(2 * cfg.reestimate_interval, args.frames),
                     workers=args.workers, process_group=pg, sink=sink, **kw)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    compute.clear()
    t0 = time.perf_counter()
    res = denoise_sequence(load, cfg, n_frames=args.frames, workers=args.workers,
                           process_group=pg, sink=sink, **kw)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        heads = sum(1 for r in res.values() if not r[1].cached)
        coords_b, colors_b = int(pool[0].coords.nbytes), int(pool[0].colors.nbytes)
        h2d = colors_b + (0 if args.static_geometry else coords_b)
        print(json.dumps({
            "e2e": {"h2d_bytes_per_step": h2d, "d2h_bytes_per_step": colors_b,
                    "host_link_bytes_per_frame": h2d + colors_b,
                    "note": "static geometry: coordinates go up once per worker"
                            if args.static_geometry else "coordinates re-sent and compared on device"},
            "metric": f"frames/sec, {args.frames}-frame video at {args.n:,} pts/frame "
                      f"(K={cfg.reestimate_interval} q reuse, e2e from pinned host frames)",
            "value": args.frames / wall, "unit": "frames/s", "n_gpus": world,
            "wall_s": wall, "higher_is_better": True, "scaling": "strong", "dtype": "f64",
            "data": "synthetic", "workers_per_gpu": args.workers,
            "device_compute_ms_sum_per_frame": 1e3 * float(np.sum(compute)) / args.frames,
            "config": {"workload": "BASELINE.json configs[3]", "kind": args.kind,
                       "n_points": args.n, "sigma": args.sigma, "frames": args.frames,
                       "rank0_heads": heads, "rank0_frames": len(res),
                       "rank0_graph_reused": sum(1 for r in res.values()
                                                 if r[1].device and r[1].device.get("graph_reused")),
                       "geometry": "static (frames share the clean cloud's coordinates)",
                       "static_geometry_flag": bool(args.static_geometry)},
        }), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# ply workload: the CLI's directory-of-PLY-frames loop,
# PLY file bytes in -> denoised PLY file bytes out, K-frame q reuse
# ---------------------------------------------------------------------------

def run_ply(args):
    if args.workers is None:
        args.workers = 2  # host-side PLY framing: a third thread costs more than it overlaps
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat
    from paper_2401_09721_b200.ply import denoise_ply, save_ply
    from paper_2401_09721_b200.sequence import denoise_sequence

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    fb.use_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        init_dist(local)
        pg = dist.group.WORLD
    # distinct noisy frames serialised as binary PLY files held in pinned memory
    clean, _ = fb.generate_cloud(args.kind, args.n, seed=0)
    files = []
    for s in range(8):
        b = save_ply(fb.add_gaussian_noise(clean, args.sigma, seed=1 + s))
        f = nat.pinned_empty((len(b),), np.uint8)
        f[...] = np.frombuffer(b, np.uint8)
        files.append(f)
    cfg = fb.FilterConfig()
    load = lambda i: files[i % len(files)]
    fn = lambda src, cfg, cached_q=None, cached_sigma_est=None: denoise_ply(
        src, cfg, cached_q, cached_sigma_est, copy=False, reuse_graph=not args.no_reuse)
    checksum = [0]

    compute = []

    def sink(i, out, rep):  # consume the output file bytes and release them
        checksum[0] += int(out[-1])
        compute.append(sum(rep.stage_timings.values()))

    denoise_sequence(load, cfg, n_frames=min(2 * cfg.reestimate_interval, args.frames),
                     workers=args.workers, process_group=pg, denoise_fn=fn, sink=sink)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    compute.clear()
    t0 = time.perf_counter()
    res = denoise_sequence(load, cfg, n_frames=args.frames, workers=args.workers,
                           process_group=pg, denoise_fn=fn, sink=sink)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    if rank == 0:
        heads = sum(1 for r in res.values() if not r[1].cached)
        print(json.dumps({
            "metric": f"frames/sec, {args.frames}-frame PLY sequence at {args.n:,} pts/frame "
                      f"(binary PLY bytes in -> PLY bytes out, K={cfg.reestimate_interval})",
            "value": args.frames / wall, "unit": "frames/s", "n_gpus": world,
            "wall_s": wall, "higher_is_better": True, "scaling": "strong", "dtype": "f64",
            "data": "synthetic", "workers_per_gpu": args.workers,
            "device_compute_ms_sum_per_frame": 1e3 * float(np.sum(compute)) / args.frames,
            "e2e": {"h2d_bytes_per_step": int(files[0].size),
                    "d2h_bytes_per_step": int(files[0].size)},
            "config": {"workload": "SURVEY 8(f) rank 2: PLY frame sequence", "kind": args.kind,
                       "n_points": args.n, "sigma": args.sigma, "frames": args.frames,
                       "rank0_heads": heads, "rank0_frames": len(res),
                       "rank0_graph_reused": sum(1 for r in res.values()
                                                 if r[1].device and r[1].device.get("graph_reused")),
                       "geometry": "static (frames share the clean cloud's coordinates)"},
        }), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# slab workload (BASELINE.json configs[4]): one big frame over N GPUs
# ---------------------------------------------------------------------------

def run_slab(args):
    """configs[4]: one 8M-point frame cut into z-slabs over the GPUs.  Each
    rank uploads, builds, estimates, filters and downloads only its slab
    (output="local"); N = 1 runs `--slab-ranks` emulated ranks on one GPU."""
    import torch

    import paper_2401_09721_b200 as fb
    from paper_2401_09721_b200 import _native as nat
    from paper_2401_09721_b200.slab import denoise_slab, slab_partition

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    fb.use_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        init_dist(local)
        pg = dist.group.WORLD
    n = args.n if args.n != N_POINTS else 8_000_000
    clean, _ = fb.generate_cloud(args.kind, n, seed=0)
    noisy = fb.add_gaussian_noise(clean, args.sigma, seed=1)
    c = nat.pinned_empty(noisy.coords.shape, np.int64)
    c[...] = noisy.coords
    y = nat.pinned_empty(noisy.colors.shape, np.float64)
    y[...] = noisy.colors
    pc = fb.PointCloud(c, y, noisy.bit_depth)
    ranks = world if world > 1 else max(1, args.slab_ranks)
    part = slab_partition(pc, ranks)

    def step():
        if pg is not None:
            idx, col, rep = denoise_slab(pc, process_group=pg, output="local", partition=part)
            return rep
        return denoise_slab(pc, emulate_ranks=ranks, partition=part)[1]

    for _ in range(warmup_steps(args)):
        rep = step()
    walls, devs, stages, per_rank = [], [], [], []
    for _ in range(args.steps):
        if pg is not None:
            import torch.distributed as dist

            dist.barrier()
        t0 = time.perf_counter()
        rep = step()
        walls.append(time.perf_counter() - t0)
        devs.append(rep.device["t_total"])
        stages.append((rep.device["t_h2d"], rep.stage_timings["graph_construction"],
                       rep.stage_timings["noise_estimation"], rep.device["t_lf_steps"],
                       rep.device["t_d2h"]))
        per_rank.append(rep.device["slab_rank_seconds"])
    wall = float(np.sum(walls))
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    st = np.mean(np.array(stages), axis=0) * 1e3
    pr = np.mean(np.array(per_rank), axis=0) * 1e3  # [rank][phase] ms
    if rank == 0:
        print(json.dumps({
            "metric": f"frames/sec, one {n:,}-point frame slab-partitioned over the GPUs",
            "value": args.steps / wall, "unit": "frames/s", "n_gpus": world,
            "ms_per_step": 1e3 * wall / args.steps, "steps": args.steps,
            "higher_is_better": True, "scaling": "strong", "dtype": "f64", "data": "synthetic",
            "device_ms_rank0": 1e3 * float(np.mean(devs)),
            "stage_ms": {"h2d": st[0], "graph_construction": st[1],
                         "noise_estimation_and_mask": st[2], "lf_steps": st[3], "d2h": st[4]},
            # per slab rank (device events around that rank's own work):
            # upload + own sort + block lists, cross-slab rows, NE + FSLR, output
            "per_rank_ms": {"upload_sort_blocks": pr[:, 0].tolist(),
                            "cross_slab_rows": pr[:, 1].tolist(),
                            "ne_fslr": pr[:, 2].tolist(), "output_d2h": pr[:, 3].tolist(),
                            "max_rank_gc_ne_h2d": float(np.max(pr[:, 0] + pr[:, 1] + pr[:, 2]))},
            "config": {"workload": "BASELINE.json configs[4]", "kind": args.kind, "n_points": n,
                       "sigma": args.sigma, "selected_q": rep.selected_q,
                       "filter_steps_S": rep.device["steps"], "slab_ranks": ranks,
                       "emulated": world == 1, "points_per_rank": part.counts.tolist()},
        }), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    what, plan = launch_plan(args.gpus, os.environ, sys.argv[1:])
    if what == "relaunch":
        sys.exit(subprocess.call(plan))
    args.gpus = plan
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "video":
        run_video(args)
    elif args.workload == "slab":
        run_slab(args)
    elif args.workload == "ply":
        run_ply(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
