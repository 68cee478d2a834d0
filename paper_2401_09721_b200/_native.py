"""ctypes binding of the C ABI in include/fgbd_b200.h.

The shared library `_lib/libfgbd_b200.so` is built in-tree by `_build.py`
(`__graft_entry__.build()`).  There is no fallback: if the library or a GPU
is missing, every device entry point raises `DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (CloudError, DeviceError, FilterError, GraphError,
                     NoiseEstimationError)

LIB_PATH = Path(os.environ.get("FGBD_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "libfgbd_b200.so")

FGBD_OK, E_CLOUD, E_GRAPH, E_NOISE, E_FILTER, E_CUDA, E_NCCL, E_ARG = range(8)
FLAG_DEVICE_PTRS = 0x1
FLAG_WEIGHTS_F64 = 0x2
FLAG_NO_TIMING = 0x4
SLAB_EMULATED = 0x1
SLAB_FULL_OUTPUT = 0x2
SLAB_EXCHANGE = 0x4
FLAG_REUSE_GRAPH = 0x8
FLAG_STATIC_GEOMETRY = 0x10
FLAG_DEVICE_NE = 0x20
MAX_PATCH = 7
TRACE_MAX = 1025

_ERRORS = {E_CLOUD: CloudError, E_GRAPH: GraphError, E_NOISE: NoiseEstimationError,
           E_FILTER: FilterError, E_CUDA: DeviceError, E_NCCL: DeviceError, E_ARG: ValueError}

c_i32, c_i64, c_u32, c_f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_double
P = C.POINTER


class Config(C.Structure):
    _fields_ = [("q_max", c_i32), ("epsilon", c_f64), ("fslr_enabled", c_i32),
                ("patch_size", c_i32), ("reestimate_interval", c_i32),
                ("fslr_sigma_floor", c_f64), ("criterion_mode", c_i32),
                ("early_exit", c_i32), ("tau_divisor", c_i32)]


class Report(C.Structure):
    _fields_ = [("selected_q", c_i32), ("sigma_est", c_f64), ("masked_fraction", c_f64),
                ("criterion_value", c_f64), ("converged", c_i32), ("cached", c_i32),
                ("eligible_count", c_i64),
                ("t_graph_construction", c_f64), ("t_noise_estimation", c_f64),
                ("t_low_pass_filter", c_f64), ("t_total", c_f64),
                ("steps", c_i32), ("all_excluded_fallback", c_i32), ("n_edges", c_i64),
                ("nnz", c_i64), ("max_degree", c_i32), ("sigma_g", c_f64),
                ("included_count", c_i64), ("per_channel_sigma", c_f64 * 3),
                ("eigenvalues", (c_f64 * MAX_PATCH) * 3), ("tail_m", c_i32 * 3),
                ("tail_tau", c_f64 * 3), ("tail_fallback", c_i32 * 3), ("n_trace", c_i32),
                ("trace", c_f64 * TRACE_MAX), ("gpu_launches", c_i32),
                ("t_lf_steps", c_f64), ("t_h2d", c_f64), ("t_d2h", c_f64),
                ("graph_reused", c_i32), ("jacobi_direct_off", c_i32 * 3),
                ("t_slab_rank", (c_f64 * 4) * 16)]


class Noise(C.Structure):
    _fields_ = [("sigma_est", c_f64), ("per_channel_sigma", c_f64 * 3),
                ("eigenvalues", (c_f64 * MAX_PATCH) * 3),
                ("covariance", ((c_f64 * MAX_PATCH) * MAX_PATCH) * 3),
                ("m", c_i32 * 3), ("tau", c_f64 * 3), ("fallback", c_i32 * 3),
                ("eligible_count", c_i64), ("patch_size", c_i32),
                ("jacobi_direct_off", c_i32 * 3)]


class GraphInfo(C.Structure):
    _fields_ = [("n", c_i64), ("n_edges", c_i64), ("nnz", c_i64), ("max_degree", c_i32),
                ("sigma_g", c_f64)]


_SIGNATURES = {
    "fgbd_abi_version": (c_i32, []),
    "fgbd_last_error": (C.c_char_p, [C.c_void_p]),
    "fgbd_ctx_create": (C.c_void_p, [c_i32, c_i64]),
    "fgbd_ctx_destroy": (None, [C.c_void_p]),
    "fgbd_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "fgbd_ctx_device_bytes": (c_i64, [C.c_void_p]),
    "fgbd_denoise": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_i32, P(Config),
                             c_i32, c_f64, C.c_void_p, P(Report), c_u32]),
    "fgbd_radix_argsort": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_i32, C.c_void_p, c_u32]),
    "fgbd_scan_line": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_i32, c_i32, C.c_void_p,
                               C.c_void_p, c_u32]),
    "fgbd_build_graph": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_i32, P(GraphInfo), c_u32]),
    "fgbd_graph_export": (c_i32, [C.c_void_p] + [C.c_void_p] * 8),
    "fgbd_estimate_noise": (c_i32, [C.c_void_p, C.c_void_p, c_i32, c_i32, P(Noise),
                                    C.c_void_p, c_u32]),
    "fgbd_fslr_mask": (c_i32, [C.c_void_p, c_f64, c_f64, C.c_void_p, P(c_i32)]),
    "fgbd_filter_steps_csr": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, c_i64,
                                      c_i64, C.c_void_p, c_i32, C.c_void_p, c_u32]),
    "fgbd_apply_filter": (c_i32, [C.c_void_p, C.c_void_p, c_i32, C.c_void_p, c_u32]),
    "fgbd_select_q": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, c_f64, P(Config), P(c_i32),
                              C.c_void_p, P(Report), c_u32]),
    "fgbd_selection_criterion": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, c_i64,
                                         c_f64, c_i32, P(c_f64), c_u32]),
    "fgbd_extract_patches": (c_i32, [C.c_void_p, C.c_void_p, c_i32, C.c_void_p, C.c_void_p,
                                     P(c_i64), c_u32]),
    "fgbd_edge_weights": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_f64, P(c_f64), C.c_void_p,
                                  c_u32]),
    "fgbd_symmetric_eigenvalues": (c_i32, [C.c_void_p, c_i32, C.c_void_p, C.c_char_p, c_i32]),
    "fgbd_symmetric_eigenvalues_ex": (c_i32, [C.c_void_p, c_i32, C.c_void_p, C.c_void_p,
                                              C.c_char_p, c_i32]),
    "fgbd_select_tail": (c_i32, [C.c_void_p, c_i32, c_i32, P(c_i32), P(c_f64), P(c_i32),
                                 C.c_char_p, c_i32]),
    "fgbd_slab_create": (C.c_void_p, [C.c_void_p, c_i32, c_i32, c_i64, c_i64, c_u32]),
    "fgbd_slab_destroy": (None, [C.c_void_p, C.c_void_p]),
    "fgbd_slab_handle_size": (c_i32, []),
    "fgbd_slab_export": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fgbd_slab_import": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fgbd_denoise_slab": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  c_i64, C.c_void_p, c_i32, P(Config), c_i32, c_f64,
                                  C.c_void_p, P(Report), c_u32]),
    "fgbd_ply_decode": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_i32, P(c_i32), P(c_i32),
                                C.c_void_p, C.c_void_p, C.c_void_p, P(c_i32), c_u32]),
    "fgbd_ply_encode": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, c_i64,
                                C.c_void_p, c_u32]),
    "fgbd_denoise_ply": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_i32, P(c_i32), P(c_i32), c_i32,
                                 P(Config), c_i32, c_f64, C.c_void_p, P(Report), c_u32]),
    "fgbd_knn_build": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_i32, c_i32,
                               P(c_i64), c_u32]),
    "fgbd_knn_export": (c_i32, [C.c_void_p] + [C.c_void_p] * 6),
    "fgbd_quantize": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, c_i64, c_i32, C.c_void_p,
                              P(c_i32), c_u32]),
    "fgbd_sq_error_sum": (c_i32, [C.c_void_p, C.c_void_p, C.c_void_p, c_i64, P(c_f64), c_u32]),
    "fgbd_gaussian_noise": (c_i32, [C.c_void_p, C.c_void_p, c_i64, c_f64, C.c_void_p,
                                    C.c_void_p, C.c_void_p, c_u32]),
    "fgbd_host_alloc": (C.c_void_p, [c_i64]),
    "fgbd_host_free": (None, [C.c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None):
    """Load (once) and type the shared library; raise DeviceError if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"B200 library not built: {p} is missing (run __graft_entry__.build()); "
                "this package has no CPU fallback")
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Context:
    """One device context (stream + scratch) for the calling thread."""

    def __init__(self, device: int = 0, max_points: int = 0):
        self.lib = load_library()
        h = self.lib.fgbd_ctx_create(int(device), int(max_points))
        if not h:
            msg = self.lib.fgbd_last_error(None).decode()
            raise DeviceError(f"cannot create B200 context on device {device}: {msg}")
        self.handle = h
        self.device = int(device)
        self.graph_token = None  # id of the Graph whose device copy this context holds

    def check(self, rc: int, what: str = ""):
        if rc == FGBD_OK:
            return
        msg = self.lib.fgbd_last_error(self.handle).decode()
        raise _ERRORS.get(rc, DeviceError)(msg or f"{what} failed with status {rc}")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fgbd_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()
_default_device = [int(os.environ.get("FGBD_DEVICE", os.environ.get("LOCAL_RANK", "0")))]


def use_device(device: int):
    """Select the GPU used by subsequent calls from this thread."""
    _tls.device = int(device)


def context() -> Context:
    dev = getattr(_tls, "device", _default_device[0])
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(dev)
    if ctx is None:
        ctx = ctxs[dev] = Context(dev)
    return ctx


def make_config(cfg) -> Config:
    c = Config()
    c.q_max = int(cfg.q_max)
    c.epsilon = float("nan") if cfg.epsilon is None else float(cfg.epsilon)
    c.fslr_enabled = 1 if cfg.fslr_enabled else 0
    c.patch_size = int(cfg.patch_size)
    c.reestimate_interval = int(cfg.reestimate_interval)
    c.fslr_sigma_floor = float(cfg.fslr_sigma_floor)
    c.criterion_mode = {"pooled": 0, "per_channel": 1}[cfg.criterion_mode]
    c.early_exit = 1 if cfg.early_exit else 0
    c.tau_divisor = {"count": 0, "count_plus_one": 1}.get(cfg.tau_divisor, -1)
    return c


class _Lease:
    """Returns a pinned block to its pool when the last array view dies."""

    __slots__ = ("pool", "size", "ptr")

    def __init__(self, pool, size, ptr):
        self.pool, self.size, self.ptr = pool, size, ptr

    def __del__(self):
        try:
            self.pool._release(self.size, self.ptr)
        except Exception:
            pass


class PinnedPool:
    """Recycled page-locked host blocks for device->host results.

    `denoise` returns its colours in one of these blocks so the D2H copy runs
    at full PCIe rate; the block goes back to the pool when the returned
    array (and every view of it) is garbage-collected.  Past `max_blocks`
    outstanding blocks it falls back to ordinary pageable memory.  Block
    sizes are rounded up to 8 classes per octave (<= 12.5% slack) so frames
    of varying size share blocks, and at most `max_free_bytes` are kept idle.
    """

    def __init__(self, max_blocks: int = 16, max_free_bytes: int = 8 << 30):
        self.max_blocks = max_blocks
        self.max_free_bytes = max_free_bytes
        self.free: dict[int, list[int]] = {}
        self.free_bytes = 0
        self.outstanding = 0
        self.allocs = 0
        self.reuses = 0
        self.lock = threading.RLock()

    def empty(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = int(np.prod(shape))
        size = size_class(max(count * dtype.itemsize, 1))
        with self.lock:
            lst = self.free.get(size)
            ptr = lst.pop() if lst else None
            if ptr is not None:
                self.free_bytes -= size
            if ptr is None and self.outstanding >= self.max_blocks:
                return np.empty(shape, dtype)
            self.outstanding += 1
            if ptr is not None:
                self.reuses += 1
        if ptr is None:
            self.allocs += 1
            ptr = load_library().fgbd_host_alloc(size)
            if not ptr:
                with self.lock:
                    self.outstanding -= 1
                return np.empty(shape, dtype)
        buf = (C.c_char * size).from_address(ptr)
        buf._lease = _Lease(self, size, ptr)
        return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)

    def _release(self, size, ptr):
        with self.lock:
            self.outstanding -= 1
            if self.free_bytes + size <= self.max_free_bytes:
                self.free.setdefault(size, []).append(ptr)
                self.free_bytes += size
                return
        load_library().fgbd_host_free(ptr)


def size_class(size: int) -> int:
    """Round up to one of 8 sizes per power of two (4 KiB minimum)."""
    if size <= 4096:
        return 4096
    step = 1 << max(0, size.bit_length() - 4)
    return (size + step - 1) // step * step


_pool = PinnedPool(max_blocks=64)    # denoise outputs
_user_pool = PinnedPool(max_blocks=1 << 20)  # explicit pinned_empty() requests


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array backed by recycled page-locked host memory (for inputs)."""
    return _user_pool.empty(shape, dtype)


def pinned_output(shape, dtype) -> np.ndarray:
    """Output buffer for denoise results (bounded pool, recycled)."""
    return _pool.empty(shape, dtype)
