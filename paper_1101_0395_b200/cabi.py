"""ctypes binding of libcqg.so (include/cqg.h).

This is the only way the Python side reaches the device: every call goes
through the C-ABI entry points declared in include/cqg.h. There is no CPU
fallback -- if the library is missing or no sm_100 device is present the
calls raise.

Array arguments may be numpy arrays (host memory) or CUDA tensors exposing
``data_ptr()`` (device memory, e.g. torch); the library detects which.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CQG_LIB") or os.path.join(PKG, "libcqg.so")  # CQG_LIB: experiment builds

CQG_OK = 0
CQG_E_INVALID = 1
CQG_E_RUNTIME = 2
CQG_E_CUDA = 3
CQG_E_NOMEM = 4

INIT_MAXIMIN = 0
INIT_KMEANSPP = 1
INIT_GIVEN = 2

# Every symbol include/cqg.h declares (checked by tests/test_cabi_symbols.py).
EXPORTS = (
    "cqg_create", "cqg_destroy", "cqg_last_error", "cqg_set_stream", "cqg_set_sm_budget", "cqg_launch_count",
    "cqg_version", "cqg_histogram", "cqg_init_maximin", "cqg_init_kmeanspp", "cqg_lloyd",
    "cqg_map", "cqg_coarse_histogram", "cqg_coarse_histogram_weighted", "cqg_quantize", "cqg_set_profiling",
    "cqg_read_profile", "cqg_bench_sweep",
    "cqg_shard_begin", "cqg_shard_assign", "cqg_shard_moments", "cqg_shard_finalize", "cqg_shard_sizes",
    "cqg_shard_donor", "cqg_shard_move", "cqg_shard_end", "cqg_shard_finalize_async", "cqg_shard_status",
    "cqg_lloyd_exact", "cqg_compute_sse", "cqg_repair_empty_clusters", "cqg_center_table",
    "cqg_kmeanspp_next_masses", "cqg_maximin_pad",
)

PROF_SWEEP, PROF_MAPSWEEP, PROF_HIST, PROF_PIXEL, PROF_INIT, PROF_REPLAY, PROF_NDC, PROF_LLOYD, PROF_MAPNDC = range(9)
PROF_N = 9


class Term(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("max_iterations", C.c_int),
                ("fixed_iterations", C.c_int), ("record_history", C.c_int)]


class LloydStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("repair_count", C.c_int), ("ndc_total", C.c_uint64),
                ("n_points", C.c_uint64), ("flagged_total", C.c_uint64),
                ("swept_total", C.c_uint64)]


class QuantizeCfg(C.Structure):
    _fields_ = [("init_kind", C.c_int), ("k", C.c_int), ("seed", C.c_uint64), ("term", Term),
                ("index_bytes", C.c_int), ("sampling", C.c_int), ("width", C.c_int), ("height", C.c_int)]


class QuantizeStats(C.Structure):
    _fields_ = [("n_unique", C.c_uint64), ("lloyd", LloydStats), ("mean_sq_dist", C.c_double),
                ("map_ndc", C.c_uint64), ("ms_histogram", C.c_double), ("ms_init", C.c_double), ("ms_lloyd", C.c_double),
                ("ms_map", C.c_double)]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * PROF_N), ("units", C.c_double * PROF_N), ("launches", C.c_uint64 * PROF_N)]


class CqgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(CqgError, ValueError):
    """The reference's std::invalid_argument."""


_lib = None
_lib_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libcqg.so (raises if it has not been built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(path)
        vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
        L.cqg_create.restype = vp
        L.cqg_create.argtypes = [i32]
        L.cqg_destroy.argtypes = [vp]
        L.cqg_last_error.restype = C.c_char_p
        L.cqg_set_stream.argtypes = [vp, vp]
        L.cqg_set_sm_budget.argtypes = [vp, i32]
        L.cqg_set_sm_budget.restype = i32
        L.cqg_coarse_histogram.argtypes = [vp, vp, u64, vp, vp, vp, vp, vp]
        L.cqg_coarse_histogram.restype = i32
        L.cqg_coarse_histogram_weighted.argtypes = [vp, vp, vp, u64, vp, vp, vp, vp, vp]
        L.cqg_coarse_histogram_weighted.restype = i32
        L.cqg_launch_count.restype = u64
        L.cqg_launch_count.argtypes = [vp]
        L.cqg_version.restype = C.c_char_p
        L.cqg_histogram.argtypes = [vp, vp, u64, vp, vp, vp, C.POINTER(u64)]
        L.cqg_init_maximin.argtypes = [vp, vp, vp, u64, u64, i32, u64, i32, vp]
        L.cqg_init_kmeanspp.argtypes = [vp, vp, vp, u64, u64, i32, u64, vp]
        L.cqg_lloyd.argtypes = [vp, vp, vp, u64, u64, vp, i32, C.POINTER(Term), vp, vp, vp,
                                C.POINTER(LloydStats), vp, vp]
        L.cqg_map.argtypes = [vp, vp, u64, vp, i32, vp, i32, vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.cqg_quantize.argtypes = [vp, vp, u64, C.POINTER(QuantizeCfg), vp, vp, vp, vp, vp, vp,
                                   C.POINTER(QuantizeStats)]
        L.cqg_set_profiling.argtypes = [vp, i32]
        L.cqg_read_profile.argtypes = [vp, C.POINTER(Profile), i32]
        L.cqg_bench_sweep.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.cqg_bench_sweep.restype = i32
        L.cqg_shard_begin.argtypes = [vp, vp, vp, u64, u64, vp, i32, C.POINTER(Term)]
        L.cqg_shard_assign.argtypes = [vp, vp]
        L.cqg_shard_moments.argtypes = [vp, vp]
        L.cqg_shard_finalize.argtypes = [vp, vp, C.POINTER(i32), C.POINTER(C.c_double)]
        L.cqg_shard_sizes.argtypes = [vp, vp]
        L.cqg_shard_finalize_async.argtypes = [vp, vp]
        L.cqg_shard_finalize_async.restype = i32
        L.cqg_shard_status.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        L.cqg_shard_status.restype = i32
        L.cqg_shard_donor.argtypes = [vp, vp, i32, C.POINTER(C.c_double), C.POINTER(u64),
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.cqg_shard_move.argtypes = [vp, u64, i32, C.c_uint32]
        L.cqg_shard_end.argtypes = [vp, vp, vp, vp, C.POINTER(i32)]
        L.cqg_lloyd_exact.argtypes = [vp, vp, vp, u64, vp, i32, C.POINTER(Term), vp, vp, vp,
                                      C.POINTER(LloydStats), vp, vp]
        L.cqg_compute_sse.argtypes = [vp, vp, vp, u64, vp, i32, vp, C.POINTER(C.c_double)]
        L.cqg_repair_empty_clusters.argtypes = [vp, vp, vp, u64, vp, i32, vp, C.POINTER(i32)]
        L.cqg_center_table.argtypes = [vp, vp, i32, vp, vp]
        L.cqg_kmeanspp_next_masses.argtypes = [vp, vp, vp, u64, vp, i32, vp]
        L.cqg_maximin_pad.argtypes = [vp, vp, u64, vp, i32, i32, vp]
        for name in ("cqg_lloyd_exact", "cqg_compute_sse", "cqg_repair_empty_clusters", "cqg_center_table",
                     "cqg_kmeanspp_next_masses", "cqg_maximin_pad"):
            getattr(L, name).restype = i32
        for name in ("cqg_shard_begin", "cqg_shard_assign", "cqg_shard_moments", "cqg_shard_finalize",
                     "cqg_shard_sizes", "cqg_shard_donor", "cqg_shard_move", "cqg_shard_end"):
            getattr(L, name).restype = i32
        for name in ("cqg_set_profiling", "cqg_read_profile", "cqg_histogram", "cqg_init_maximin", "cqg_init_kmeanspp", "cqg_lloyd",
                     "cqg_map", "cqg_quantize", "cqg_set_stream"):
            getattr(L, name).restype = i32
        _lib = L
        return L


def check(rc: int) -> None:
    if rc == CQG_OK:
        return
    msg = load().cqg_last_error().decode()
    if rc == CQG_E_INVALID:
        raise InvalidArgument(rc, msg)
    raise CqgError(rc, msg)


def ptr(x) -> int | None:
    """Raw address of a numpy array or a CUDA tensor (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)!r}")


class Context:
    """One device context (cqg_ctx): owns a CUDA stream and device buffers."""

    def __init__(self, device: int = 0):
        self.L = load()
        h = self.L.cqg_create(device)
        if not h:
            raise CqgError(CQG_E_CUDA, self.L.cqg_last_error().decode())
        self.h = C.c_void_p(h)
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.cqg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def launches(self) -> int:
        return int(self.L.cqg_launch_count(self.h))

    def set_profiling(self, on: bool):
        check(self.L.cqg_set_profiling(self.h, 1 if on else 0))

    def read_profile(self, reset: bool = True) -> Profile:
        p = Profile()
        check(self.L.cqg_read_profile(self.h, C.byref(p), 1 if reset else 0))
        return p

    def bench_sweep(self, reps: int = 20):
        """(ms per launch, units per launch) of back-to-back WALK sweeps on the
        context's last Lloyd state (cqg_bench_sweep)."""
        ms, units = C.c_double(0), C.c_double(0)
        check(self.L.cqg_bench_sweep(self.h, reps, C.byref(ms), C.byref(units)))
        return ms.value, units.value

    def coarse_histogram_raw(self, rgb, P, out):
        """cqg_coarse_histogram into out (5 x 32768 int64: count, sum_r, sum_g, sum_b, sum_sq)."""
        check(self.L.cqg_coarse_histogram(self.h, ptr(rgb), P, ptr(out[0]), ptr(out[1]), ptr(out[2]),
                                          ptr(out[3]), ptr(out[4])))

    def coarse_histogram_weighted_raw(self, colors, counts, n, out):
        check(self.L.cqg_coarse_histogram_weighted(self.h, ptr(colors), ptr(counts), n, ptr(out[0]), ptr(out[1]),
                                                   ptr(out[2]), ptr(out[3]), ptr(out[4])))

    def set_sm_budget(self, sms: int):
        """Restrict this context's grids to `sms` SMs (0: the whole device), so
        several contexts can run their cooperative kernels side by side."""
        check(self.L.cqg_set_sm_budget(self.h, int(sms)))

    def set_stream(self, stream_ptr: int | None):
        check(self.L.cqg_set_stream(self.h, stream_ptr))

    # raw C-ABI calls (buffers already allocated by the caller) -----------------
    def histogram_raw(self, rgb, P, colors, counts, first=None) -> int:
        n = C.c_uint64(0)
        check(self.L.cqg_histogram(self.h, ptr(rgb), P, ptr(colors), ptr(counts), ptr(first),
                                   C.byref(n)))
        return n.value

    def init_raw(self, kind, colors, counts, n, P, k, seed, centers, weighted_first=True):
        if kind == INIT_MAXIMIN:
            check(self.L.cqg_init_maximin(self.h, ptr(colors), ptr(counts), n, P, k, seed,
                                          1 if weighted_first else 0, ptr(centers)))
        else:
            check(self.L.cqg_init_kmeanspp(self.h, ptr(colors), ptr(counts), n, P, k, seed,
                                           ptr(centers)))

    def lloyd_raw(self, colors, counts, n, P, init, k, term: Term, centers, labels, sse,
                  hist_labels=None, hist_centers=None) -> LloydStats:
        st = LloydStats()
        check(self.L.cqg_lloyd(self.h, ptr(colors), ptr(counts), n, P, ptr(init), k,
                               C.byref(term), ptr(centers), ptr(labels), ptr(sse), C.byref(st),
                               ptr(hist_labels), ptr(hist_centers)))
        return st

    def lloyd_exact_raw(self, points, weights, n, init, k, term: Term, centers, labels, sse,
                        hist_labels=None, hist_centers=None) -> LloydStats:
        """cqg_lloyd_exact: wsm for arbitrary weights, kmeans_full when weights is None."""
        st = LloydStats()
        check(self.L.cqg_lloyd_exact(self.h, ptr(points), ptr(weights), n, ptr(init), k, C.byref(term),
                                     ptr(centers), ptr(labels), ptr(sse), C.byref(st), ptr(hist_labels),
                                     ptr(hist_centers)))
        return st

    def compute_sse_raw(self, points, weights, n, centers, k, labels) -> float:
        out = C.c_double(0)
        check(self.L.cqg_compute_sse(self.h, ptr(points), ptr(weights), n, ptr(centers), k, ptr(labels),
                                     C.byref(out)))
        return out.value

    def repair_raw(self, points, weights, n, centers, k, labels) -> int:
        r = C.c_int(0)
        check(self.L.cqg_repair_empty_clusters(self.h, ptr(points), ptr(weights), n, ptr(centers), k,
                                               ptr(labels), C.byref(r)))
        return r.value

    def center_table_raw(self, centers, k, dist, order):
        check(self.L.cqg_center_table(self.h, ptr(centers), k, ptr(dist), ptr(order)))

    def next_masses_raw(self, colors, weights, n, centers, k, masses):
        check(self.L.cqg_kmeanspp_next_masses(self.h, ptr(colors), ptr(weights), n, ptr(centers), k, ptr(masses)))

    def maximin_pad_raw(self, colors, n, centers, k0, k, out):
        check(self.L.cqg_maximin_pad(self.h, ptr(colors), n, ptr(centers), k0, k, ptr(out)))

    def map_raw(self, rgb, P, palette, k, indices, index_bytes, quantized, with_ndc: bool = False):
        """cqg_map: the mean squared distance, or (mse, MappingResult::ndc) with with_ndc."""
        mse, ndc = C.c_double(0), C.c_uint64(0)
        check(self.L.cqg_map(self.h, ptr(rgb), P, ptr(palette), k, ptr(indices), index_bytes,
                             ptr(quantized), C.byref(mse), C.byref(ndc) if with_ndc else None))
        return (mse.value, ndc.value) if with_ndc else mse.value

    def quantize_raw(self, rgb, P, cfg: QuantizeCfg, init, palette, labels, sse, indices,
                     quantized) -> QuantizeStats:
        st = QuantizeStats()
        check(self.L.cqg_quantize(self.h, ptr(rgb), P, C.byref(cfg), ptr(init), ptr(palette),
                                  ptr(labels), ptr(sse), ptr(indices), ptr(quantized),
                                  C.byref(st)))
        return st


_default = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        _default[device] = ctx
    return ctx
