"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker (never as the product).

* ``Oracle``  -> oracle/libcqoracle.so, the plain-C restatement (cq_oracle.c).
* ``RefLib``  -> oracle/_ref/libquantref.so, the reference's own sources compiled
  in place (oracle/Makefile) behind oracle/ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libcqoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libquantref.so")

UPDATE_REFERENCE = 0
UPDATE_EXACT = 1

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


def build(quiet: bool = True) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)
    # the reference's unit tests against the drop-in (needs libquant_b200.so)
    if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1101_0395_b200", "libquant_b200.so")):
        from oracle import refsuite
        refsuite.build(quiet=quiet)


def _nullable(arr):
    return None if arr is None else arr.ctypes.data_as(C.c_void_p)


@dataclass
class LloydResult:
    centers: np.ndarray
    labels: np.ndarray
    sse_trace: np.ndarray
    iterations: int
    ndc_total: int
    repairs: int
    hist_labels: np.ndarray | None = None
    hist_centers: np.ndarray | None = None
    seconds: float = 0.0

    def ndc_per_point_iter(self) -> float:
        n = self.labels.shape[0]
        return 0.0 if n == 0 or self.iterations == 0 else self.ndc_total / (n * self.iterations)


class Oracle:
    """The C restatement of the reference hot path."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.cqo_histogram.restype = C.c_int64
        L.cqo_histogram.argtypes = [_u8p, C.c_uint64, _u32p, _u32p, C.c_void_p]
        L.cqo_coarse_histogram.restype = None
        L.cqo_coarse_histogram.argtypes = [_u32p, _u32p, C.c_uint64, C.c_void_p]
        L.cqo_weights.argtypes = [_u32p, C.c_uint64, C.c_uint64, _f64p]
        L.cqo_center_table.argtypes = [_f64p, C.c_int, _f64p, _u32p]
        L.cqo_wsm.restype = C.c_int
        L.cqo_wsm.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, _f64p, C.c_int, C.c_double,
                              C.c_int, C.c_int, C.c_int, _f64p, _u32p, _f64p,
                              C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                              C.c_void_p, C.c_void_p]
        L.cqo_init_maximin.restype = C.c_int
        L.cqo_init_maximin.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                       C.c_int, _f64p]
        L.cqo_init_kmeanspp.restype = C.c_int
        L.cqo_init_kmeanspp.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                        _f64p]
        L.cqo_map_pixels.restype = C.c_int
        L.cqo_map_pixels.argtypes = [_u8p, C.c_uint64, _f64p, C.c_int, C.c_int, _u32p, _u8p,
                                     C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.cqo_psnr.restype = C.c_double
        L.cqo_psnr.argtypes = [C.c_double]
        L.cqo_rng_size.restype = C.c_int
        L.cqo_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.cqo_rng_u64.restype = C.c_uint64
        L.cqo_rng_u64.argtypes = [C.c_void_p]
        L.cqo_rng_unit.restype = C.c_double
        L.cqo_rng_unit.argtypes = [C.c_void_p]
        L.cqo_rng_below.restype = C.c_uint64
        L.cqo_rng_below.argtypes = [C.c_void_p, C.c_uint64]

    # --- stage 1 -----------------------------------------------------------
    def histogram(self, rgb: np.ndarray):
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8).reshape(-1)
        P = rgb.size // 3
        cap = min(P, 1 << 24)
        colors = np.empty(cap, np.uint32)
        counts = np.empty(cap, np.uint32)
        first = np.empty(cap, np.uint32)
        n = self.L.cqo_histogram(rgb, P, colors, counts, first.ctypes.data_as(C.c_void_p))
        if n < 0:
            raise ValueError("build_histogram: no pixels")
        return colors[:n].copy(), counts[:n].copy(), first[:n].copy()

    def weights(self, counts: np.ndarray, P: int) -> np.ndarray:
        counts = np.ascontiguousarray(counts, np.uint32)
        w = np.empty(counts.size, np.float64)
        self.L.cqo_weights(counts, counts.size, P, w)
        return w

    def center_table(self, centers: np.ndarray):
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        K = c.size // 3
        d2 = np.empty(K * K, np.float64)
        order = np.empty(K * K, np.uint32)
        self.L.cqo_center_table(c, K, d2, order)
        return d2.reshape(K, K), order.reshape(K, K)

    # --- stages 2+3 --------------------------------------------------------
    def wsm(self, colors, counts, P, init, eps=1e-3, max_it=100, fixed_it=0,
            mode=UPDATE_EXACT, history=False) -> LloydResult:
        colors = np.ascontiguousarray(colors, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        init = np.ascontiguousarray(init, np.float64).reshape(-1)
        n = colors.size
        K = init.size // 3
        limit = fixed_it if fixed_it > 0 else max_it
        centers = np.empty(3 * K, np.float64)
        labels = np.empty(n, np.uint32)
        sse = np.zeros(max(limit, 1), np.float64)
        it, ndc, rep = C.c_int(0), C.c_uint64(0), C.c_int(0)
        hl = np.empty(limit * n, np.uint32) if history else None
        hc = np.empty(limit * 3 * K, np.float64) if history else None
        rc = self.L.cqo_wsm(colors, counts, n, P, init, K, eps, max_it, fixed_it, mode, centers,
                            labels, sse, C.byref(it), C.byref(ndc), C.byref(rep), _nullable(hl),
                            _nullable(hc))
        if rc != 0:
            raise ValueError(f"oracle wsm failed: code {rc}")
        iters = it.value
        return LloydResult(centers.reshape(K, 3), labels, sse[:iters].copy(), iters, ndc.value,
                           rep.value,
                           None if hl is None else hl[: iters * n].reshape(iters, n),
                           None if hc is None else hc[: iters * 3 * K].reshape(iters, K, 3))

    # --- init -----------------------------------------------------------------
    def init_maximin(self, colors, counts, P, K, seed, weighted_first=True):
        c = np.empty(3 * K, np.float64)
        rc = self.L.cqo_init_maximin(np.ascontiguousarray(colors, np.uint32),
                                     np.ascontiguousarray(counts, np.uint32), len(colors), P, K,
                                     seed, 1 if weighted_first else 0, c)
        if rc != 0:
            raise ValueError(f"oracle init_maximin failed: code {rc}")
        return c.reshape(K, 3)

    def init_kmeanspp(self, colors, counts, P, K, seed):
        c = np.empty(3 * K, np.float64)
        rc = self.L.cqo_init_kmeanspp(np.ascontiguousarray(colors, np.uint32),
                                      np.ascontiguousarray(counts, np.uint32), len(colors), P, K,
                                      seed, c)
        if rc != 0:
            raise ValueError(f"oracle init_kmeanspp failed: code {rc}")
        return c.reshape(K, 3)

    # --- stage 4 --------------------------------------------------------------
    def map_pixels(self, rgb, palette, mode=UPDATE_EXACT):
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
        P = rgb.size // 3
        pal = np.ascontiguousarray(palette, np.float64).reshape(-1)
        K = pal.size // 3
        idx = np.empty(P, np.uint32)
        q = np.empty(3 * P, np.uint8)
        mse, ndc = C.c_double(0), C.c_uint64(0)
        rc = self.L.cqo_map_pixels(rgb, P, pal, K, mode, idx, q, C.byref(mse), C.byref(ndc))
        if rc != 0:
            raise ValueError(f"oracle map_pixels failed: code {rc}")
        return idx, q.reshape(P, 3), mse.value, ndc.value

    def psnr(self, mse: float) -> float:
        return self.L.cqo_psnr(mse)

    def coarse_histogram(self, colors, counts):
        """(count, sum_r, sum_g, sum_b, sum_sq), 32768 int64 each (precluster.cpp:13-47)."""
        out = np.empty(5 * 32768, np.int64)
        self.L.cqo_coarse_histogram(np.ascontiguousarray(colors, np.uint32), np.ascontiguousarray(counts, np.uint32),
                                    len(colors), out.ctypes.data_as(C.c_void_p))
        return out.reshape(5, 32768)

    # --- rng ------------------------------------------------------------------
    def rng(self, seed: int):
        buf = C.create_string_buffer(self.L.cqo_rng_size())
        self.L.cqo_rng_seed(buf, seed)
        return buf


class RefLib:
    """The reference's own library (compiled in place), through ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_synthetic_photo.argtypes = [C.c_int, C.c_int, C.c_uint64, _u8p]
        L.ref_coarse_histogram.restype = C.c_int
        L.ref_coarse_histogram.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                           C.c_void_p]
        L.ref_histogram.restype = C.c_int64
        L.ref_histogram.argtypes = [_u8p, C.c_uint64, C.c_uint64, _u32p, _u32p, C.c_void_p]
        L.ref_init.argtypes = [C.c_int, _u32p, _u32p, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                               _f64p, C.POINTER(C.c_int)]
        L.ref_wsm.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint64, _f64p, C.c_int, C.c_double,
                              C.c_int, C.c_int, _f64p, _u32p, _f64p, C.POINTER(C.c_int),
                              C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                              C.POINTER(C.c_double)]
        L.ref_map_pixels.argtypes = [_u8p, C.c_int, C.c_int, _f64p, C.c_int, C.c_void_p,
                                     C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_double)]
        L.ref_run_quantize.argtypes = [_u8p, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_uint64,
                                       C.c_double, C.c_int, C.c_int, C.c_char_p, C.c_int, _f64p,
                                       C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_char_p, C.c_void_p, C.c_void_p]
        L.ref_run_quantize_s.argtypes = L.ref_run_quantize.argtypes + [C.c_char_p]
        for nm in ("ref_lloyd_general", "ref_compute_sse", "ref_repair", "ref_center_table", "ref_next_masses",
                   "ref_maximin_pad"):
            getattr(L, nm).restype = C.c_int
        L.ref_lloyd_general.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_double,
                                        C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.c_void_p, C.c_void_p]
        L.ref_compute_sse.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p,
                                      C.POINTER(C.c_double)]
        L.ref_repair.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p,
                                 C.POINTER(C.c_int)]
        L.ref_center_table.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_next_masses.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
        L.ref_maximin_pad.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_int,
                                      C.c_void_p, C.POINTER(C.c_int)]
        L.ref_time_pipeline.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                        C.c_double, C.c_int, C.c_int, _f64p,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                        C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            raise ValueError(self.L.ref_last_error().decode())

    # --- the general API (real points, arbitrary weights) ---------------------
    def lloyd_general(self, points, weights, init, eps=1e-3, max_it=100, fixed_it=0, history=False):
        """wsm(points, weights, init) or, with weights None, kmeans_full(points, init)."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        init = np.ascontiguousarray(init, np.float64).reshape(-1, 3)
        n, K = pts.shape[0], init.shape[0]
        limit = fixed_it if fixed_it > 0 else max_it
        centers = np.empty((K, 3), np.float64)
        labels = np.empty(n, np.uint32)
        sse = np.zeros(limit, np.float64)
        it, ndc, rep = C.c_int(0), C.c_uint64(0), C.c_int(0)
        hl = np.empty((limit, n), np.uint32) if history else None
        hc = np.empty((limit, K, 3), np.float64) if history else None
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self._check(self.L.ref_lloyd_general(pts.ctypes.data_as(C.c_void_p), _nullable(w), n,
                                             init.ctypes.data_as(C.c_void_p), K, eps, max_it, fixed_it,
                                             centers.ctypes.data_as(C.c_void_p), labels.ctypes.data_as(C.c_void_p),
                                             sse.ctypes.data_as(C.c_void_p), C.byref(it), C.byref(ndc),
                                             C.byref(rep), _nullable(hl), _nullable(hc)))
        iters = it.value
        return LloydResult(centers, labels, sse[:iters].copy(), iters, ndc.value, rep.value,
                           None if hl is None else hl[:iters].copy(), None if hc is None else hc[:iters].copy())

    def compute_sse(self, points, weights, centers, labels):
        pts = np.ascontiguousarray(points, np.float64)
        c = np.ascontiguousarray(centers, np.float64)
        m = np.ascontiguousarray(labels, np.uint32)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        out = C.c_double(0)
        self._check(self.L.ref_compute_sse(pts.ctypes.data_as(C.c_void_p), _nullable(w), m.size,
                                           c.ctypes.data_as(C.c_void_p), c.size // 3, m.ctypes.data_as(C.c_void_p),
                                           C.byref(out)))
        return out.value

    def repair(self, points, weights, centers, labels):
        pts = np.ascontiguousarray(points, np.float64)
        c = np.array(centers, np.float64, copy=True, order="C")
        m = np.array(labels, np.uint32, copy=True, order="C")
        w = np.ascontiguousarray(weights, np.float64)
        r = C.c_int(0)
        self._check(self.L.ref_repair(pts.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), m.size,
                                      c.ctypes.data_as(C.c_void_p), c.size // 3, m.ctypes.data_as(C.c_void_p),
                                      C.byref(r)))
        return r.value, c, m

    def center_table(self, centers):
        c = np.ascontiguousarray(centers, np.float64)
        K = c.size // 3
        d = np.empty((K, K), np.float64)
        o = np.empty((K, K), np.uint32)
        self._check(self.L.ref_center_table(c.ctypes.data_as(C.c_void_p), K, d.ctypes.data_as(C.c_void_p),
                                            o.ctypes.data_as(C.c_void_p)))
        return d, o

    def next_masses(self, colors, weights, centers):
        cols = np.ascontiguousarray(colors, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        out = np.empty(w.size, np.float64)
        self._check(self.L.ref_next_masses(cols.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), w.size,
                                           c.ctypes.data_as(C.c_void_p), c.shape[0], out.ctypes.data_as(C.c_void_p)))
        return out

    def maximin_pad(self, colors, weights, centers, k):
        cols = np.ascontiguousarray(colors, np.float64)
        w = np.ascontiguousarray(weights, np.float64)
        c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        out = np.empty((max(k, c.shape[0], 1), 3), np.float64)
        ko = C.c_int(0)
        self._check(self.L.ref_maximin_pad(cols.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), w.size,
                                           c.ctypes.data_as(C.c_void_p), c.shape[0], k,
                                           out.ctypes.data_as(C.c_void_p), C.byref(ko)))
        return out[:ko.value].copy()

    def coarse_histogram(self, rgb=None, colors=None, counts=None):
        """quant::build_coarse_histogram from pixels (rgb) or from a weighted
        histogram (colors, counts): a (5, 32768) int64 array."""
        out = np.empty(5 * 32768, np.int64)
        if colors is None:
            px = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
            rc = self.L.ref_coarse_histogram(px.ctypes.data_as(C.c_void_p), px.size // 3, None, None, 0,
                                             out.ctypes.data_as(C.c_void_p))
        else:
            c = np.ascontiguousarray(colors, np.uint32)
            n = np.ascontiguousarray(counts, np.uint32)
            rc = self.L.ref_coarse_histogram(None, 0, c.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p),
                                             c.size, out.ctypes.data_as(C.c_void_p))
        self._check(rc)
        return out.reshape(5, 32768)

    def synthetic_photo(self, w, h, seed):
        out = np.empty(w * h * 3, np.uint8)
        self.L.ref_synthetic_photo(w, h, seed, out)
        return out.reshape(h, w, 3)

    def histogram(self, rgb, seed=1):
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
        P = rgb.size // 3
        cap = min(P, 1 << 24)
        colors = np.empty(cap, np.uint32)
        counts = np.empty(cap, np.uint32)
        w = np.empty(cap, np.float64)
        n = self.L.ref_histogram(rgb, P, seed, colors, counts, w.ctypes.data_as(C.c_void_p))
        if n < 0:
            self._check(-1)
        return colors[:n].copy(), counts[:n].copy(), w[:n].copy()

    def init(self, kind, colors, counts, P, K, seed):
        kinds = {"mmx": 0, "kpp": 1, "wu": 2}
        c = np.zeros(3 * K, np.float64)
        ko = C.c_int(0)
        self._check(self.L.ref_init(kinds[kind], np.ascontiguousarray(colors, np.uint32),
                                    np.ascontiguousarray(counts, np.uint32), len(colors), P, K,
                                    seed, c, C.byref(ko)))
        return c[: 3 * ko.value].reshape(ko.value, 3)

    def wsm(self, colors, counts, P, init, eps=1e-3, max_it=100, fixed_it=0, history=False):
        colors = np.ascontiguousarray(colors, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        init = np.ascontiguousarray(init, np.float64).reshape(-1)
        n, K = colors.size, init.size // 3
        limit = fixed_it if fixed_it > 0 else max_it
        centers = np.empty(3 * K, np.float64)
        labels = np.empty(n, np.uint32)
        sse = np.zeros(limit, np.float64)
        it, ndc, rep, secs = C.c_int(0), C.c_uint64(0), C.c_int(0), C.c_double(0)
        hl = np.empty(limit * n, np.uint32) if history else None
        hc = np.empty(limit * 3 * K, np.float64) if history else None
        self._check(self.L.ref_wsm(colors, counts, n, P, init, K, eps, max_it, fixed_it, centers,
                                   labels, sse, C.byref(it), C.byref(ndc), C.byref(rep),
                                   _nullable(hl), _nullable(hc), C.byref(secs)))
        iters = it.value
        return LloydResult(centers.reshape(K, 3), labels, sse[:iters].copy(), iters, ndc.value,
                           rep.value,
                           None if hl is None else hl[: iters * n].reshape(iters, n),
                           None if hc is None else hc[: iters * 3 * K].reshape(iters, K, 3),
                           secs.value)

    def map_pixels(self, rgb, w, h, palette):
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
        pal = np.ascontiguousarray(palette, np.float64).reshape(-1)
        P = w * h
        idx = np.empty(P, np.uint32)
        q = np.empty(3 * P, np.uint8)
        mse, ndc, secs = C.c_double(0), C.c_uint64(0), C.c_double(0)
        self._check(self.L.ref_map_pixels(rgb, w, h, pal, pal.size // 3,
                                          idx.ctypes.data_as(C.c_void_p),
                                          q.ctypes.data_as(C.c_void_p), C.byref(mse),
                                          C.byref(ndc), C.byref(secs)))
        return idx, q.reshape(P, 3), mse.value, ndc.value

    def run_quantize(self, rgb, w, h, method, k, seed, eps=1e-3, max_it=100, fixed_it=0,
                     name="", run=0, sampling="unique", outputs=False):
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
        pal = np.zeros(3 * k, np.float64)
        ka, it = C.c_int(0), C.c_int(0)
        ndc, mse, tms = C.c_double(0), C.c_double(0), C.c_double(0)
        csv = C.create_string_buffer(512)
        idx = np.zeros(w * h, np.uint32) if outputs else None
        q = np.zeros(w * h * 3, np.uint8) if outputs else None
        self._check(self.L.ref_run_quantize_s(rgb, w, h, method.encode(), k, seed, eps, max_it,
                                              fixed_it, name.encode(), run, pal, C.byref(ka),
                                              C.byref(it), C.byref(ndc), C.byref(mse), C.byref(tms),
                                              csv, _nullable(idx), _nullable(q), sampling.encode()))
        out = dict(palette=pal[: 3 * ka.value].reshape(-1, 3), k_actual=ka.value,
                   iterations=it.value, ndc_per_point_iter=ndc.value, mse=mse.value,
                   time_ms=tms.value, csv_row=csv.value.decode())
        if outputs:
            out["indices"] = idx
            out["quantized"] = q.reshape(h, w, 3)
        return out

    def time_pipeline(self, rgb, w, h, init_kind, k, seed, eps=1e-3, max_it=100, fixed_it=0):
        rgb = np.ascontiguousarray(rgb, np.uint8).reshape(-1)
        st = np.zeros(4, np.float64)
        nu, it, mse = C.c_uint64(0), C.c_int(0), C.c_double(0)
        self._check(self.L.ref_time_pipeline(rgb, w, h, 1 if init_kind == "kpp" else 0, k, seed,
                                             eps, max_it, fixed_it, st, C.byref(nu), C.byref(it),
                                             C.byref(mse)))
        return dict(stage_s=st, n_unique=nu.value, iterations=it.value, mse=mse.value)


def have_ref() -> bool:
    return os.path.exists(REF_SO)
