"""Python mirror of the reference quantiser API for the hot path.

Same names, argument meaning and error behaviour as the reference's C++ API in
proj/include/quant/*.hpp (cited per function); everything is computed by
libcqg.so through the C-ABI (cabi.py). std::invalid_argument maps to
``ValueError`` (cabi.InvalidArgument), std::runtime_error to ``RuntimeError``.

Images are numpy uint8 arrays of shape (H, W, 3) (quant::RawImage,
image.hpp:13-24) or flat P*3 byte arrays; palettes / centres are (K, 3) float64
(quant::ColorPoint, color.hpp:21-45).
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import cabi

# ---------------------------------------------------------------------------
# colour helpers (color.hpp:47-72)


def channel_to_u8(v: np.ndarray | float) -> np.ndarray:
    """Round half up, clamp to [0, 255] (color.hpp:63-68)."""
    r = np.floor(np.asarray(v, np.float64) + 0.5)
    return np.clip(r, 0.0, 255.0).astype(np.uint8)


def pack_colors(rgb: np.ndarray) -> np.ndarray:
    rgb = np.asarray(rgb, np.uint8).reshape(-1, 3).astype(np.uint32)
    return (rgb[:, 0] << 16) | (rgb[:, 1] << 8) | rgb[:, 2]


def unpack_colors(c: np.ndarray) -> np.ndarray:
    c = np.asarray(c, np.uint32)
    return np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], axis=1).astype(np.float64)


def _pixels(image) -> tuple[np.ndarray, int, int]:
    if isinstance(image, RawImage):
        arr = image.pixels
    else:
        arr = image
    if hasattr(arr, "data_ptr") and not isinstance(arr, np.ndarray):  # device tensor
        shape = tuple(arr.shape)
        if len(shape) == 3:
            return arr, shape[1], shape[0]
        return arr, arr.numel() // 3, 1
    arr = np.ascontiguousarray(arr, np.uint8)
    if arr.ndim == 3:
        return arr, arr.shape[1], arr.shape[0]
    return arr.reshape(-1), arr.size // 3, 1


@dataclass
class RawImage:
    """quant::RawImage (image.hpp:13-24): interleaved 8-bit RGB, row-major."""
    width: int
    height: int
    pixels: np.ndarray  # (H, W, 3) uint8

    def pixel_count(self) -> int:
        return self.width * self.height


def load_image(path: str) -> RawImage:
    """quant::load_image (image.hpp:36) for binary PPM (P6, maxval 255): header
    tokens separated by whitespace, '#' comments to end of line, exactly one
    whitespace byte before the raster. Errors are the reference's
    RuntimeError messages "<path>: <what>". PNG needs libpng (not linked)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"{path}: cannot open file") from None
    if len(data) < 2:
        raise RuntimeError(f"{path}: file too short to identify")
    if data[:2] == b"\x89P":
        raise RuntimeError(f"{path}: PNG input needs libpng, which this build does not link")
    if data[:2] != b"P6":
        raise RuntimeError(f"{path}: unsupported format (expected binary PPM 'P6' or PNG)")
    pos = 2

    def field(name):
        nonlocal pos
        tok = b""
        while pos < len(data):
            c = data[pos:pos + 1]
            pos += 1
            if c == b"#":
                while pos < len(data) and data[pos:pos + 1] != b"\n":
                    pos += 1
                pos += 1 if pos < len(data) else 0
                continue
            if c.isspace():
                if tok:
                    break
                continue
            tok += c
        if not tok:
            raise RuntimeError(f"{path}: truncated PPM header (missing {name})")
        try:
            return int(tok.decode("ascii"), 10)
        except ValueError:
            raise RuntimeError(f"{path}: malformed PPM {name} '{tok.decode('latin-1')}'") from None

    w, h, maxval = field("width"), field("height"), field("maxval")
    if w <= 0 or h <= 0:
        raise RuntimeError(f"{path}: non-positive PPM dimensions")
    if maxval != 255:
        raise RuntimeError(f"{path}: unsupported PPM maxval {maxval} (only 255)")
    need = w * h * 3
    raster = data[pos:pos + need]
    if len(raster) != need:
        raise RuntimeError(f"{path}: truncated PPM pixel data (expected {need} bytes, got {len(raster)})")
    return RawImage(w, h, np.frombuffer(raster, np.uint8).reshape(h, w, 3).copy())


def save_image(image: RawImage, path: str) -> None:
    """quant::save_image / save_ppm (image.hpp:39-42): "P6\\n<w> <h>\\n255\\n" + raw RGB."""
    low = path.lower()
    if low.endswith(".png"):
        raise RuntimeError(f"{path}: PNG output needs libpng, which this build does not link")
    if not low.endswith(".ppm"):
        raise RuntimeError(f"{path}: unknown output extension (use .ppm or .png)")
    px = np.ascontiguousarray(image.pixels, np.uint8)
    if image.width <= 0 or image.height <= 0 or px.size != image.width * image.height * 3:
        raise ValueError("save_ppm: inconsistent image dimensions")
    try:
        with open(path, "wb") as f:
            f.write(f"P6\n{image.width} {image.height}\n255\n".encode("ascii"))
            f.write(px.tobytes())
    except OSError:
        raise RuntimeError(f"{path}: cannot open file for writing") from None


# ---------------------------------------------------------------------------
# stage 1 (histogram.hpp:19-60)

SAMPLING_TOKENS = {"none": "None", "2to1": "TwoToOne", "unique": "Unique", "both": "TwoToOneUnique"}


# QuantizeConfig::sampling -> CQG_SAMPLING_* (include/cqg.h)
SAMPLING_CODES = {"unique": 0, "none": 1, "2to1": 2, "both": 3}


def parse_sampling_mode(token: str) -> str:
    """histogram.cpp:19-26."""
    if token not in SAMPLING_TOKENS:
        raise ValueError(f"unknown sampling mode '{token}' (expected none|2to1|unique|both)")
    return token


@dataclass
class WeightedHistogram:
    """quant::WeightedHistogram (histogram.hpp:43-51), first-occurrence order."""
    colors: np.ndarray                  # (N', 3) float64
    weights: np.ndarray                 # (N',) float64 = counts * (1/P)
    counts: np.ndarray                  # (N',) uint32
    source_pixel_count: int
    packed: np.ndarray = field(repr=False, default=None)  # (N',) uint32 0x00RRGGBB
    first: np.ndarray = field(repr=False, default=None)   # first pixel index per colour

    def size(self) -> int:
        return int(self.counts.size)


def build_histogram(pixels, seed: int = 1, ctx: Optional[cabi.Context] = None) -> WeightedHistogram:
    """quant::build_histogram (histogram.hpp:57, histogram.cpp:69-104) on the device.

    ``seed`` only seeds the reference's hash coefficients; the output does not
    depend on it (the device dedups through a direct 2^24 table)."""
    ctx = ctx or cabi.default_context()
    arr, w, h = _pixels(pixels)
    P = w * h
    if P == 0:
        raise ValueError("build_histogram: no pixels")
    cap = min(P, 1 << 24)
    colors = np.empty(cap, np.uint32)
    counts = np.empty(cap, np.uint32)
    first = np.empty(cap, np.uint32)
    n = ctx.histogram_raw(arr, P, colors, counts, first)
    colors, counts, first = colors[:n].copy(), counts[:n].copy(), first[:n].copy()
    inv = 1.0 / float(P)
    weights = counts.astype(np.float64) * inv
    return WeightedHistogram(unpack_colors(colors), weights, counts, P, colors, first)


@dataclass
class CoarseHistogram:
    """quant::CoarseHistogram (precluster.hpp:16-30): 32x32x32 bins (5 bits per
    channel, r-major), per bin the pixel count and the sums of the original
    r, g, b and r^2+g^2+b^2."""
    count: np.ndarray   # (32768,) uint64
    sum_r: np.ndarray   # (32768,) int64
    sum_g: np.ndarray
    sum_b: np.ndarray
    sum_sq: np.ndarray
    grid = 32
    bins = 32768

    @staticmethod
    def bin_index(br: int, bg: int, bb: int) -> int:
        return (br * 32 + bg) * 32 + bb


def build_coarse_histogram(source, ctx: Optional[cabi.Context] = None) -> CoarseHistogram:
    """quant::build_coarse_histogram (precluster.hpp:32-34, precluster.cpp:13-47)
    on the device, from pixels or from a WeightedHistogram (same integers)."""
    ctx = ctx or cabi.default_context()
    out = np.empty((5, 32768), np.int64)
    if isinstance(source, WeightedHistogram):
        if source.size() == 0:
            raise ValueError("build_coarse_histogram: empty histogram")
        packed = source.packed if source.packed is not None else pack_colors(source.colors)
        ctx.coarse_histogram_weighted_raw(np.ascontiguousarray(packed, np.uint32),
                                          np.ascontiguousarray(source.counts, np.uint32), source.size(), out)
    else:
        arr, w, h = _pixels(source)
        if w * h == 0:
            raise ValueError("build_coarse_histogram: no pixels")
        ctx.coarse_histogram_raw(arr, w * h, out)
    return CoarseHistogram(out[0].view(np.uint64).copy(), out[1].copy(), out[2].copy(), out[3].copy(),
                           out[4].copy())


# ---------------------------------------------------------------------------
# stages 2+3 (kmeans.hpp:17-129)


@dataclass
class Termination:
    """quant::Termination (kmeans.hpp:17-21)."""
    epsilon: float = 1e-3
    max_iterations: int = 100
    fixed_iterations: Optional[int] = None


@dataclass
class ClusterOptions:
    """quant::ClusterOptions (kmeans.hpp:28-35)."""
    term: Termination = field(default_factory=Termination)
    record_history: bool = False


@dataclass
class IterationSnapshot:
    centers: np.ndarray
    memberships: np.ndarray


@dataclass
class ClusterState:
    """quant::ClusterState (kmeans.hpp:42-56)."""
    centers: np.ndarray = None
    memberships: np.ndarray = None
    sse_trace: np.ndarray = None
    iterations: int = 0
    ndc_total: int = 0
    repair_count: int = 0
    history: list = field(default_factory=list)
    flagged_total: int = 0  # device diagnostic: points replayed in exact FP64
    swept_total: int = 0    # device diagnostic: points evaluated against every centre

    def ndc_per_point_iter(self, point_count: int) -> float:
        if point_count == 0 or self.iterations == 0:
            return 0.0
        return float(self.ndc_total) / (float(point_count) * float(self.iterations))


def check_convergence(sse_prev: float, sse_cur: float, epsilon: float) -> bool:
    """kmeans.cpp:9-12."""
    if sse_cur == 0.0:
        return True
    return (sse_prev - sse_cur) / sse_cur <= epsilon


def _term_struct(term: Termination, record_history: bool) -> cabi.Term:
    if term.fixed_iterations is not None and term.fixed_iterations <= 0:
        raise ValueError("clustering: fixed_iterations < 1")  # kmeans.cpp:187-188
    return cabi.Term(float(term.epsilon), int(term.max_iterations),
                     int(term.fixed_iterations or 0), 1 if record_history else 0)


def wsm_hist(hist: WeightedHistogram, init, options: ClusterOptions = None,
             ctx: Optional[cabi.Context] = None) -> ClusterState:
    """quant::wsm (kmeans.hpp:128-129, kmeans.cpp:271-277) over a histogram's
    count-weighted colours (weights = counts / source_pixel_count)."""
    return wsm_counts(hist.packed if hist.packed is not None else pack_colors(hist.colors),
                      hist.counts, hist.source_pixel_count, init, options, ctx)


def wsm_counts(colors_packed, counts, P: int, init, options: ClusterOptions = None,
               ctx: Optional[cabi.Context] = None) -> ClusterState:
    """Weighted sort-means on packed colours with integer counts (weights = counts/P)."""
    options = options or ClusterOptions()
    term = _term_struct(options.term, options.record_history)
    ctx = ctx or cabi.default_context()
    colors_packed = np.ascontiguousarray(colors_packed, np.uint32)
    counts = np.ascontiguousarray(counts, np.uint32)
    init = np.ascontiguousarray(np.asarray(init, np.float64).reshape(-1, 3))
    n, k = colors_packed.size, init.shape[0]
    limit = term.fixed_iterations if term.fixed_iterations > 0 else max(term.max_iterations, 1)
    centers = np.empty((max(k, 1), 3), np.float64)
    labels = np.empty(max(n, 1), np.uint32)
    sse = np.zeros(limit, np.float64)
    hl = np.empty((limit, n), np.uint32) if options.record_history else None
    hc = np.empty((limit, max(k, 1), 3), np.float64) if options.record_history else None
    st = ctx.lloyd_raw(colors_packed, counts, n, P, init if k else np.zeros((1, 3)), k, term,
                       centers, labels, sse, hl, hc)
    it = st.iterations
    hist = []
    if options.record_history:
        hist = [IterationSnapshot(hc[i].copy(), hl[i].copy()) for i in range(it)]
    return ClusterState(centers[:k].copy(), labels[:n].copy(), sse[:it].copy(), it,
                        int(st.ndc_total), int(st.repair_count), hist, int(st.flagged_total),
                        int(st.swept_total))


def wsm(points, weights, init, options: ClusterOptions = None,
        ctx: Optional[cabi.Context] = None) -> ClusterState:
    """quant::wsm(points, weights, init, options) (kmeans.hpp:128-129).

    Count-weighted substrates on the 8-bit grid (w_i == c_i * (1/P), what
    run_quantize builds) run on the hot-path engine (exact integer moments);
    any other points or positive weights run on the general exact-FP64 device
    engine (cqg_lloyd_exact), which reproduces the reference's sequential sums."""
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    w = np.asarray(weights, np.float64).reshape(-1)
    init = np.asarray(init, np.float64).reshape(-1, 3)
    n, k = pts.shape[0], init.shape[0]
    if k == 0:
        raise ValueError("clustering: no initial centers")
    if n == 0:
        raise ValueError("clustering: no points")
    if k > n:
        raise ValueError(f"clustering: k ({k}) exceeds number of points ({n})")
    if w.size != n:
        raise ValueError("clustering: weights/points size mismatch")
    if not np.all(w > 0.0):
        raise ValueError("wsm: weights must be positive")
    if np.any(pts != np.round(pts)) or pts.min() < 0 or pts.max() > 255:
        return _lloyd_exact(pts, w, init, options, ctx)
    # recover integer counts: w_i = c_i * (1/P) exactly (histogram.cpp:99-102)
    wmin = float(w.min())
    counts, P = None, None
    for cmin in range(1, 257):
        cand_p = int(round(cmin / wmin))
        if cand_p <= 0:
            continue
        c = np.round(w * cand_p)
        if int(c.sum()) == cand_p and np.array_equal(c * (1.0 / float(cand_p)), w):
            counts, P = c, cand_p
            break
    if P is None:
        return _lloyd_exact(pts, w, init, options, ctx)
    packed = pack_colors(pts.astype(np.uint8))
    return wsm_counts(packed, np.asarray(counts, np.uint32), P, init, options, ctx)


def _lloyd_exact(pts, w, init, options, ctx):
    """The general exact-FP64 engine (cqg_lloyd_exact): wsm when w is given,
    kmeans_full when w is None."""
    options = options or ClusterOptions()
    term = _term_struct(options.term, options.record_history)
    ctx = ctx or cabi.default_context()
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    init = np.ascontiguousarray(np.asarray(init, np.float64).reshape(-1, 3))
    n, k = pts.shape[0], init.shape[0]
    limit = term.fixed_iterations if term.fixed_iterations > 0 else max(term.max_iterations, 1)
    centers = np.empty((max(k, 1), 3), np.float64)
    labels = np.empty(max(n, 1), np.uint32)
    sse = np.zeros(limit, np.float64)
    hl = np.empty((limit, max(n, 1)), np.uint32) if options.record_history else None
    hc = np.empty((limit, max(k, 1), 3), np.float64) if options.record_history else None
    wv = None if w is None else np.ascontiguousarray(w, np.float64)
    st = ctx.lloyd_exact_raw(pts if n else np.zeros((1, 3)), wv, n, init if k else np.zeros((1, 3)), k, term,
                             centers, labels, sse, hl, hc)
    it = st.iterations
    hist = [IterationSnapshot(hc[i].copy(), hl[i][:n].copy()) for i in range(it)] if options.record_history else []
    return ClusterState(centers[:k].copy(), labels[:n].copy(), sse[:it].copy(), it, int(st.ndc_total),
                        int(st.repair_count), hist, 0, int(st.swept_total))


def kmeans_full(points, init, options: ClusterOptions = None,
                ctx: Optional[cabi.Context] = None) -> ClusterState:
    """quant::kmeans_full (kmeans.hpp:119, kmeans.cpp:263-268): plain k-means on
    unweighted points -- full scan every iteration, arithmetic means, no
    repair (an empty cluster keeps its centre); on the device."""
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    return _lloyd_exact(pts, None, init, options, ctx)


def compute_sse(points, *args, ctx: Optional[cabi.Context] = None) -> float:
    """quant::compute_sse (kmeans.hpp:99-105): compute_sse(points, weights,
    centers, memberships) or the unit-weight compute_sse(points, centers,
    memberships); one sequential FP64 chain in point order, on the device."""
    if len(args) == 3:
        weights, centers, memberships = args
    elif len(args) == 2:
        weights, (centers, memberships) = None, args
    else:
        raise TypeError("compute_sse(points, [weights,] centers, memberships)")
    ctx = ctx or cabi.default_context()
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    m = np.ascontiguousarray(memberships, np.uint32)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    return ctx.compute_sse_raw(pts, w, pts.shape[0], c, c.shape[0], m)


def repair_empty_clusters(points, weights, centers: np.ndarray, memberships: np.ndarray,
                          ctx: Optional[cabi.Context] = None) -> int:
    """quant::repair_empty_clusters (kmeans.hpp:112-115, kmeans.cpp:124-169) on
    the device; ``centers`` (k, 3) float64 and ``memberships`` uint32 are
    updated in place. Returns the number of clusters repaired."""
    ctx = ctx or cabi.default_context()
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    w = np.ascontiguousarray(weights, np.float64)
    if not (centers.dtype == np.float64 and centers.flags["C_CONTIGUOUS"] and
            memberships.dtype == np.uint32 and memberships.flags["C_CONTIGUOUS"]):
        raise ValueError("repair_empty_clusters: centers float64 and memberships uint32, C-contiguous")
    return ctx.repair_raw(pts, w, pts.shape[0], centers, centers.shape[0], memberships)


@dataclass
class CenterDistanceTable:
    """quant::CenterDistanceTable (kmeans.hpp:62-69)."""
    k: int
    dist2: np.ndarray  # (k, k) float64
    order: np.ndarray  # (k, k) uint32, order[i, 0] == i

    def d2(self, i: int, j: int) -> float:
        return float(self.dist2[i, j])

    def order_at(self, i: int, n: int) -> int:
        return int(self.order[i, n])


def build_center_distance_table(centers, ctx: Optional[cabi.Context] = None) -> CenterDistanceTable:
    """quant::build_center_distance_table (kmeans.hpp:73, kmeans.cpp:14-38) on the device."""
    ctx = ctx or cabi.default_context()
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    k = c.shape[0]
    dist = np.zeros((k, k), np.float64)
    order = np.zeros((k, k), np.uint32)
    if k:
        ctx.center_table_raw(c, k, dist, order)
    return CenterDistanceTable(k, dist, order)


# ---------------------------------------------------------------------------
# init (init.hpp:17-72)


@dataclass
class SeedConfig:
    """quant::SeedConfig (init.hpp:17-27), the fields the device initialisers use."""
    k: int = 8
    seed: int = 1
    maximin_weighted_first: bool = True


def init_maximin(hist: WeightedHistogram, cfg: SeedConfig,
                 ctx: Optional[cabi.Context] = None) -> np.ndarray:
    """quant::init_maximin (init.hpp:40, init.cpp:127-138)."""
    return _init(cabi.INIT_MAXIMIN, hist, cfg, ctx)


def init_kmeanspp(hist: WeightedHistogram, cfg: SeedConfig,
                  ctx: Optional[cabi.Context] = None) -> np.ndarray:
    """quant::init_kmeanspp (init.hpp:60, init.cpp:295-314)."""
    return _init(cabi.INIT_KMEANSPP, hist, cfg, ctx)


def kmeanspp_next_masses(hist: WeightedHistogram, centers, ctx: Optional[cabi.Context] = None) -> np.ndarray:
    """quant::kmeanspp_next_masses (init.hpp:65-66, init.cpp:316-323): weight x
    min squared distance to the chosen centres (the weights when none), on the device."""
    ctx = ctx or cabi.default_context()
    c = np.ascontiguousarray(np.asarray(centers, np.float64).reshape(-1, 3))
    cols = np.ascontiguousarray(hist.colors, np.float64)
    w = np.ascontiguousarray(hist.weights, np.float64)
    out = np.empty(max(hist.size(), 1), np.float64)
    ctx.next_masses_raw(cols, w, hist.size(), c if c.shape[0] else None, c.shape[0], out)
    return out[:hist.size()].copy()


def maximin_pad(hist: WeightedHistogram, centers, k: int, ctx: Optional[cabi.Context] = None) -> np.ndarray:
    """quant::maximin_pad (init.hpp:71-72, init.cpp:325-335): extend a short
    centre set to k by maximin picks over the histogram, on the device."""
    ctx = ctx or cabi.default_context()
    c = np.ascontiguousarray(np.asarray(centers, np.float64).reshape(-1, 3))
    k0 = c.shape[0]
    out = np.empty((max(k, k0, 1), 3), np.float64)
    ctx.maximin_pad_raw(np.ascontiguousarray(hist.colors, np.float64), hist.size(), c if k0 else None, k0, int(k),
                        out)
    return out[:max(k, k0)].copy()


def _init(kind, hist, cfg, ctx):
    ctx = ctx or cabi.default_context()
    k = int(cfg.k)
    out = np.empty((max(k, 1), 3), np.float64)
    packed = hist.packed if hist.packed is not None else pack_colors(hist.colors)
    ctx.init_raw(kind, np.ascontiguousarray(packed, np.uint32),
                 np.ascontiguousarray(hist.counts, np.uint32), hist.size(),
                 hist.source_pixel_count, k, int(cfg.seed), out, cfg.maximin_weighted_first)
    return out[:k].copy()


# ---------------------------------------------------------------------------
# stage 4 (metrics.hpp:14-57)


@dataclass
class MappingResult:
    """quant::MappingResult (metrics.hpp:14-22)."""
    indices: np.ndarray     # (P,) uint32 (or uint8 when requested)
    quantized: np.ndarray   # (H, W, 3) uint8
    mean_sq_dist: float
    ndc: int = 0


def map_pixels(image, palette, index_bytes: int = 4,
               ctx: Optional[cabi.Context] = None) -> MappingResult:
    """quant::map_pixels (metrics.hpp:28, metrics.cpp:15-55)."""
    ctx = ctx or cabi.default_context()
    pal = np.ascontiguousarray(np.asarray(palette, np.float64).reshape(-1, 3))
    arr, w, h = _pixels(image)
    P = w * h
    k = pal.shape[0]
    if k == 0:
        raise ValueError("map_pixels: empty palette")
    if P == 0:
        raise ValueError("map_pixels: empty image")
    idx = np.empty(P, np.uint8 if index_bytes == 1 else np.uint32)
    q = np.empty((h, w, 3) if h > 1 or isinstance(image, RawImage) else (P, 3), np.uint8)
    mse, ndc = ctx.map_raw(arr, P, pal, k, idx, index_bytes, q, with_ndc=True)
    return MappingResult(idx, q, mse, ndc)


def mse(a, b) -> float:
    """metrics.cpp:57-69 (host helper, integer exact)."""
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    if a.shape != b.shape:
        raise ValueError("mse: image dimensions differ")
    if a.size == 0:
        raise ValueError("mse: empty images")
    return float(((a - b) ** 2).sum()) / float(a.size // 3)


def psnr_from_mse(mse_value: float) -> float:
    """metrics.cpp:71-75."""
    if mse_value < 0.0:
        raise ValueError("psnr_from_mse: negative mse")
    if mse_value == 0.0:
        return math.inf
    return 20.0 * math.log10(255.0 / math.sqrt(mse_value))


@dataclass
class QuantReport:
    """quant::QuantReport (metrics.hpp:37-57) with the frozen CSV/JSON formats
    of metrics.cpp:96-150."""
    image: str = ""
    method: str = ""
    k_requested: int = 0
    k_actual: int = 0
    run: int = 0
    seed: int = 0
    sampling: str = "unique"
    mse: float = 0.0
    psnr: float = 0.0
    iterations: int = 0
    ndc_per_point_iter: float = 0.0
    time_ms: float = 0.0
    flags: list = field(default_factory=list)

    @staticmethod
    def csv_header() -> str:
        return ("image,method,k,run,seed,sampling,mse,psnr,iterations,ndc_per_point_iter,"
                "time_ms,actual_k,flags")

    def csv_row(self) -> str:
        def f(spec, v):
            return spec % v
        mse_s = "nan" if math.isnan(self.mse) else f("%.6f", self.mse)
        if math.isinf(self.psnr):
            psnr_s = "inf"
        elif math.isnan(self.psnr):
            psnr_s = "nan"
        else:
            psnr_s = f("%.4f", self.psnr)
        return ",".join([self.image, self.method, str(self.k_requested), str(self.run),
                         str(self.seed), self.sampling, mse_s, psnr_s, str(self.iterations),
                         f("%.4f", self.ndc_per_point_iter), f("%.3f", self.time_ms),
                         str(self.k_actual), ";".join(self.flags)])

    def to_json(self) -> str:
        return json.dumps({
            "image": self.image, "method": self.method, "k": self.k_requested,
            "actual_k": self.k_actual, "run": self.run, "seed": self.seed,
            "sampling": self.sampling, "mse": self.mse,
            "psnr": "inf" if math.isinf(self.psnr) else self.psnr,
            "iterations": self.iterations, "ndc_per_point_iter": self.ndc_per_point_iter,
            "time_ms": self.time_ms, "flags": list(self.flags)}, indent=2)


# ---------------------------------------------------------------------------
# pipeline (pipeline.hpp:19-53)

PRECLUSTER_TOKENS = ["mc", "ott", "oct", "wan", "wu", "bs"]
INIT_TOKENS = ["fgy", "lbg", "mmx", "den", "var", "sff", "kpp"]
DEVICE_INITS = {"mmx": cabi.INIT_MAXIMIN, "kpp": cabi.INIT_KMEANSPP}


@dataclass
class MethodSpec:
    """quant::MethodSpec (pipeline.hpp:19-24)."""
    refine: bool = False
    base: str = ""

    def token(self) -> str:
        return "wsm-" + self.base if self.refine else self.base


def parse_method(method: str, init: str = "") -> MethodSpec:
    """pipeline.cpp:20-45 (token grammar and messages)."""
    spec = MethodSpec()
    if method == "wsm":
        spec.refine, spec.base = True, (init or "fgy")
    elif method.startswith("wsm-"):
        if init:
            raise ValueError(f"method '{method}' already names its initializer; drop --init")
        spec.refine, spec.base = True, method[4:]
    else:
        if init:
            raise ValueError(f"--init only applies to wsm methods, not '{method}'")
        spec.refine, spec.base = False, method
    if spec.refine:
        if spec.base not in INIT_TOKENS and spec.base not in PRECLUSTER_TOKENS:
            raise ValueError(f"unknown initializer '{spec.base}' "
                             "(expected fgy|lbg|mmx|den|var|sff|kpp|mc|ott|oct|wan|wu|bs)")
    elif spec.base not in PRECLUSTER_TOKENS:
        raise ValueError(f"unknown method '{method}' (expected mc|ott|oct|wan|wu|bs, wsm, or wsm-<init>)")
    return spec


def all_method_tokens() -> list[str]:
    """pipeline.cpp:47-52."""
    return PRECLUSTER_TOKENS + ["wsm-" + t for t in INIT_TOKENS] + ["wsm-" + t for t in PRECLUSTER_TOKENS]


@dataclass
class QuantizeConfig:
    """quant::QuantizeConfig (pipeline.hpp:33-40), the reference's fields.
    ``index_bytes`` (1 or 4) is this build's option for the mapping indices."""
    method: MethodSpec = field(default_factory=lambda: parse_method("wsm-mmx"))
    k: int = 8
    sampling: str = "unique"
    seed: int = 1
    term: Termination = field(default_factory=Termination)
    record_history: bool = False
    index_bytes: int = 4


@dataclass
class QuantizeResult:
    """quant::QuantizeResult (pipeline.hpp:42-48)."""
    palette: np.ndarray
    mapping: MappingResult
    state: ClusterState
    report: QuantReport
    substrate_points: int = 0
    stage_ms: dict = field(default_factory=dict)


def run_quantize(image, config: QuantizeConfig, ctx: Optional[cabi.Context] = None,
                 init_centers=None) -> QuantizeResult:
    """quant::run_quantize (pipeline.hpp:53, pipeline.cpp:81-164) for the
    device path: every sampling mode (none | 2to1 | unique | both), refined
    methods wsm-mmx / wsm-kpp, or any wsm-<x> whose k initial centres are
    supplied as ``init_centers`` (the C++ overload run_quantize(image, config,
    init_centers)). ``config.record_history`` is forwarded to the engine
    (pipeline.cpp:126-130): the stages then run as separate device calls."""
    ctx = ctx or cabi.default_context()
    arr, w, h = _pixels(image)
    P = w * h
    if P == 0:
        raise ValueError("run_quantize: empty image")
    if config.k < 1:
        raise ValueError("run_quantize: k must be at least 1")
    sampling = SAMPLING_CODES[parse_sampling_mode(config.sampling)]
    if not config.method.refine:
        raise ValueError("run_quantize: standalone preclusterers are outside the device path")
    k = int(config.k)
    if init_centers is not None:
        kind = cabi.INIT_GIVEN
        init = np.ascontiguousarray(np.asarray(init_centers, np.float64).reshape(-1, 3))
        if init.shape[0] != k:
            raise ValueError("run_quantize: init_centers must hold k centres")
    elif config.method.base in DEVICE_INITS:
        kind = DEVICE_INITS[config.method.base]
        init = None
    else:
        raise ValueError(f"run_quantize: initializer '{config.method.base}' is outside the device "
                         "path; supply init_centers")
    if config.record_history:
        return _run_quantize_history(arr, w, h, config, kind, init, ctx)
    term = _term_struct(config.term, False)
    cfg = cabi.QuantizeCfg(kind, k, int(config.seed), term, int(config.index_bytes), sampling, w, h)
    limit = term.fixed_iterations if term.fixed_iterations > 0 else term.max_iterations
    palette = np.empty((k, 3), np.float64)
    labels = np.empty(P, np.uint32)  # the substrate: <= 2^24 colours, or every sampled pixel
    sse = np.zeros(limit, np.float64)
    idx = np.empty(P, np.uint8 if config.index_bytes == 1 else np.uint32)
    q = np.empty((h, w, 3), np.uint8)
    t0 = time.perf_counter()
    st = ctx.quantize_raw(arr, P, cfg, init, palette, labels, sse, idx, q)
    t1 = time.perf_counter()
    n = int(st.n_unique)
    it = st.lloyd.iterations
    state = ClusterState(palette.copy(), labels[:n].copy(), sse[:it].copy(), it,
                         int(st.lloyd.ndc_total), int(st.lloyd.repair_count), [],
                         int(st.lloyd.flagged_total), int(st.lloyd.swept_total))
    mapping = MappingResult(idx, q, float(st.mean_sq_dist), int(st.map_ndc))
    rep = QuantReport(method=config.method.token(), k_requested=k, k_actual=k,
                      seed=int(config.seed), sampling=config.sampling, mse=mapping.mean_sq_dist,
                      psnr=psnr_from_mse(mapping.mean_sq_dist), iterations=it,
                      ndc_per_point_iter=state.ndc_per_point_iter(n),
                      time_ms=(t1 - t0) * 1e3)
    if state.repair_count > 0:
        rep.flags.append(f"repairs:{state.repair_count}")
    return QuantizeResult(palette, mapping, state, rep, n,
                          dict(histogram=st.ms_histogram, init=st.ms_init, lloyd=st.ms_lloyd,
                               map=st.ms_map))


def _run_quantize_history(arr, w, h, config: QuantizeConfig, kind, init, ctx) -> QuantizeResult:
    """run_quantize with record_history: histogram -> initialiser -> wsm (with
    per-iteration snapshots) -> mapping as separate device calls."""
    if hasattr(arr, "data_ptr") and not isinstance(arr, np.ndarray):
        arr = arr.cpu().numpy()
    img = np.ascontiguousarray(arr, np.uint8).reshape(h, w, 3)
    sub = config.sampling in ("2to1", "both")
    dedup = config.sampling in ("unique", "both")
    sampled = img[::2, ::2] if sub else img
    t0 = time.perf_counter()
    hist = build_histogram(sampled, config.seed, ctx=ctx)
    if init is None:
        sc = SeedConfig(k=int(config.k), seed=int(config.seed))
        init = init_maximin(hist, sc, ctx=ctx) if kind == cabi.INIT_MAXIMIN else init_kmeanspp(hist, sc, ctx=ctx)
    opt = ClusterOptions(term=config.term, record_history=True)
    if dedup:
        st = wsm_hist(hist, init, opt, ctx=ctx)
        n = hist.size()
    else:
        px = pack_colors(sampled)
        st = wsm_counts(px, np.ones(px.size, np.uint32), px.size, init, opt, ctx=ctx)
        n = px.size
    mapping = map_pixels(img, st.centers, index_bytes=config.index_bytes, ctx=ctx)
    t1 = time.perf_counter()
    k = int(config.k)
    rep = QuantReport(method=config.method.token(), k_requested=k, k_actual=k, seed=int(config.seed),
                      sampling=config.sampling, mse=mapping.mean_sq_dist, psnr=psnr_from_mse(mapping.mean_sq_dist),
                      iterations=st.iterations, ndc_per_point_iter=st.ndc_per_point_iter(n), time_ms=(t1 - t0) * 1e3)
    if st.repair_count > 0:
        rep.flags.append(f"repairs:{st.repair_count}")
    return QuantizeResult(st.centers.copy(), mapping, st, rep, n)
