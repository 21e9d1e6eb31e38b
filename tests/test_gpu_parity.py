"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle and
the reference library, on seeded inputs, golden fixtures and edge cases.

Bar:
  histogram            colours, counts, first index: bit-exact, first-occurrence order
  init (mmx, kpp)      centres bit-exact (any P)
  Lloyd                per-iteration labels, iterations, NDC, repairs: bit-exact vs the
                       reference; centres and SSE trace bit-exact vs the exact-moment
                       oracle; vs the reference: centres bit-exact when P is a power of
                       two (else |d| <= 1e-9), SSE rel <= 1e-12
  mapping              indices + quantized pixels bit-exact; MSE bit-exact vs the
                       exact-moment oracle, rel <= 1e-12 vs the reference
"""
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import UPDATE_EXACT, UPDATE_REFERENCE
from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS, synth_image

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def packed(colors_rgb):
    return quant.pack_colors(colors_rgb)


def gpu_hist(ctx, img):
    return quant.build_histogram(img, ctx=ctx)


def assert_lloyd_equal(dev, ora, P, ref=None):
    assert dev.iterations == ora.iterations
    assert dev.ndc_total == ora.ndc_total
    assert dev.repair_count == ora.repairs
    assert np.array_equal(dev.memberships, ora.labels)
    assert np.array_equal(dev.centers.view(np.uint64), ora.centers.view(np.uint64))
    assert np.array_equal(dev.sse_trace.view(np.uint64), ora.sse_trace.view(np.uint64))
    if dev.history:
        hl = np.stack([h.memberships for h in dev.history])
        assert np.array_equal(hl, ora.hist_labels)
    if ref is not None:
        assert dev.iterations == ref.iterations and dev.ndc_total == ref.ndc_total
        assert np.array_equal(dev.memberships, ref.labels)
        if P & (P - 1) == 0:
            assert np.array_equal(dev.centers, ref.centers)
        else:
            assert np.max(np.abs(dev.centers - ref.centers)) <= 1e-9
        assert np.max(np.abs(dev.sse_trace - ref.sse_trace) / np.maximum(ref.sse_trace, 1e-300)) <= 1e-12


# ---------------------------------------------------------------------------
# stage 1

@pytest.mark.parametrize("case", ["ref_order", "single", "tail15", "noise64", "cfg1", "cfg2",
                                  "few_colours", "unaligned"])
def test_histogram_bit_exact(ctx, oracle, case):
    if case == "ref_order":  # tests/test_histogram.cpp:102-118
        img = np.array([(10, 20, 30), (200, 100, 50), (10, 20, 30), (0, 0, 0), (200, 100, 50),
                        (10, 20, 30)], np.uint8)
    elif case == "single":
        img = np.array([[7, 8, 9]], np.uint8)
    elif case == "tail15":
        img = np.random.default_rng(1).integers(0, 4, (15, 3), dtype=np.uint8)
    elif case == "noise64":
        img = np.random.default_rng(99).integers(0, 256, (64, 64, 3), dtype=np.uint8)
    elif case == "few_colours":
        img = (np.random.default_rng(5).integers(0, 3, (300, 301, 3)) * 100).astype(np.uint8)
    elif case == "unaligned":
        base = synth_image(97, 31, 3, nblobs=4)
        buf = np.zeros(base.size + 5, np.uint8)
        buf[5:] = base.reshape(-1)
        img = buf[5:]  # 5-byte offset: exercises the scalar path
    else:
        img = CONFIGS[case].image()
    h = gpu_hist(ctx, img)
    c, n, f = oracle.histogram(img)
    assert np.array_equal(h.packed, c)
    assert np.array_equal(h.counts, n)
    assert np.array_equal(h.first, f)
    P = img.size // 3
    assert np.array_equal(h.weights, oracle.weights(n, P))
    assert int(h.counts.sum()) == P


def test_histogram_device_pointers(ctx, oracle):
    torch = pytest.importorskip("torch")
    img = CONFIGS["cfg2"].image()
    d = torch.from_numpy(img).cuda()
    P = img.shape[0] * img.shape[1]
    cap = min(P, 1 << 24)
    col = torch.empty(cap, dtype=torch.int32, device="cuda")
    cnt = torch.empty(cap, dtype=torch.int32, device="cuda")
    n = ctx.histogram_raw(d, P, col, cnt)
    torch.cuda.synchronize()
    c, k, _ = oracle.histogram(img)
    assert n == c.size
    assert np.array_equal(col[:n].cpu().numpy().view(np.uint32), c)
    assert np.array_equal(cnt[:n].cpu().numpy().view(np.uint32), k)


@pytest.mark.parametrize("case", ["2048sq", "odd2049", "unaligned_large", "few_large", "flat_large",
                                  "one_bucket", "two_colours"])
def test_histogram_large_images(ctx, oracle, case):
    # P >= 2^22: the colour-bucketed partition (hist.cu: part_count ->
    # part_scatter -> bucket_agg in shared memory), first-occurrence bitmap,
    # pixel-order emit; odd sizes and unaligned buffers take the scalar paths,
    # a flat image puts every pixel in one bucket and one shared-memory slot
    rng = np.random.default_rng(2024)
    if case == "2048sq":
        img = synth_image(2048, 2048, 11, nblobs=20, sigma=20.0, noise=0.3)
    elif case == "odd2049":
        img = synth_image(2049, 2049, 12, nblobs=20, sigma=20.0, noise=0.3)
    elif case == "unaligned_large":
        base = synth_image(2050, 2047, 13, nblobs=10, sigma=25.0, noise=0.5)
        buf = np.zeros(base.size + 7, np.uint8)
        buf[7:] = base.reshape(-1)
        img = buf[7:]
    elif case == "flat_large":
        img = np.full((2048, 2049, 3), 77, np.uint8)
    elif case == "one_bucket":  # r = 0, g < 64: bucket 0 holds every pixel
        img = rng.integers(0, 256, (2048, 2050, 3)).astype(np.uint8)
        img[..., 0] = 0
        img[..., 1] &= 63
    elif case == "two_colours":
        img = np.where(rng.random((2051, 2048, 1)) < 0.999, 10, 200).astype(np.uint8).repeat(3, axis=2)
    else:
        img = (rng.integers(0, 4, (2100, 2000, 3)) * 60).astype(np.uint8)
    assert img.size // 3 >= (1 << 22)
    h = gpu_hist(ctx, img)
    c, n, f = oracle.histogram(img)
    assert np.array_equal(h.packed, c)
    assert np.array_equal(h.counts, n)
    assert np.array_equal(h.first, f)
    # the tables are clean for the next (small) call
    small = synth_image(64, 48, 3, nblobs=3)
    hs = gpu_hist(ctx, small)
    cs, ns, _ = oracle.histogram(small)
    assert np.array_equal(hs.packed, cs) and np.array_equal(hs.counts, ns)


def test_histogram_repeated_calls_keep_table_clean(ctx, oracle):
    for seed in range(3):
        img = synth_image(200, 150, 40 + seed, nblobs=5, sigma=9.0, noise=0.05)
        h = gpu_hist(ctx, img)
        c, n, f = oracle.histogram(img)
        assert np.array_equal(h.packed, c) and np.array_equal(h.counts, n)


# ---------------------------------------------------------------------------
# init

@pytest.mark.parametrize("w,h,K,seed", [(40, 40, 8, 3), (64, 64, 32, 11), (512, 512, 64, 5),
                                        (300, 200, 256, 9), (768, 512, 128, 4)])
def test_init_bit_exact(ctx, oracle, w, h, K, seed):
    img = synth_image(w, h, seed, nblobs=10, sigma=15.0, noise=0.02)
    P = w * h
    hist = gpu_hist(ctx, img)
    c, n = hist.packed, hist.counts
    kpp = quant.init_kmeanspp(hist, quant.SeedConfig(k=K, seed=seed), ctx=ctx)
    assert np.array_equal(kpp, oracle.init_kmeanspp(c, n, P, K, seed))
    mmx = quant.init_maximin(hist, quant.SeedConfig(k=K, seed=seed), ctx=ctx)
    assert np.array_equal(mmx, oracle.init_maximin(c, n, P, K, seed))
    mmx_u = quant.init_maximin(hist, quant.SeedConfig(k=K, seed=seed, maximin_weighted_first=False), ctx=ctx)
    assert np.array_equal(mmx_u, oracle.init_maximin(c, n, P, K, seed, weighted_first=False))


def test_init_validation(ctx):
    img = np.array([[1, 2, 3], [4, 5, 6]], np.uint8)
    hist = gpu_hist(ctx, img)
    with pytest.raises(ValueError, match=r"k \(3\) exceeds distinct colors \(2\)"):
        quant.init_maximin(hist, quant.SeedConfig(k=3), ctx=ctx)
    with pytest.raises(ValueError, match="k must be at least 1"):
        quant.init_kmeanspp(hist, quant.SeedConfig(k=0), ctx=ctx)


# ---------------------------------------------------------------------------
# Lloyd

def test_lloyd_reference_cases(ctx, oracle):
    with open(os.path.join(GOLD, "ref_cases.json")) as f:
        cases = json.load(f)
    for c in cases:
        colors = np.array(c["hist_colors"], np.uint32)
        counts = np.array(c["hist_counts"], np.uint32)
        init = np.array([float.fromhex(v) for v in c["init_centers"]]).reshape(-1, 3)
        dev = quant.wsm_counts(colors, counts, 1600, init, quant.ClusterOptions(record_history=True), ctx=ctx)
        ora = oracle.wsm(colors, counts, 1600, init, mode=UPDATE_EXACT, history=True)
        assert_lloyd_equal(dev, ora, 1600)
        assert dev.iterations == c["iterations"] and dev.ndc_total == c["ndc_total"]
        assert dev.memberships.tolist() == c["labels"]
        assert [h.memberships.tolist() for h in dev.history] == c["history_labels"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_lloyd_configs(ctx, oracle, name):
    cfg = CONFIGS[name]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = gpu_hist(ctx, img)
    c, n = hist.packed, hist.counts
    init = (oracle.init_kmeanspp if cfg.init == "kpp" else oracle.init_maximin)(c, n, P, cfg.k, cfg.seed)
    dev = quant.wsm_counts(c, n, P, init, quant.ClusterOptions(record_history=True), ctx=ctx)
    ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT, history=True)
    assert_lloyd_equal(dev, ora, P)


def test_lloyd_vs_reference_library(ctx, oracle, reflib):
    for seed, K, kind, (w, h) in [(21, 48, "kpp", (256, 256)), (22, 100, "mmx", (320, 240))]:
        img = synth_image(w, h, seed, nblobs=12, sigma=14.0, noise=0.03)
        P = w * h
        hist = gpu_hist(ctx, img)
        c, n = hist.packed, hist.counts
        init = reflib.init(kind, c, n, P, K, seed)
        dev = quant.wsm_counts(c, n, P, init, quant.ClusterOptions(record_history=True), ctx=ctx)
        ref = reflib.wsm(c, n, P, init, history=True)
        ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT, history=True)
        assert_lloyd_equal(dev, ora, P, ref)
        hl = np.stack([x.memberships for x in dev.history])
        assert np.array_equal(hl, ref.hist_labels)


@pytest.mark.parametrize("K", [300, 520])
def test_lloyd_wide_k(ctx, oracle, K):
    img = synth_image(256, 128, 77, nblobs=30, sigma=18.0, noise=0.05)
    P = 256 * 128
    hist = gpu_hist(ctx, img)
    c, n = hist.packed, hist.counts
    init = oracle.init_maximin(c, n, P, K, 77)
    opts = quant.ClusterOptions(quant.Termination(max_iterations=12), record_history=True)
    dev = quant.wsm_counts(c, n, P, init, opts, ctx=ctx)
    ora = oracle.wsm(c, n, P, init, max_it=12, mode=UPDATE_EXACT, history=True)
    assert_lloyd_equal(dev, ora, P)


def test_lloyd_fixed_iterations_and_eps0(ctx, oracle):
    img = CONFIGS["cfg1"].image()
    P = img.shape[0] * img.shape[1]
    hist = gpu_hist(ctx, img)
    c, n = hist.packed, hist.counts
    init = oracle.init_maximin(c, n, P, 16, 1)
    dev = quant.wsm_counts(c, n, P, init, quant.ClusterOptions(quant.Termination(fixed_iterations=7)), ctx=ctx)
    ora = oracle.wsm(c, n, P, init, fixed_it=7, mode=UPDATE_EXACT)
    assert dev.iterations == 7
    assert_lloyd_equal(dev, ora, P)
    dev = quant.wsm_counts(c, n, P, init, quant.ClusterOptions(quant.Termination(epsilon=0.0, max_iterations=40)), ctx=ctx)
    ora = oracle.wsm(c, n, P, init, eps=0.0, max_it=40, mode=UPDATE_EXACT)
    assert_lloyd_equal(dev, ora, P)


def test_lloyd_empty_cluster_repair(ctx, oracle):
    # tests/test_kmeans.cpp:210-223: two points, two identical centres -> one repair
    colors = packed(np.array([[0, 0, 0], [9, 0, 0]], np.uint8))
    counts = np.array([1, 1], np.uint32)
    init = np.array([[5, 0, 0], [5, 0, 0]], float)
    dev = quant.wsm_counts(colors, counts, 2, init, ctx=ctx)
    ora = oracle.wsm(colors, counts, 2, init, mode=UPDATE_EXACT)
    assert dev.repair_count == 1 and dev.iterations == 1 and dev.sse_trace[0] == 0.0
    assert_lloyd_equal(dev, ora, 2)
    # many empty clusters: adversarial init far from the data
    img = synth_image(64, 64, 5, nblobs=3, sigma=4.0)
    hist = gpu_hist(ctx, img)
    init = np.array([[250.0, 250.0, 250.0 - i] for i in range(12)])
    dev = quant.wsm_counts(hist.packed, hist.counts, 4096, init, ctx=ctx)
    ora = oracle.wsm(hist.packed, hist.counts, 4096, init, mode=UPDATE_EXACT)
    assert dev.repair_count > 0
    assert_lloyd_equal(dev, ora, 4096)


def test_lloyd_termination_rules(ctx, oracle):
    # tests/test_kmeans.cpp:246-262: perfect init stops at iteration 1 (sse 0);
    # k = 1 needs a second iteration to observe the zero drop
    rng = np.random.default_rng(11)
    keys = rng.choice(1 << 24, 64, replace=False).astype(np.uint32)
    counts = np.ones(64, np.uint32)
    pts = quant.unpack_colors(keys)
    dev = quant.wsm_counts(keys, counts, 64, pts, ctx=ctx)
    assert dev.iterations == 1 and dev.sse_trace[-1] == 0.0
    dev1 = quant.wsm_counts(keys, counts, 64, np.zeros((1, 3)), ctx=ctx)
    assert dev1.iterations == 2 and dev1.sse_trace[0] >= dev1.sse_trace[1]


def test_lloyd_validation_messages(ctx):
    colors = packed(np.array([[0, 0, 0], [1, 1, 1]], np.uint8))
    counts = np.array([1, 1], np.uint32)
    three = np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2]], float)
    with pytest.raises(ValueError, match=r"clustering: k \(3\) exceeds number of points \(2\)"):
        quant.wsm_counts(colors, counts, 2, three, ctx=ctx)
    with pytest.raises(ValueError, match="negative epsilon"):
        quant.wsm_counts(colors, counts, 2, three[:1], quant.ClusterOptions(quant.Termination(epsilon=-1.0)), ctx=ctx)
    with pytest.raises(ValueError, match="max_iterations < 1"):
        quant.wsm_counts(colors, counts, 2, three[:1], quant.ClusterOptions(quant.Termination(max_iterations=0)), ctx=ctx)
    with pytest.raises(ValueError, match="weights must be positive"):
        quant.wsm_counts(colors, np.array([1, 0], np.uint32), 2, three[:1], ctx=ctx)


def test_lloyd_device_resident_buffers(ctx, oracle):
    torch = pytest.importorskip("torch")
    cfg = CONFIGS["cfg2"]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = gpu_hist(ctx, img)
    c, n = hist.packed, hist.counts
    init = oracle.init_kmeanspp(c, n, P, 64, 3)
    dc = torch.from_numpy(c.view(np.int32)).cuda()
    dn = torch.from_numpy(n.view(np.int32)).cuda()
    di = torch.from_numpy(init.copy()).cuda()
    cen = torch.empty((64, 3), dtype=torch.float64, device="cuda")
    lab = torch.empty(c.size, dtype=torch.int32, device="cuda")
    sse = np.zeros(100)
    st = ctx.lloyd_raw(dc, dn, c.size, P, di, 64, cabi.Term(1e-3, 100, 0, 0), cen, lab, sse)
    ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT)
    assert st.iterations == ora.iterations
    assert np.array_equal(cen.cpu().numpy(), ora.centers)
    assert np.array_equal(lab.cpu().numpy().view(np.uint32), ora.labels)


# ---------------------------------------------------------------------------
# mapping

@pytest.mark.parametrize("K,ib", [(8, 4), (32, 1), (256, 4), (256, 1), (300, 4)])
def test_map_bit_exact(ctx, oracle, reflib, K, ib):
    img = synth_image(160, 120, 31 + K, nblobs=9, sigma=16.0, noise=0.05)
    rng = np.random.default_rng(K)
    pal = rng.random((K, 3)) * 255.0
    m = quant.map_pixels(img, pal, index_bytes=ib, ctx=ctx)
    idx, q, mse_e, ndc_e = oracle.map_pixels(img, pal, mode=UPDATE_EXACT)
    assert np.array_equal(m.indices.astype(np.uint32), idx)
    assert np.array_equal(m.quantized.reshape(-1, 3), q)
    assert m.mean_sq_dist == mse_e
    assert m.ndc == ndc_e
    i2, q2, mse_r, ndc_r = reflib.map_pixels(img, 160, 120, pal)
    assert np.array_equal(m.indices.astype(np.uint32), i2)
    assert abs(m.mean_sq_dist - mse_r) <= 1e-12 * mse_r
    assert m.ndc == ndc_r  # MappingResult::ndc (metrics.cpp:36-48)


@pytest.mark.parametrize("w,h,K,ib", [(1031, 1025, 256, 4), (1024, 1024, 64, 1), (1100, 977, 300, 4)])
def test_map_large_streaming(ctx, oracle, w, h, K, ib):
    # P >= 2^20: the vectorised 16-pixel path of pixel_kernel; 1031x1025 and
    # 1100x977 leave a remainder for its scalar tail
    img = synth_image(w, h, 5 + K, nblobs=12, sigma=18.0, noise=0.2)
    rng = np.random.default_rng(w + K)
    pal = rng.random((K, 3)) * 255.0
    m = quant.map_pixels(img, pal, index_bytes=ib, ctx=ctx)
    idx, q, mse_e, ndc_e = oracle.map_pixels(img, pal, mode=UPDATE_EXACT)
    assert np.array_equal(m.indices.astype(np.uint32), idx)
    assert np.array_equal(m.quantized.reshape(-1, 3), q)
    assert m.mean_sq_dist == mse_e
    assert m.ndc == ndc_e


def test_map_reference_cases(ctx):
    # tests/test_metrics.cpp:66-92
    img = np.array([[[1, 0, 0]]], np.uint8)
    m = quant.map_pixels(img, np.array([[2, 0, 0], [0, 0, 0]], float), ctx=ctx)
    assert m.indices[0] == 0
    m = quant.map_pixels(img, np.array([[0, 0, 0], [2, 0, 0]], float), ctx=ctx)
    assert m.indices[0] == 0
    img = np.array([[[0, 0, 0], [1, 0, 0]]], np.uint8)
    m = quant.map_pixels(img, np.array([[0.5, 0, 0]]), ctx=ctx)
    assert m.mean_sq_dist == pytest.approx(0.25, rel=1e-12)
    assert m.quantized.reshape(-1, 3)[0, 0] == 1
    with pytest.raises(ValueError, match="empty palette"):
        quant.map_pixels(img, np.zeros((0, 3)), ctx=ctx)


def test_map_ties_to_lowest_index(ctx, oracle):
    # integer palette on the colour grid: many exact FP64 ties
    rng = np.random.default_rng(8)
    pal = rng.integers(0, 256, (64, 3)).astype(float)
    pal[10] = pal[3]  # duplicate entry: must never be chosen over 3
    img = rng.integers(0, 256, (128, 128, 3), dtype=np.uint8)
    m = quant.map_pixels(img, pal, ctx=ctx)
    idx, _, mse_e, ndc_e = oracle.map_pixels(img, pal, mode=UPDATE_EXACT)
    assert np.array_equal(m.indices, idx)
    assert not np.any(m.indices == 10)
    assert m.mean_sq_dist == mse_e
    assert m.ndc == ndc_e  # cutoff ties (D == 4 d2 exactly) are evaluated: '>' break


# ---------------------------------------------------------------------------
# pipeline

def test_pipeline_golden_sweep_rows(ctx):
    with open(os.path.join(GOLD, "sweep_a_rows.csv")) as f:
        rows = f.read().strip().split("\n")[1:]
    with open(os.path.join(GOLD, "wu_init.json")) as f:
        wu = json.load(f)
    got = []
    for img_seed in (61, 62):
        img = np.fromfile(os.path.join(GOLD, f"acc_{img_seed}.rgb"), np.uint8).reshape(40, 40, 3)
        for method in ("wsm-kpp", "wsm-wu"):
            for run in (0, 1):
                cfg = quant.QuantizeConfig(method=quant.parse_method(method), k=8, seed=3 + run)
                init = np.array(wu[str(img_seed)]) if method == "wsm-wu" else None
                r = quant.run_quantize(img, cfg, ctx=ctx, init_centers=init)
                rep = r.report
                rep.image, rep.run, rep.time_ms = f"acc_{img_seed}.ppm", run, 0.0
                got.append(rep.csv_row())
    assert sorted(got) == sorted(r for r in rows if ",wu," not in r)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_pipeline_vs_reference(ctx, oracle, reflib, name):
    cfg = CONFIGS[name]
    img = cfg.image()
    h, w = img.shape[:2]
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-" + cfg.init), k=cfg.k, seed=cfg.seed)
    r = quant.run_quantize(img, qc, ctx=ctx)
    ref = reflib.run_quantize(img, w, h, "wsm-" + cfg.init, cfg.k, cfg.seed)
    assert r.report.iterations == ref["iterations"]
    assert r.report.ndc_per_point_iter == ref["ndc_per_point_iter"]
    assert np.array_equal(r.palette, ref["palette"])  # P = 2^18
    assert abs(r.report.mse - ref["mse"]) <= 1e-12 * ref["mse"]
    # mapping outputs bit-exact vs the exact oracle on the same palette
    idx, q, mse_e, ndc_e = oracle.map_pixels(img, r.palette, mode=UPDATE_EXACT)
    assert np.array_equal(r.mapping.indices, idx)
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), q)
    assert r.report.mse == mse_e
    assert r.mapping.ndc == ndc_e


# ---------------------------------------------------------------------------
# coarse histogram (precluster.cpp:13-47): exact integers, both overloads

@pytest.mark.parametrize("w,h,noise", [(160, 120, 0.05), (1031, 1025, 0.3), (1, 1, 0.0)])
def test_coarse_histogram_vs_reference(ctx, oracle, reflib, w, h, noise):
    img = synth_image(w, h, 11 + w, nblobs=9, sigma=14.0, noise=noise)
    ch = quant.build_coarse_histogram(img, ctx=ctx)
    ref_px = reflib.coarse_histogram(rgb=img)
    got = np.stack([ch.count.view(np.int64), ch.sum_r, ch.sum_g, ch.sum_b, ch.sum_sq])
    assert np.array_equal(got, ref_px)
    hist = quant.build_histogram(img, ctx=ctx)
    chw = quant.build_coarse_histogram(hist, ctx=ctx)
    got_w = np.stack([chw.count.view(np.int64), chw.sum_r, chw.sum_g, chw.sum_b, chw.sum_sq])
    assert np.array_equal(got_w, reflib.coarse_histogram(colors=hist.packed, counts=hist.counts))
    assert np.array_equal(got_w, oracle.coarse_histogram(hist.packed, hist.counts))
    assert int(ch.count.sum()) == w * h


def test_coarse_histogram_errors(ctx):
    with pytest.raises(ValueError, match="build_coarse_histogram: no pixels"):
        quant.build_coarse_histogram(np.zeros((0, 3), np.uint8), ctx=ctx)
    empty = quant.WeightedHistogram(colors=np.zeros((0, 3)), weights=np.zeros(0), counts=np.zeros(0, np.uint32),
                                    source_pixel_count=0, packed=np.zeros(0, np.uint32))
    with pytest.raises(ValueError, match="build_coarse_histogram: empty histogram"):
        quant.build_coarse_histogram(empty, ctx=ctx)
