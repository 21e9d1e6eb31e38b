"""The general exact-FP64 device engine (csrc/exact.cu) against the reference
library itself (oracle/_ref): wsm with arbitrary positive weights and real
points, kmeans_full, and the kmeans.hpp / init.hpp helpers. Bar: every output
bit-identical (labels, centres, sse_trace, iterations, ndc_total, repairs,
history), since the engine reproduces the reference's sequential FP64 sums
(kmeans.cpp:107-122, 192-260) in order.

Scenarios follow the reference's own unit tests (tests/test_kmeans.cpp,
tests/test_init.cpp): random weights, adversarial initial centres, duplicate
points, coincident centres, repair fallbacks.
"""
import numpy as np
import pytest

from paper_1101_0395_b200 import quant

pytestmark = pytest.mark.gpu


def distinct_colors(rng, n):
    keys = rng.choice(1 << 24, size=n, replace=False)
    return np.stack([(keys >> 16) & 255, (keys >> 8) & 255, keys & 255], 1).astype(np.float64)


def random_weights(rng, n):
    w = 0.05 + rng.random(n)
    return w / w.sum()


def same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.uint64), b.view(np.uint64))
    return np.array_equal(a, b)


def check_state(st, ref):
    assert st.iterations == ref.iterations
    assert st.ndc_total == ref.ndc_total
    assert st.repair_count == ref.repairs
    assert same(st.memberships, ref.labels)
    assert same(st.centers, ref.centers)
    assert same(st.sse_trace, ref.sse_trace)
    if ref.hist_labels is not None:
        assert len(st.history) == ref.iterations
        for it, snap in enumerate(st.history):
            assert same(snap.memberships, ref.hist_labels[it])
            assert same(snap.centers, ref.hist_centers[it])


@pytest.mark.parametrize("trial", range(6))
def test_wsm_random_weights(ctx, reflib, trial):
    # tests/test_kmeans.cpp:193-208: random weights, adversarial initial colours
    rng = np.random.default_rng(888 + trial)
    n = 100 + int(rng.integers(0, 400))
    k = 2 + int(rng.integers(0, 30))
    pts = distinct_colors(rng, n)
    w = random_weights(rng, n)
    init = distinct_colors(rng, k)
    opt = quant.ClusterOptions(record_history=True)
    st = quant.wsm(pts, w, init, opt, ctx=ctx)
    ref = reflib.lloyd_general(pts, w, init, history=True)
    check_state(st, ref)
    assert np.all(np.diff(st.sse_trace) <= 0)


def test_wsm_real_valued_points(ctx, reflib):
    rng = np.random.default_rng(5)
    pts = rng.random((700, 3)) * 300.0 - 20.0  # off the 8-bit grid, some negative
    w = random_weights(rng, 700)
    init = pts[rng.choice(700, 24, replace=False)]
    st = quant.wsm(pts, w, init, quant.ClusterOptions(term=quant.Termination(fixed_iterations=12)), ctx=ctx)
    ref = reflib.lloyd_general(pts, w, init, fixed_it=12)
    check_state(st, ref)


def test_wsm_repairs_with_generic_weights(ctx, reflib):
    # many coincident initial centres: empty clusters every early iteration
    rng = np.random.default_rng(17)
    pts = distinct_colors(rng, 300)
    w = random_weights(rng, 300)
    init = np.repeat(pts[:4], 8, axis=0)
    st = quant.wsm(pts, w, init, quant.ClusterOptions(record_history=True), ctx=ctx)
    ref = reflib.lloyd_general(pts, w, init, history=True)
    assert ref.repairs > 0
    check_state(st, ref)


@pytest.mark.parametrize("fixed", [0, 20])
def test_kmeans_full(ctx, reflib, fixed):
    # tests/test_kmeans.cpp:140-151 and 153-191: full scan, no repair, exact NDC
    rng = np.random.default_rng(31 + fixed)
    pts = distinct_colors(rng, 120)
    init = pts[:8]
    opt = quant.ClusterOptions(term=quant.Termination(fixed_iterations=fixed or None), record_history=True)
    st = quant.kmeans_full(pts, init, opt, ctx=ctx)
    ref = reflib.lloyd_general(pts, None, init, fixed_it=fixed, history=True)
    check_state(st, ref)
    assert st.ndc_total == 8 * 120 * st.iterations


def test_kmeans_full_empty_cluster_keeps_centre(ctx, reflib):
    # duplicated points and a centre nobody is nearest to (kmeans.cpp:240-243)
    pts = np.array([[10, 0, 0]] * 3 + [[90, 0, 0]] + [[200, 200, 200]], np.float64)
    init = np.array([[0, 0, 0], [100, 0, 0], [255, 0, 255], [254, 0, 255]], np.float64)
    st = quant.kmeans_full(pts, init, quant.ClusterOptions(term=quant.Termination(fixed_iterations=3)), ctx=ctx)
    ref = reflib.lloyd_general(pts, None, init, fixed_it=3)
    check_state(st, ref)
    assert same(st.centers[2], init[2])  # (254, 0, 255) takes the far point: centre 2 stays empty


def test_weighted_histogram_equals_duplicated_points(ctx):
    # tests/test_kmeans.cpp:287-305
    raw = np.array([[10, 0, 0]] * 3 + [[90, 0, 0]], np.float64)
    hp = np.array([[10, 0, 0], [90, 0, 0]], np.float64)
    init = np.array([[0, 0, 0], [100, 0, 0]], np.float64)
    opt = quant.ClusterOptions(term=quant.Termination(fixed_iterations=3))
    full = quant.kmeans_full(raw, init, opt, ctx=ctx)
    fast = quant.wsm(hp, np.array([0.75, 0.25]), init, opt, ctx=ctx)
    assert np.allclose(fast.sse_trace, full.sse_trace / 4.0, rtol=1e-12, atol=0)
    assert same(fast.centers, full.centers)


def test_compute_sse_both_overloads(ctx, reflib):
    rng = np.random.default_rng(3)
    pts = rng.random((5000, 3)) * 255.0
    w = random_weights(rng, 5000)
    cen = rng.random((40, 3)) * 255.0
    lab = rng.integers(0, 40, 5000).astype(np.uint32)
    assert quant.compute_sse(pts, w, cen, lab, ctx=ctx) == reflib.compute_sse(pts, w, cen, lab)
    assert quant.compute_sse(pts, cen, lab, ctx=ctx) == reflib.compute_sse(pts, None, cen, lab)
    # tests/test_kmeans.cpp:14-21: 0.75 * 1 + 0.25 * 9
    assert quant.compute_sse(np.array([[0, 0, 0], [4, 0, 0]], float), np.array([0.75, 0.25]),
                             np.array([[1, 0, 0]], float), np.array([0, 0], np.uint32), ctx=ctx) == 3.0


@pytest.mark.parametrize("case", ["donor", "fallback", "chain"])
def test_repair_empty_clusters(ctx, reflib, case):
    if case == "donor":  # tests/test_kmeans.cpp:210-223
        pts = np.array([[0, 0, 0], [9, 0, 0]], float)
        w = np.array([0.5, 0.5])
        cen = np.array([[5, 0, 0], [5, 0, 0]], float)
        lab = np.array([0, 0], np.uint32)
    elif case == "fallback":  # every point on its centre: first point of a cluster of size >= 2
        pts = np.array([[3, 3, 3]] * 4 + [[7, 7, 7]], float)
        w = np.full(5, 0.2)
        cen = np.array([[3, 3, 3], [7, 7, 7], [50, 50, 50]], float)
        lab = np.array([0, 0, 0, 0, 1], np.uint32)
    else:  # a donor's own cluster empties: the scan restarts at 0
        rng = np.random.default_rng(9)
        pts = distinct_colors(rng, 64)
        w = random_weights(rng, 64)
        cen = distinct_colors(rng, 12)
        lab = np.zeros(64, np.uint32)
        lab[::2] = 1
    r_ref, c_ref, l_ref = reflib.repair(pts, w, cen, lab)
    c = cen.copy()
    m = lab.copy()
    r = quant.repair_empty_clusters(pts, w, c, m, ctx=ctx)
    assert r == r_ref
    assert same(c, c_ref) and same(m, l_ref)


def test_repair_impossible(ctx):
    pts = np.array([[1, 1, 1]], float)
    with pytest.raises(RuntimeError, match="more clusters than points"):
        quant.repair_empty_clusters(pts, np.array([1.0]), np.array([[1, 1, 1], [2, 2, 2]], float),
                                    np.array([0], np.uint32), ctx=ctx)


@pytest.mark.parametrize("K", [3, 37, 256, 600])
def test_center_table(ctx, reflib, K):
    rng = np.random.default_rng(K)
    cen = np.floor(rng.random((K, 3)) * 6.0) * 40.0  # coarse grid: many distance ties, coincident centres
    t = quant.build_center_distance_table(cen, ctx=ctx)
    d, o = reflib.center_table(cen)
    assert same(t.dist2, d) and same(t.order, o)
    assert all(t.order_at(i, 0) == i for i in range(K))


def test_center_table_reference_case(ctx):
    # tests/test_kmeans.cpp:23-55
    t = quant.build_center_distance_table(np.array([[0, 0, 0], [10, 0, 0], [3, 0, 0]], float), ctx=ctx)
    assert t.d2(0, 1) == 100.0 and t.d2(0, 2) == 9.0 and t.d2(1, 2) == 49.0
    assert [t.order_at(0, j) for j in range(3)] == [0, 2, 1]
    assert [t.order_at(1, j) for j in range(3)] == [1, 2, 0]
    t = quant.build_center_distance_table(np.array([[5, 5, 5], [5, 5, 5], [9, 9, 9]], float), ctx=ctx)
    assert t.order_at(0, 0) == 0 and t.order_at(1, 0) == 1


def test_kmeanspp_next_masses_and_maximin_pad(ctx, reflib):
    rng = np.random.default_rng(21)
    cols = distinct_colors(rng, 3000)
    w = random_weights(rng, 3000)
    hist = quant.WeightedHistogram(cols, w, np.ones(3000, np.uint32), 3000)
    for k0 in (0, 1, 5):
        got = quant.kmeanspp_next_masses(hist, cols[:k0], ctx=ctx)
        assert same(got, reflib.next_masses(cols, w, cols[:k0]))
    short = rng.random((3, 3)) * 255.0  # a preclusterer's real-valued palette
    got = quant.maximin_pad(hist, short, 40, ctx=ctx)
    assert same(got, reflib.maximin_pad(cols, w, short, 40))
    assert same(quant.maximin_pad(hist, cols[:50], 40, ctx=ctx), cols[:50])  # long enough: unchanged
    with pytest.raises(ValueError, match="need at least one center"):
        quant.maximin_pad(hist, np.zeros((0, 3)), 4, ctx=ctx)


def test_maximin_pad_reference_case(ctx):
    # tests/test_init.cpp:296-311 shape: a 3-colour histogram, pad 1 -> 3
    cols = np.array([[0, 0, 0], [255, 0, 0], [0, 0, 255]], float)
    hist = quant.WeightedHistogram(cols, np.full(3, 1 / 3), np.ones(3, np.uint32), 3)
    got = quant.maximin_pad(hist, cols[:1], 3, ctx=ctx)
    assert same(got[0], cols[0]) and {tuple(x) for x in got} == {tuple(x) for x in cols}
