"""Distance-bound pruning of the WALK sweep.

Points whose label is proven unchanged by the (ub, lb) bounds skip the centre
loop. The bar is unchanged: labels, iterations, NDC, repairs, centres and SSE
bit-exact against the oracle. These cases add the paths the other parity tests
do not reach with pruning on: the CUDA-graph loop (N' above the persistent
kernel's limit), the persistent kernel without history, repairs after pruned
iterations, and pruned == unpruned on the same inputs.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import UPDATE_EXACT
from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import CONFIGS, synth_image

from test_gpu_parity import assert_lloyd_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx_noprune():
    old = os.environ.get("CQG_NO_PRUNE")
    os.environ["CQG_NO_PRUNE"] = "1"
    try:
        c = cabi.Context(0)
    finally:
        if old is None:
            del os.environ["CQG_NO_PRUNE"]
        else:
            os.environ["CQG_NO_PRUNE"] = old
    yield c
    c.close()


def _run(ctx, c, n, P, init, **term):
    opts = quant.ClusterOptions(quant.Termination(**term)) if term else quant.ClusterOptions()
    return quant.wsm_counts(c, n, P, init, opts, ctx=ctx)


def test_prune_persistent_path(ctx, ctx_noprune, oracle):
    # cfg2 substrate (N' = 168K): the persistent cooperative kernel, no history
    cfg = CONFIGS["cfg2"]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    c, n = hist.packed, hist.counts
    init = oracle.init_kmeanspp(c, n, P, cfg.k, cfg.seed)
    dev = _run(ctx, c, n, P, init)
    ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT)
    assert_lloyd_equal(dev, ora, P)
    dense = _run(ctx_noprune, c, n, P, init)
    assert_lloyd_equal(dense, ora, P)
    assert dense.swept_total == c.size * dense.iterations
    # pruning is active: later iterations sweep a fraction of the points (the
    # persistent loop keeps only the Hamerly bound: DESIGN.md section 4)
    assert dev.swept_total < 0.75 * c.size * dev.iterations


def test_prune_graph_path(ctx, ctx_noprune, oracle):
    # N' above the persistent limit (148*2*256*8 = 606K): sweep kernels in the CUDA graph loop
    img = synth_image(1400, 1400, 909, nblobs=40, sigma=30.0, noise=0.5)
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    c, n = hist.packed, hist.counts
    assert c.size > 620_000
    init = oracle.init_maximin(c, n, P, 64, 909)
    dev = _run(ctx, c, n, P, init, max_iterations=25)
    ora = oracle.wsm(c, n, P, init, max_it=25, mode=UPDATE_EXACT)
    assert_lloyd_equal(dev, ora, P)
    assert dev.swept_total < 0.6 * c.size * dev.iterations
    dense = _run(ctx_noprune, c, n, P, init, max_iterations=25)
    assert np.array_equal(dense.memberships, dev.memberships)
    assert np.array_equal(dense.centers.view(np.uint64), dev.centers.view(np.uint64))


def test_prune_fixed_iterations_long_run(ctx, oracle):
    # many iterations after convergence: bounds keep tightening, labels never move
    img = CONFIGS["cfg1"].image()
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    c, n = hist.packed, hist.counts
    init = oracle.init_maximin(c, n, P, 32, 101)
    dev = _run(ctx, c, n, P, init, fixed_iterations=60)
    ora = oracle.wsm(c, n, P, init, fixed_it=60, mode=UPDATE_EXACT)
    assert dev.iterations == 60
    assert_lloyd_equal(dev, ora, P)


@pytest.mark.parametrize("seed", range(6))
def test_prune_repairs_and_small_substrates(ctx, ctx_noprune, oracle, seed):
    # few unique colours, K close to N': empty clusters appear (also after
    # pruned iterations); repairs must void the bounds
    rng = np.random.default_rng(1000 + seed)
    nu = int(rng.integers(40, 400))
    keys = rng.choice(1 << 24, nu, replace=False).astype(np.uint32)
    counts = rng.integers(1, 50, nu).astype(np.uint32)
    P = int(counts.sum())
    K = int(rng.integers(nu // 4, nu // 2 + 2))
    pts = quant.unpack_colors(keys).astype(np.float64)
    # clumped init: many centres start near each other -> empties
    init = pts[rng.integers(0, 6, K)] + rng.normal(0, 0.5, (K, 3))
    dev = _run(ctx, keys, counts, P, init, max_iterations=40)
    ora = oracle.wsm(keys, counts, P, init, max_it=40, mode=UPDATE_EXACT)
    assert_lloyd_equal(dev, ora, P)
    dense = _run(ctx_noprune, keys, counts, P, init, max_iterations=40)
    assert_lloyd_equal(dense, ora, P)


@pytest.mark.parametrize("history", [True, False])
def test_ndc_code_table_exact_ties(ctx, oracle, history):
    # Integer centres 6 apart on the red axis; each cluster = its centre plus
    # c +- 3 on green / blue, so the means stay integer. From iteration 2 the
    # NDC cutoff 4*pd = 36 equals the neighbour distance D = 36 exactly: the
    # 16-bit code of the cutoff ties with the row entry and the FP64 value decides.
    cen = np.array([[20 + 6 * i, 128, 128] for i in range(36)], np.int64)
    pts = []
    for c in cen:
        pts.append(c)
        for off in ([0, 3, 0], [0, -3, 0], [0, 0, 3], [0, 0, -3]):
            pts.append(c + np.array(off))
    pts = np.array(pts, np.uint8)
    keys = quant.pack_colors(pts)
    counts = np.ones(keys.size, np.uint32)
    P = keys.size
    init = cen.astype(np.float64) + 0.25
    opts = quant.ClusterOptions(quant.Termination(fixed_iterations=4), record_history=history)
    dev = quant.wsm_counts(keys, counts, P, init, opts, ctx=ctx)
    ora = oracle.wsm(keys, counts, P, init, fixed_it=4, mode=UPDATE_EXACT, history=history)
    assert_lloyd_equal(dev, ora, P)


@pytest.mark.parametrize("w,h,k,fixed", [(300, 200, 32, 1), (300, 200, 32, 2), (700, 500, 64, 0), (900, 800, 16, 0)])
def test_pruned_mapping(ctx, ctx_noprune, oracle, w, h, k, fixed):
    # run_quantize ('unique' sampling) maps the image through the bounds Lloyd
    # left behind (MODE_MAPW): after the FULL iteration only (fixed 1), after a
    # WALK iteration, through the persistent kernel (<= 606K colours) and the
    # graph loop (900x800 with noise). Indices, pixels and MSE are bit-exact
    # against the oracle's mapping and against the unpruned context.
    img = synth_image(w, h, 77 + k, nblobs=10, sigma=14.0, noise=0.5 if w == 900 else 0.03)
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-kpp"), k=k, seed=k,
                              term=quant.Termination(fixed_iterations=fixed or None))
    r = quant.run_quantize(img, qc, ctx=ctx)
    idx, q, mse_e, _ = oracle.map_pixels(img, r.palette, mode=UPDATE_EXACT)
    assert np.array_equal(r.mapping.indices, idx)
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), q)
    assert r.report.mse == mse_e
    r0 = quant.run_quantize(img, qc, ctx=ctx_noprune)
    assert np.array_equal(r0.palette, r.palette)
    assert np.array_equal(r0.mapping.indices, r.mapping.indices)
    assert r0.report.mse == r.report.mse


@pytest.mark.parametrize("dup", [1, 3])
def test_quantize_repair_after_deferred_check(ctx, oracle, dup):
    # run_quantize checks the persistent Lloyd kernel's status only after the
    # mapping is enqueued; duplicated initial centres leave clusters empty in
    # the first iteration, so the run must fall back to the repairing loop and
    # map again. Everything bit-exact against the oracle pipeline.
    img = synth_image(96, 80, 41 + dup, nblobs=7, sigma=16.0, noise=0.05)
    P = 96 * 80
    rng = np.random.default_rng(dup)
    init = rng.integers(0, 256, (12, 3)).astype(np.float64)
    init[1:1 + dup] = init[0]  # clusters 1..dup tie with 0 and lose: empty
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-kpp"), k=12, seed=1)
    r = quant.run_quantize(img, qc, ctx=ctx, init_centers=init)
    c, n, _ = oracle.histogram(img)
    ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT)
    assert ora.repairs >= 1
    assert r.state.repair_count == ora.repairs
    assert r.state.iterations == ora.iterations
    assert r.state.ndc_total == ora.ndc_total
    assert np.array_equal(r.palette, ora.centers)
    assert np.array_equal(r.state.memberships, ora.labels)
    idx, q, mse_e, _ = oracle.map_pixels(img, ora.centers, mode=UPDATE_EXACT)
    assert np.array_equal(r.mapping.indices, idx)
    assert np.array_equal(r.mapping.quantized.reshape(-1, 3), q)
    assert r.report.mse == mse_e


@pytest.fixture(scope="module")
def ctx_win3():
    # the persistent loop's deferred-NDC window capped at 3 WALK iterations:
    # every launch ends in the window-full state and the host relaunches
    old = os.environ.get("CQG_DBG_NDC_WIN")
    os.environ["CQG_DBG_NDC_WIN"] = "3"
    try:
        c = cabi.Context(0)
    finally:
        if old is None:
            del os.environ["CQG_DBG_NDC_WIN"]
        else:
            os.environ["CQG_DBG_NDC_WIN"] = old
    yield c
    c.close()


def test_deferred_ndc_window_relaunch(ctx_win3, oracle):
    # cfg2 substrate, 20 iterations in launches of 3: NDC, labels, centres, SSE
    # bit-exact; then the pipeline (deferred status check -> synchronous rerun)
    cfg = CONFIGS["cfg2"]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx_win3)
    c, n = hist.packed, hist.counts
    init = oracle.init_kmeanspp(c, n, P, cfg.k, cfg.seed)
    dev = _run(ctx_win3, c, n, P, init)
    ora = oracle.wsm(c, n, P, init, mode=UPDATE_EXACT)
    assert ora.iterations > 7
    assert_lloyd_equal(dev, ora, P)
    qc = quant.QuantizeConfig(method=quant.parse_method("wsm-kpp"), k=cfg.k, seed=cfg.seed)
    r = quant.run_quantize(img, qc, ctx=ctx_win3)
    assert r.state.iterations == ora.iterations
    assert r.state.ndc_total == ora.ndc_total
    assert np.array_equal(r.palette, ora.centers)


@pytest.mark.parametrize("seed", range(3))
def test_deferred_ndc_window_with_repairs(ctx_win3, oracle, seed):
    rng = np.random.default_rng(2000 + seed)
    nu = int(rng.integers(60, 400))
    keys = rng.choice(1 << 24, nu, replace=False).astype(np.uint32)
    counts = rng.integers(1, 50, nu).astype(np.uint32)
    P = int(counts.sum())
    K = int(rng.integers(nu // 4, nu // 2 + 2))
    pts = quant.unpack_colors(keys).astype(np.float64)
    init = pts[rng.integers(0, 6, K)] + rng.normal(0, 0.5, (K, 3))
    dev = _run(ctx_win3, keys, counts, P, init, max_iterations=40)
    ora = oracle.wsm(keys, counts, P, init, max_it=40, mode=UPDATE_EXACT)
    assert_lloyd_equal(dev, ora, P)


def test_prune_graph_path_in_sweep_filter(oracle):
    # CQG_NO_FILTER_LIST=1: the stay test inside the sweep kernel (no separate
    # survivor-list pass) on the graph path; bit-exact like the default
    old = os.environ.get("CQG_NO_FILTER_LIST")
    os.environ["CQG_NO_FILTER_LIST"] = "1"
    try:
        c0 = cabi.Context(0)
    finally:
        if old is None:
            del os.environ["CQG_NO_FILTER_LIST"]
        else:
            os.environ["CQG_NO_FILTER_LIST"] = old
    try:
        img = synth_image(1400, 1400, 909, nblobs=40, sigma=30.0, noise=0.5)
        P = img.shape[0] * img.shape[1]
        hist = quant.build_histogram(img, ctx=c0)
        c, n = hist.packed, hist.counts
        init = oracle.init_maximin(c, n, P, 64, 909)
        dev = _run(c0, c, n, P, init, max_iterations=12)
        ora = oracle.wsm(c, n, P, init, max_it=12, mode=UPDATE_EXACT)
        assert_lloyd_equal(dev, ora, P)
    finally:
        c0.close()
