"""Initialisers on the cooperative (large substrate) kernels: bit-exact
against the oracle for the two grid layouts -- colour-space tiles with box
pruning (default) and {colour, md} records in histogram order
(CQG_NO_INIT_TILE=1) -- and for
both mass arithmetics (P a power of two: exact integers; otherwise 2^-88
fixed point with the sequential FP64 fallback). Small inputs reach the same
kernels with the cluster initialiser switched off (CQG_NO_CLUSTER_INIT=1).
A substrate with repeated colours (no one-colour-per-slot tile layout) falls
back to the record layout.
"""
import os

import numpy as np
import pytest

from paper_1101_0395_b200 import cabi, quant
from paper_1101_0395_b200.synth import synth_image

pytestmark = pytest.mark.gpu


def _ctx(**env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return cabi.Context(0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def ctxs():
    cs = {"tile": _ctx(CQG_NO_CLUSTER_INIT="1", CQG_INIT_TILE_MIN="0"),
          "rec": _ctx(CQG_NO_CLUSTER_INIT="1", CQG_NO_INIT_TILE="1")}
    yield cs
    for c in cs.values():
        c.close()


def _check(ctx, oracle, img, K, seed):
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    c, n = hist.packed, hist.counts
    sc = quant.SeedConfig(k=K, seed=seed)
    assert np.array_equal(quant.init_kmeanspp(hist, sc, ctx=ctx), oracle.init_kmeanspp(c, n, P, K, seed))
    assert np.array_equal(quant.init_maximin(hist, sc, ctx=ctx), oracle.init_maximin(c, n, P, K, seed))
    sc_u = quant.SeedConfig(k=K, seed=seed, maximin_weighted_first=False)
    assert np.array_equal(quant.init_maximin(hist, sc_u, ctx=ctx),
                          oracle.init_maximin(c, n, P, K, seed, weighted_first=False))
    return c.size


@pytest.mark.parametrize("layout", ["tile", "rec"])
@pytest.mark.parametrize("w,h,K,seed", [(40, 40, 8, 3), (300, 200, 64, 9), (512, 512, 33, 5)])
def test_init_cooperative_small(ctxs, oracle, layout, w, h, K, seed):
    img = synth_image(w, h, seed, nblobs=10, sigma=15.0, noise=0.02)
    _check(ctxs[layout], oracle, img, K, seed)


@pytest.mark.parametrize("layout", ["tile", "rec"])
@pytest.mark.parametrize("w,h", [(1024, 1024), (1100, 900)])  # P = 2^20 (exact) / not a power of two
def test_init_cooperative_large(ctxs, ctx, oracle, layout, w, h):
    img = synth_image(w, h, 4242, nblobs=30, sigma=25.0, noise=0.7)
    n = _check(ctxs[layout], oracle, img, 64, 4242)
    assert n > 16 * 1024 * 32  # beyond the cluster initialiser
    # the default context takes the same path at this size
    _check(ctx, oracle, img, 64, 4242)


@pytest.mark.parametrize("kind", ["kpp", "mmx"])
def test_init_tile_repeated_colours(ctxs, oracle, kind):
    # every colour twice (with different counts): two points share a Morton
    # slot, so the tile layout declines and the record layout runs
    rng = np.random.default_rng(17)
    base = np.unique(rng.integers(0, 1 << 24, 150_000, dtype=np.uint32))
    c = np.concatenate([base, base[::-1]]).astype(np.uint32)
    n = rng.integers(1, 5, c.size).astype(np.uint32)
    P = int(n.sum())
    hist = quant.WeightedHistogram(colors=quant.unpack_colors(c), weights=n / P, counts=n,
                                   source_pixel_count=P, packed=c)
    sc = quant.SeedConfig(k=48, seed=6)
    f, o = (quant.init_kmeanspp, oracle.init_kmeanspp) if kind == "kpp" else (quant.init_maximin, oracle.init_maximin)
    for layout in ("tile", "rec"):
        assert np.array_equal(f(hist, sc, ctx=ctxs[layout]), o(c, n, P, 48, 6))


def test_init_tile_sparse_colours(ctxs, oracle):
    # colours spread thin over the cube (large tile boxes, little pruning) and
    # clustered ones (tight boxes) in one substrate
    rng = np.random.default_rng(23)
    sparse = rng.integers(0, 1 << 24, 200_000, dtype=np.uint32)
    blob = (np.clip(rng.normal(128, 6, (600_000, 3)), 0, 255).astype(np.uint32))
    dense = (blob[:, 0] << 16) | (blob[:, 1] << 8) | blob[:, 2]
    c = np.unique(np.concatenate([sparse, dense]))
    rng.shuffle(c)
    c = c.astype(np.uint32)
    n = rng.integers(1, 4, c.size).astype(np.uint32)
    P = int(n.sum())
    hist = quant.WeightedHistogram(colors=quant.unpack_colors(c), weights=n / P, counts=n,
                                   source_pixel_count=P, packed=c)
    sc = quant.SeedConfig(k=96, seed=11)
    assert np.array_equal(quant.init_kmeanspp(hist, sc, ctx=ctxs["tile"]), oracle.init_kmeanspp(c, n, P, 96, 11))
    assert np.array_equal(quant.init_maximin(hist, sc, ctx=ctxs["tile"]), oracle.init_maximin(c, n, P, 96, 11))


@pytest.mark.slow
def test_init_bench_size_cfg3(ctx, oracle):
    # the cfg3 substrate (6.3M colours): the grid size and the per-block segment
    # count reach their largest values here (warp_locate capacity, kLocateMax)
    from paper_1101_0395_b200.synth import CONFIGS
    cfg = CONFIGS["cfg3"]
    img = cfg.image()
    P = img.shape[0] * img.shape[1]
    hist = quant.build_histogram(img, ctx=ctx)
    c, n = hist.packed, hist.counts
    sc = quant.SeedConfig(k=cfg.k, seed=cfg.seed)
    assert np.array_equal(quant.init_maximin(hist, sc, ctx=ctx), oracle.init_maximin(c, n, P, cfg.k, cfg.seed))
    assert np.array_equal(quant.init_kmeanspp(hist, sc, ctx=ctx), oracle.init_kmeanspp(c, n, P, cfg.k, cfg.seed))
