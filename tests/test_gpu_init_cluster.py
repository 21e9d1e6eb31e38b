"""Cluster initialiser variants (substrates up to 16 x 1024 x 12 colours),
bit-exact against the oracle: the register-resident kernel (default: the CTA
shape with the fewest padded slots; CQG_CLUSTER_NT forces 512..1024 threads)
at each points-per-thread instantiation and both mass arithmetics (P a
power of two: exact integers; otherwise 2^-88 fixed point), and the register
kernel's rare sequential paths forced on every draw (CQG_DBG_INIT_FORCE_SEQ=1: ambiguous decision; =2: target beyond
every prefix) -- the reference replay must give the same centres.
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
    cs = {"reg": _ctx(),
          "nt1024": _ctx(CQG_CLUSTER_NT="1024"),
          "nt896": _ctx(CQG_CLUSTER_NT="896"),
          "nt768": _ctx(CQG_CLUSTER_NT="768"),
          "nt640": _ctx(CQG_CLUSTER_NT="640"),
          "nt512": _ctx(CQG_CLUSTER_NT="512"),
          "force_amb": _ctx(CQG_DBG_INIT_FORCE_SEQ="1"),
          "force_nf": _ctx(CQG_DBG_INIT_FORCE_SEQ="2")}
    yield cs
    for c in cs.values():
        c.close()


def _ppt(n):
    per = -(-n // 16)
    return (-(-per // 1024) + 3) & ~3


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


# (w, h, noise, K, seed, points per thread); P = w*h a power of two or not
CASES = [(256, 256, 0.3, 64, 3, 4), (300, 200, 0.02, 64, 9, 4),
         (512, 256, 0.3, 128, 5, 8), (360, 300, 0.5, 96, 7, 8),
         (512, 512, 0.02, 256, 5, 12), (384, 384, 0.6, 200, 11, 12)]


@pytest.mark.parametrize("variant", ["reg", "nt1024", "nt896", "nt768", "nt640", "nt512"])
@pytest.mark.parametrize("w,h,noise,K,seed,ppt", CASES)
def test_init_cluster_variants(ctxs, oracle, variant, w, h, noise, K, seed, ppt):
    img = synth_image(w, h, 5, nblobs=10, sigma=15.0, noise=noise)
    n = _check(ctxs[variant], oracle, img, K, seed)
    assert _ppt(n) == ppt


@pytest.mark.parametrize("variant", ["force_amb", "force_nf"])
@pytest.mark.parametrize("w,h,K,seed", [(40, 40, 8, 3), (64, 48, 16, 4), (128, 128, 12, 6)])
def test_init_cluster_sequential_paths(ctxs, oracle, variant, w, h, K, seed):
    img = synth_image(w, h, seed, nblobs=10, sigma=15.0, noise=0.02)
    _check(ctxs[variant], oracle, img, K, seed)


@pytest.mark.parametrize("variant", ["reg", "nt1024", "nt896", "nt768", "nt640", "nt512"])
@pytest.mark.parametrize("w,h", [(400, 400), (448, 400), (300, 260)])
def test_init_cluster_shapes_near_unique(ctxs, oracle, variant, w, h):
    # near-all-unique colours: every CTA shape at its largest points per
    # thread (the forced sizes fall back to 1024 threads when they do not fit)
    img = np.random.default_rng(w + h).integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    _check(ctxs[variant], oracle, img, 64, 4)


def test_init_cluster_tiny_and_duplicates(ctxs, oracle):
    # fewer colours than CTAs x threads: most threads and whole CTAs own padding only
    rng = np.random.default_rng(1)
    for ctx in (ctxs["reg"], ctxs["nt1024"]):
        img = rng.integers(0, 3, size=(17, 13, 3), dtype=np.uint8) * 100
        n = quant.build_histogram(img, ctx=ctx).packed.size
        _check(ctx, oracle, img, min(n, 5), 2)
        img = np.zeros((7, 5, 3), np.uint8)
        img[0, 0] = 255
        _check(ctx, oracle, img, 2, 1)
